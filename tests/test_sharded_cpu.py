"""N>1 sample sharding on CPU: world_size-2 gloo process group.

Each rank takes its block of samples (paper_2305_12019_b200.parallel.shard_problem,
the same host logic the GPU path uses) and runs the sharded restatement of
the iteration (oracle.solve with allreduce = torch.distributed gloo), which
mirrors the device decomposition: every sum over samples all-reduced,
feature-space work replicated.  Rank 0 compares with the unsharded solve."""

import os
import socket

import numpy as np
import pytest

CASES = [  # (synth config, d, n, backend, iterations)
    ("c3", 40, 300, "direct", 25),
    ("c1", 60, 90, "iterative", 25),
    ("c4", 3000, 2000, "iterative", 15),
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from oracle import gdwd_oracle as O
    from paper_2305_12019_b200 import parallel, synth

    dist.init_process_group("gloo", rank=rank, world_size=world)

    def ar(v):
        t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).clone()
        dist.all_reduce(t)
        return t.numpy()

    out = []
    for cfgname, d, n, backend, iters in CASES:
        prob = synth.make_problem(synth.CONFIGS[cfgname].scaled(d=d, n=n), 0)
        local = parallel.shard_problem(prob, rank, world)
        cfg = O.OracleConfig(max_iter=iters, backend=backend)
        r = O.solve(local, cfg, operator="csc", allreduce=ar, n_global=n, record=False)
        lo, hi = parallel.shard_bounds(n, world, rank)
        out.append(dict(w=r.state["w"], beta=r.state["beta"], r=r.state["r"], alpha=r.state["alpha"], lo=lo,
                        hi=hi, iterations=r.iterations, doubles=r.double_count, psqmr=r.psqmr_total,
                        err=r.train_error_pct, res=r.residuals))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_bounds_cover():
    from paper_2305_12019_b200 import parallel

    for n in (1, 7, 1000):
        for world in (1, 2, 3, 8):
            b = [parallel.shard_bounds(n, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))


def test_shard_problem_sparse_and_dense():
    from paper_2305_12019_b200 import parallel, synth

    for name, d, n in (("c1", 30, 50), ("c4", 2000, 700)):
        prob = synth.make_problem(synth.CONFIGS[name].scaled(d=d, n=n), 0)
        parts = [parallel.shard_problem(prob, r, 3) for r in range(3)]
        full = prob.z_tilde.toarray()
        back = np.concatenate([p.z_tilde.toarray() for p in parts], axis=1)
        assert np.array_equal(full, back)
        assert np.array_equal(np.concatenate([p.y for p in parts]), prob.y)


def test_sharded_two_ranks_gloo_matches_unsharded():
    import multiprocessing as mp

    from oracle import gdwd_oracle as O
    from paper_2305_12019_b200 import synth

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for ci, (cfgname, d, n, backend, iters) in enumerate(CASES):
        prob = synth.make_problem(synth.CONFIGS[cfgname].scaled(d=d, n=n), 0)
        ref = O.solve(prob, O.OracleConfig(max_iter=iters, backend=backend), operator="csc", record=False)
        a, b = res[0][ci], res[1][ci]
        # replicated feature-space state is identical on both ranks
        assert np.array_equal(a["w"], b["w"]) and a["beta"] == b["beta"]
        assert a["iterations"] == ref.iterations and a["doubles"] == ref.double_count
        assert abs(a["psqmr"] - ref.psqmr_total) <= 1
        rel = np.linalg.norm(a["w"] - ref.state["w"]) / np.linalg.norm(ref.state["w"])
        assert rel < 1e-9, (cfgname, rel)
        for part in (a, b):
            sl = slice(part["lo"], part["hi"])
            assert np.linalg.norm(part["r"] - ref.state["r"][sl]) <= 1e-9 * np.linalg.norm(ref.state["r"][sl])
            assert np.linalg.norm(part["alpha"] - ref.state["alpha"][sl]) <= 1e-9 * (
                1 + np.linalg.norm(ref.state["alpha"][sl]))
        assert a["err"] == ref.train_error_pct
        assert abs(a["res"]["obj_primal"] - ref.residuals["obj_primal"]) <= 1e-9 * abs(ref.residuals["obj_primal"])
