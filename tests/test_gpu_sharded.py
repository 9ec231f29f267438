"""Sample-sharded device path on one GPU (pytest -m gpu).

* NCCL communicator with a single rank: exercises the partial kernels, the
  all-reduce calls (inside the captured CUDA graph) and the epilogue kernels.
* Two virtual ranks: two host threads, each with its own context and shard on
  the same GPU, exchanging bundles through a host all-reduce (the kernels of
  the two ranks never wait on one another on the device)."""

import threading

import numpy as np
import pytest

import paper_2305_12019_b200 as G
from paper_2305_12019_b200 import parallel, synth

pytestmark = pytest.mark.gpu

CASES = [("c3", 400, 3000, "direct", 30), ("c1", 6000, 1500, "iterative", 12), ("c4", 8000, 30000, "iterative", 12)]


def relerr(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("case", CASES, ids=[c[0] + c[3] for c in CASES])
def test_nccl_single_rank_matches_unsharded(case):
    name, d, n, backend, iters = case
    prob = synth.make_problem(synth.CONFIGS[name].scaled(d=d, n=n), 0)
    cfg = G.SolverConfig(q=prob.q, max_iter=iters, backend=G.Backend(backend))
    ref = G.sgs_admm_solve(prob, cfg)
    local = parallel.shard_problem(prob, 0, 1)
    comm = parallel.NcclCommunicator(1, 0, lambda uid: uid)
    parallel.attach(local, comm, n)
    out = G.sgs_admm_solve(local, cfg)
    assert out.iterations == ref.iterations and out.double_count == ref.double_count
    assert relerr(out.final_state.w, ref.final_state.w) < 1e-10
    assert relerr(out.final_state.alpha, ref.final_state.alpha) < 1e-10


@pytest.mark.parametrize("case", CASES, ids=[c[0] + c[3] for c in CASES])
def test_two_virtual_ranks_match_unsharded(case):
    name, d, n, backend, iters = case
    prob = synth.make_problem(synth.CONFIGS[name].scaled(d=d, n=n), 0)
    cfg = G.SolverConfig(q=prob.q, max_iter=iters, backend=G.Backend(backend))
    ref = G.sgs_admm_solve(prob, cfg)
    world = 2
    ranks = parallel.ThreadRanks(world)
    locals_ = [parallel.shard_problem(prob, r, world) for r in range(world)]
    for r in range(world):
        G.device_problem(locals_[r], 0)  # upload serially
    outs, errs = [None] * world, []

    def run(r):
        try:
            comm = parallel.HostCommunicator(ranks.allreduce_for(r), world, r)
            parallel.attach(locals_[r], comm, n)
            outs[r] = G.sgs_admm_solve(locals_[r], cfg)
        except BaseException as exc:
            errs.append(exc)
            ranks.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    a, b = outs
    assert np.array_equal(a.final_state.w, b.final_state.w)  # replicated state identical
    assert a.iterations == ref.iterations and a.double_count == ref.double_count
    assert relerr(a.final_state.w, ref.final_state.w) < 1e-9
    for r, o in enumerate(outs):
        lo, hi = parallel.shard_bounds(n, world, r)
        assert relerr(o.final_state.alpha, ref.final_state.alpha[lo:hi]) < 1e-9
    assert abs(a.final_residuals.obj_primal - ref.final_residuals.obj_primal) <= 1e-9 * abs(
        ref.final_residuals.obj_primal)


def _ref_solve(case):
    name, d, n, backend, iters = case
    prob = synth.make_problem(synth.CONFIGS[name].scaled(d=d, n=n), 0)
    cfg = G.SolverConfig(q=prob.q, max_iter=iters, backend=G.Backend(backend))
    return prob, cfg, G.sgs_admm_solve(prob, cfg)


@pytest.mark.parametrize("case", CASES, ids=[c[0] + c[3] for c in CASES])
def test_solve_on_devices_one_process(case):
    """The single-process multi-device entry point (sgs_admm_solve(...,
    devices=[...])): two ranks on one GPU through the host exchange, and one
    NCCL rank; global train error and concatenated sample-space iterates."""
    prob, cfg, ref = _ref_solve(case)
    for devices, comm in (([0, 0], "host"), ([0], "nccl")):
        out = parallel.solve_on_devices(prob, cfg, devices, comm=comm)
        assert out.iterations == ref.iterations and out.double_count == ref.double_count, comm
        assert relerr(out.final_state.w, ref.final_state.w) < 1e-9, comm
        assert relerr(out.final_state.alpha, ref.final_state.alpha) < 1e-9, comm
        assert out.final_state.alpha.shape == ref.final_state.alpha.shape
        assert out.train_error_pct == ref.train_error_pct, comm


def test_two_processes_gloo_one_gpu(tmp_path):
    """Two OS processes (gloo over 127.0.0.1), each running the library's
    sharded path on its half of the samples; the replicated state is
    bit-identical on both and matches the unsharded solve."""
    import os
    import socket
    import subprocess
    import sys

    case = CASES[0]
    prob, cfg, ref = _ref_solve(case)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    worker = os.path.join(os.path.dirname(__file__), "sharded_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), "2", str(port), str(tmp_path / f"r{r}.npz"),
                               case[0], str(case[1]), str(case[2]), case[3], str(case[4])])
             for r in range(2)]
    for p in procs:
        assert p.wait(timeout=600) == 0
    a, b = (np.load(tmp_path / f"r{r}.npz") for r in range(2))
    assert np.array_equal(a["w"], b["w"]) and float(a["beta"]) == float(b["beta"])
    assert int(a["iterations"]) == ref.iterations and int(a["double_count"]) == ref.double_count
    assert relerr(a["w"], ref.final_state.w) < 1e-9
    assert relerr(np.concatenate([a["alpha"], b["alpha"]]), ref.final_state.alpha) < 1e-9
    assert float(a["train_error"]) == float(b["train_error"]) == ref.train_error_pct
    assert abs(float(a["obj_primal"]) - ref.final_residuals.obj_primal) <= 1e-9 * abs(ref.final_residuals.obj_primal)
