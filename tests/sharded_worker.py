"""One rank of a multi-process sharded solve (tests/test_gpu_sharded.py):
gloo process group on 127.0.0.1, the library's sharded path with a
HostCommunicator whose all-reduce is torch.distributed over gloo.  Every rank
drives the same GPU (cuda:0); their kernels never wait on one another -- the
exchange is on the host.

    python tests/sharded_worker.py RANK WORLD PORT OUT.npz CFG D N BACKEND ITERS
"""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    rank, world, port, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    cfgname, d, n, backend, iters = sys.argv[5], int(sys.argv[6]), int(sys.argv[7]), sys.argv[8], int(sys.argv[9])
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2305_12019_b200 as G
    from paper_2305_12019_b200 import parallel, synth

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)

    def allreduce(x):
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy()

    prob = synth.make_problem(synth.CONFIGS[cfgname].scaled(d=d, n=n), 0)
    local = parallel.shard_problem(prob, rank, world)
    parallel.attach(local, parallel.HostCommunicator(allreduce, world, rank), n, 0)
    res = G.sgs_admm_solve(local, G.SolverConfig(q=prob.q, max_iter=iters, backend=G.Backend(backend)))
    np.savez(out, w=res.final_state.w, alpha=res.final_state.alpha, beta=res.final_state.beta,
             iterations=res.iterations, double_count=res.double_count, psqmr_total=res.psqmr_total,
             train_error=res.train_error_pct, obj_primal=res.final_residuals.obj_primal)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
