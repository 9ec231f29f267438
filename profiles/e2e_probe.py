"""End-to-end timing of sgs_admm_solve from pinned host buffers (the bench's
e2e leg), repeated: upload / solve-call / download split and the library's
setup / loop device times.  python profiles/e2e_probe.py [config] [iters] [reps]"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
import torch
import paper_2305_12019_b200 as G
from paper_2305_12019_b200 import synth

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
prob = synth.make_problem(synth.CONFIGS[cfgname], 0)
z = prob.z_tilde
buf = torch.empty(z.values.size, dtype=torch.float64, pin_memory=True).numpy()
buf[:] = z.values
for rep in range(reps):
    zp = G.SparseMatrixCSC.from_dense_samples(buf.reshape(z.ncols, z.nrows))
    pp = G.ProblemData(zp, prob.y, prob.e, prob.weights, prob.C, prob.q, prob.z_scale)
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = G.sgs_admm_solve(pp, G.SolverConfig(q=pp.q, max_iter=iters))
    dt = time.perf_counter() - t
    G.solver.device_problem(pp).close()
    print(f"rep {rep}: {dt*1e3:7.3f} ms  {iters/dt:8.1f} it/s  " +
          "  ".join(f"{k}={v*1e3 if k.endswith('_s') else v:.3f}" for k, v in out.timings.items()), flush=True)

# finer split of the upload leg: context creation, upload call, set_problem
import ctypes as C
from paper_2305_12019_b200 import _lib
lib = _lib.load()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = C.c_void_p()
    lib.gdwd_ctx_create(0, C.byref(h))
    t1 = time.perf_counter()
    lib.gdwd_upload_hint(h, 0, 1.0)
    lib.gdwd_upload_dense(h, _lib.ptr(buf), prob.d, prob.n)
    t2 = time.perf_counter()
    lib.gdwd_set_problem(h, _lib.ptr(prob.y), _lib.ptr(prob.e), _lib.ptr(prob.weights), prob.C, prob.q, prob.z_scale)
    t3 = time.perf_counter()
    lib.gdwd_ctx_destroy(h)
    t4 = time.perf_counter()
    print(f"ctx_create {1e3*(t1-t0):.3f}  upload {1e3*(t2-t1):.3f}  set_problem {1e3*(t3-t2):.3f}  destroy {1e3*(t4-t3):.3f} ms")
