import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_2305_12019_b200 as G
from paper_2305_12019_b200 import synth
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
prob = synth.make_problem(synth.CONFIGS[cfgname], 0)
for rep in range(5):
    pp = G.ProblemData(prob.z_tilde, prob.y, prob.e, prob.weights, prob.C, prob.q, prob.z_scale)
    t = time.perf_counter()
    out = G.sgs_admm_solve(pp, G.SolverConfig(q=pp.q, max_iter=20))
    dt = time.perf_counter() - t
    G.solver.device_problem(pp).close()
    print(f"pageable rep {rep}: {dt*1e3:7.3f} ms  " + "  ".join(f"{k}={v*1e3 if k.endswith('_s') else v:.3f}" for k, v in out.timings.items()), flush=True)
