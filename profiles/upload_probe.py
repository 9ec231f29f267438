import os, sys, time, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2305_12019_b200 as G
from paper_2305_12019_b200 import synth
prob = synth.make_problem(synth.CONFIGS["c2"], 0)
for mode in ["pageable", "register", "staged", "staged", "pageable", "register"]:
    os.environ["GDWD_UPLOAD"] = mode
    t = time.perf_counter(); dp = G.DeviceProblem(prob, 0); dt = time.perf_counter() - t
    print(mode, f"{dt*1e3:.1f} ms  {8*prob.n*prob.d/dt/1e9:.1f} GB/s", flush=True); dp.close()
