"""Small driver for ncu captures: config 2, Gram-space SMW2, a few solves."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2305_12019_b200 as G
from paper_2305_12019_b200 import synth

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
prob = synth.make_problem(synth.CONFIGS["c2"], 0)
for rep in range(2):
    t = time.perf_counter()
    out = G.sgs_admm_solve(prob, G.SolverConfig(q=prob.q, max_iter=iters))
    print(f"rep {rep}: {out.iterations} iterations, loop {out.loop_ms:.3f} ms, setup {out.setup_ms:.3f} ms, "
          f"{time.perf_counter() - t:.3f} s", flush=True)
