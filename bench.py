#!/usr/bin/env python
"""Benchmark: sGS-ADMM iterations/s (BASELINE.json metric).

A "step" is one ADMM iteration of the reference algorithm (solver.py:493-555)
over the whole problem.  One JSON line on rank 0 (driver contract).

N = 1 (default): BASELINE.json configs[1] ("c2": HDLSS dense fp64
d=20000 x n=2000, q=1, C=10, 10% label flips, SMW2 regime with the n x n Gram
built on the FP64 tensor cores), plus -- as the anchor of the multi-GPU curve
-- config 5 on one GPU (``strong_scaling_anchor``).

N > 1: config 5 (dense fp64 d=20000 x n=1e6, 160 GB, generated in HBM shard
by shard), sharded by samples over the N GPUs with NCCL all-reduces: the SAME
global problem at every N ("scaling": "strong"); ``value`` is iterations/s of
that global problem.  Launched by torchrun (one process per GPU, RANK /
LOCAL_RANK / WORLD_SIZE from the environment) or, without torchrun, from this
one process (one host thread per GPU, parallel.solve_on_devices' layout).
SMW2 (c2) couples all samples through its n x n Gram and is not sharded.

  value        iterations/s, device time (CUDA events on each rank's solve
               stream) of exactly --steps iterations after --warmup, max over
               ranks
  e2e          the same metric through the public API (sgs_admm_solve) from
               pinned host buffers: X upload, factorisation, iterations and
               result download inside the timed region (N = 1)
  roofline     dominant kernel of the timed region
  cpu_baseline the CPU oracle port (scipy CSC products = the reference's own
               operator) on a bounded sample, rank 0 at N = 1 only

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config c1..c5]
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "sGS-ADMM iters/s"
WORKLOADS = {
    "c1": "c1: dense fp64 d=2000 x n=1000, q=1, C=1, DIRECT",
    "c2": "c2: dense fp64 d=20000 x n=2000, q=1, C=10, 10% label flips, SMW2",
    "c3": "c3: dense fp64 d=1000 x n=200000 AR(1), q=2, C=1, DIRECT",
    "c4": "c4: sparse CSC/CSR d=50000 x n=500000 (0.1%), q=1, C=1, ITERATIVE (PSQMR)",
    "c5": "c5: dense fp64 d=20000 x n=1e6, q=4, C=5, 5% flips, ITERATIVE (PSQMR)",
}
UNIT = "iter/s"
PROBE_PEAKS = ROOT / "profiles" / "r02" / "peaks_probe.json"


def traffic_of(tag):
    """DRAM bytes per launch from a committed ncu capture (profiles/traffic.json)."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    return json.loads(p.read_text()).get(tag)


def peaks():
    """HBM peak (MEASURED_PEAKS.json, driver-written) and the probe-measured
    FP64 DMMA and L2 read peaks (profiles/r02/peaks_probe.json, committed)."""
    out = {"hbm_gbs": 6650.0, "hbm_source": "fallback (B200_PROFILING.md)"}
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        out.update(hbm_gbs=float(json.loads(p.read_text())["hbm_gbs"]), hbm_source="measured MEASURED_PEAKS.json")
    if PROBE_PEAKS.exists():
        j = json.loads(PROBE_PEAKS.read_text())
        out.update(l2_gbs=float(j["l2_read_gbs"]), fp64_tflops=float(j["fp64_dmma_tflops"]),
                   probe_source="measured profiles/r02/peaks_probe.json (profiles/probes/peaks_probe.cu)")
    return out


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# distributed plumbing (torchrun launches)
# ---------------------------------------------------------------------------
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.dist = None
        if self.world > 1:
            import torch
            import torch.distributed as dist

            backend = "nccl" if torch.cuda.is_available() else "gloo"
            if backend == "nccl":
                from paper_2305_12019_b200.parallel import pin_nccl_determinism

                pin_nccl_determinism()  # before torch's NCCL reads its parameters
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend=backend)
            self.dist, self.torch = dist, torch

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def _reduce(self, v, op):
        t = self.torch.tensor(np.atleast_1d(np.asarray(v, dtype=np.float64)),
                              device="cuda" if self.torch.cuda.is_available() else "cpu")
        self.dist.all_reduce(t, op=op)
        return t.cpu().numpy()

    def max(self, v: float) -> float:
        return v if not self.dist else float(self._reduce(v, self.dist.ReduceOp.MAX)[0])

    def sum(self, v: np.ndarray) -> np.ndarray:
        return v if not self.dist else self._reduce(v, self.dist.ReduceOp.SUM)

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


# ---------------------------------------------------------------------------
# algorithmic bytes per launch
# ---------------------------------------------------------------------------
def kernel_bytes(tag: str, n: int, d: int, nnz: int | None = None) -> float | None:
    """Algorithmic HBM bytes of one launch: the matrix once plus the vectors
    read/written.  Sparse X: 12 B per stored entry (f64 value + int32 index)
    for the CSR products, 10 B for the feature-blocked Z~^T w (16-bit
    indices).  n is the local (per-rank) sample count."""
    x = 8.0 * n * d if nnz is None else 12.0 * nnz + 8.0 * (max(n, d) + 1)
    if nnz is not None and tag.startswith("ztmv_"):
        nb = -(-d // 8192)
        return 10.0 * nnz + 4.0 * n * nb + 8.0 * (d + 6 * n)
    if nnz is not None and tag.startswith("zmv_"):
        # sample-blocked sliced ELL: 8-byte value + 16-bit index per entry,
        # t staged per block, one partial per (block, feature) written
        nb = -(-n // 12288)
        return 10.0 * nnz + 8.0 * (2 * n + nb * d + 2 * d)
    if tag.startswith("zft_"):
        return x + 8.0 * (3 * d + 10 * n)  # X once, w in, 6 sample vectors in / 4 out, 2 d-products out
    if tag.startswith("zmv_"):
        return x + 8.0 * (5 * n + 2 * d)   # up to 2 RHS in (+ inputs), 2 d-vectors out
    if tag.startswith("ztmv_"):
        return x + 8.0 * (d + 6 * n)       # w in; per-sample epilogue vectors
    if tag.startswith("sp_prep"):
        return 8.0 * 6 * n
    if tag.startswith("gemv_Ginv") or tag.startswith("gemv_K"):
        return 8.0 * n * n + 8.0 * 3 * n
    if tag.startswith("gemv_Ainv") or tag.startswith("gemv_gram"):
        return 8.0 * (d + 1) ** 2 + 16.0 * (d + 1)
    return None


def pinned_problem(G, prob, buf=None):
    """The same ProblemData with Z~'s stored values in page-locked host memory
    (the e2e contract: inputs copied from pinned host buffers).  Built outside
    the timed region; the library sees an ordinary numpy array.  ``buf``: a
    page-locked array to (re)fill instead of allocating another one."""
    import torch

    z = prob.z_tilde
    if not torch.cuda.is_available():
        return prob
    if buf is None:
        buf = torch.empty(z.values.size, dtype=torch.float64, pin_memory=True).numpy()
    buf[:] = z.values
    if z.is_dense:
        zp = G.SparseMatrixCSC.from_dense_samples(buf.reshape(z.ncols, z.nrows))
    else:
        zp = G.SparseMatrixCSC(z.nrows, z.ncols, z.colptr, z.rowidx, buf)
    pp = G.ProblemData(zp, prob.y, prob.e, prob.weights, prob.C, prob.q, prob.z_scale)
    object.__setattr__(pp, "_pinned_values", buf)  # keeps the page-locked block alive with the problem
    return pp


def solver_cfg(_lib, prob, iters, x_space=False, persistent=True):
    from paper_2305_12019_b200.solver import SolverConfig, _eps_c

    conf = SolverConfig(q=prob.q, max_iter=iters)
    return _lib.GdwdConfig(max_iter=conf.max_iter, backend=0, use_sgs=1, psqmr_switch_steps=50, ell=10, seed=0,
                           use_graph=1, poll_every=16, smw_gram_space=int(not x_space), persistent=int(persistent),
                           steplength=conf.steplength, tol_feas=conf.tol_feas, tol_cgap=conf.tol_cgap,
                           tol_cap=conf.tol_cap, sigma0=float("nan"), epsilon_c=_eps_c(prob, conf), mu=conf.mu)


def time_steps(lib, dp, ccfg, W, K):
    """Warm-up W iterations, then exactly K timed on the device (CUDA events
    on the solve stream); returns (ms, iterations timed, launches, setup_ms)."""
    from paper_2305_12019_b200 import _lib
    from paper_2305_12019_b200.solver import _check

    _check(lib.gdwd_solve_begin(dp.ctx, C.byref(ccfg), None, 0), dp.ctx, "begin")
    ms = C.c_double()
    done = C.c_int32()
    _check(lib.gdwd_time_iterations(dp.ctx, W, C.byref(ms), C.byref(done)), dp.ctx, "warmup")
    lib.gdwd_reset_counters(dp.ctx)
    _check(lib.gdwd_time_iterations(dp.ctx, K, C.byref(ms), C.byref(done)), dp.ctx, "timed")
    launches = C.c_int64()
    lib.gdwd_get_profile(dp.ctx, None, 0, C.byref(launches))
    res = _lib.GdwdResult()
    _check(lib.gdwd_solve_end(dp.ctx, C.byref(res)), dp.ctx, "end")
    return ms.value, done.value - W, int(launches.value), float(res.setup_ms)


def kernel_profile(lib, dp, ccfg, iters, n, d, nnz):
    """Per-kernel device times from an instrumented pass (events around every
    launch on the solve stream), same state sizes as the timed region."""
    from paper_2305_12019_b200 import _lib
    from paper_2305_12019_b200.solver import _check

    res = _lib.GdwdResult()
    lib.gdwd_set_profile(dp.ctx, 1)
    _check(lib.gdwd_solve_begin(dp.ctx, C.byref(ccfg), None, 0), dp.ctx, "begin")
    _check(lib.gdwd_solve_iterate(dp.ctx, 3, _lib.ITER_CB(), None, None, None), dp.ctx, "prof warm")
    lib.gdwd_reset_counters(dp.ctx)
    _check(lib.gdwd_solve_iterate(dp.ctx, iters, _lib.ITER_CB(), None, None, None), dp.ctx, "prof")
    buf = C.create_string_buffer(1 << 16)
    lib.gdwd_get_profile(dp.ctx, buf, len(buf), None)
    _check(lib.gdwd_solve_end(dp.ctx, C.byref(res)), dp.ctx, "end")
    lib.gdwd_set_profile(dp.ctx, 0)
    prof = {}
    for line in buf.value.decode().strip().splitlines():
        tag, cnt, tot = line.split()
        prof[tag] = (int(cnt), float(tot))
    total = sum(t for _, t in prof.values()) or 1.0
    kernels = []
    for tag, (cnt, tot) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        avg = tot / cnt
        b = kernel_bytes(tag, n, d, nnz)
        kernels.append({"tag": tag, "launches": cnt, "avg_us": round(avg * 1e3, 2), "share": round(tot / total, 4),
                        "gbs": round(b / (avg * 1e-3) / 1e9, 1) if b else None})
    return kernels


def hbm_roofline(kernels, n, d, nnz, pk, config):
    top = next(k for k in kernels if k["gbs"] is not None)
    tr = traffic_of(f"{config}:{top['tag']}")
    return {"bound": "hbm", "kernel": top["tag"], "achieved": top["gbs"], "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": round(top["gbs"] / pk["hbm_gbs"], 4), "peak_source": pk["hbm_source"],
            "traffic": tr["bytes"] if tr else None, "share_of_step": top["share"],
            "algorithmic_bytes_per_launch": kernel_bytes(top["tag"], n, d, nnz)}


# ---------------------------------------------------------------------------
# N = 1
# ---------------------------------------------------------------------------
def run_single(args, dist: Dist):
    import paper_2305_12019_b200 as G
    from paper_2305_12019_b200 import _lib, synth

    lib = _lib.load()
    device = dist.local
    cfg_syn = synth.CONFIGS[args.config]
    t0 = time.perf_counter()
    on_device = cfg_syn.kind != "sparse" and 8.0 * cfg_syn.n * cfg_syn.d > 40e9  # config 5: in HBM
    prob = (synth.make_device_problem(cfg_syn, args.seed, device) if on_device
            else synth.make_problem(cfg_syn, args.seed))
    gen_s = time.perf_counter() - t0
    n, d = prob.n, prob.d
    nnz = None if (prob.z_tilde is None or prob.z_tilde.is_dense) else prob.z_tilde.nnz
    K, W = args.steps, args.warmup
    pk = peaks()

    # ---- device-resident timing ----------------------------------------------
    dp = G.device_problem(prob, device)
    ccfg = solver_cfg(_lib, prob, W + K + 1, args.x_space, not args.no_persistent)
    dist.barrier()
    with Clocks(device) as clk:
        ms, iters_timed, launches, setup_ms = time_steps(lib, dp, ccfg, W, K)
    t_ms = dist.max(ms)
    if iters_timed <= 0:
        raise RuntimeError("the solve stopped before the timed region")
    step_ms = t_ms / iters_timed
    value = dist.world * iters_timed / (t_ms / 1e3)

    kernels = kernel_profile(lib, dp, ccfg, min(max(8, K // 4), 64), n, d, nnz)
    kind_name = G.select_solver(n, d).value
    persistent = bool(ccfg.persistent) and not args.x_space and nnz is None and n <= 2500 and (
        (kind_name == "smw2" and n <= d) or (kind_name == "direct" and 2 * n <= d))
    if persistent:
        roofline = persistent_roofline(n, iters_timed, t_ms, pk, args.config)
    else:
        roofline = hbm_roofline(kernels, n, d, nnz, pk, args.config)
    roofline_x = xspace_roofline(G, lib, dp, ccfg, n, d, nnz, pk) if (args.config == "c2" and not args.x_space) else None
    gram = gram_roofline(lib, dp, n, d, pk) if (persistent or kind_name == "direct") and nnz is None else None

    # ---- end to end through the public API ------------------------------------
    e2e = None
    if on_device:
        e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "note": "X generated in HBM (160 GB exceeds host memory); no host-buffer path"}
    elif not args.no_e2e:
        e2e = measure_e2e(G, synth, cfg_syn, args, device, dist, K, n, d, nnz)

    # ---- time to KKT 1e-5 (feasibility), factorisation included --------------------
    ttk = None
    if args.kkt_iters < 0:
        args.kkt_iters = 2000 if args.config in ("c1", "c2") else 100
    if args.kkt_iters > 0 and not on_device:
        ttk = time_to_kkt(G, prob, args, device)

    nxt = None
    if not args.no_next and not on_device and dist.rank == 0:
        nxt = measure_next_rows(G, prob, device, args)
    dp.close()

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": dist.world, "steps": iters_timed,
        "warmup": W, "ms_per_step": round(step_ms, 5), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded generator with BASELINE %s shapes (paper_2305_12019_b200.synth%s)"
                % (args.config, ", generated on the device" if on_device else ""),
        "config": {"workload": WORKLOADS.get(args.config, args.config),
                   "path": ("Gram-space iteration in one persistent cooperative kernel (n x n Gram on FP64 DMMA, "
                            "explicit G^-1)" if persistent else "CUDA-graph / host-driven kernel sequence"),
                   "d": d, "n": n, "parallelism": "replicas" if dist.world > 1 else "single",
                   "l2": ("inputs larger than L2 (X = %.0f MB > 126 MB); the Gram-space loop never reads X -- its "
                          "working set (K, G^-1 K: %.0f MB) is L2-resident by design, no flush inside the single "
                          "persistent launch" % (8 * n * d / 1e6, 16 * n * n / 1e6)) if persistent else
                         "inputs larger than L2 (X = %.0f MB > 126 MB)" % (8 * n * d / 1e6 if nnz is None else
                                                                             12 * nnz / 1e6),
                   "setup_ms": round(setup_ms, 3), "gen_s": round(gen_s, 2)},
        "roofline": roofline, "roofline_x_stream": roofline_x, "gram": gram, "kernels": kernels[:12],
        "gpu_launches": launches,
        "clocks": clk.summary(), "e2e": e2e, "time_to_kkt": ttk, "next_rows": nxt,
    }
    return line


def persistent_roofline(n, iters, t_ms, pk, config):
    """The Gram-space persistent kernel: K and G^-1 K (n x n each) are swept
    twice per iteration from tensor memory / L2; DRAM sees only the one cold
    load.  Bound: on-chip (L2) latency, reported against the measured L2 read
    rate -- not HBM."""
    alg = 8.0 * n * n * 4.0 * iters
    ach = alg / (t_ms * 1e-3) / 1e9
    tr = traffic_of("c2:gram_smw_persistent3") if config == "c2" else None
    l2 = pk.get("l2_gbs")
    r = {"bound": "l2", "kernel": "gram_smw_persistent3", "achieved": round(ach, 1),
         "peak": l2, "unit": "GB/s", "frac": round(ach / l2, 4) if l2 else None,
         "peak_source": pk.get("probe_source", "unmeasured"),
         "traffic": round(tr["per_iteration"] * iters) if tr else None,
         "algorithmic_bytes_per_launch": alg, "share_of_step": 1.0,
         "hbm_frac_of_dram_traffic": round(tr["per_iteration"] * iters / (t_ms * 1e-3) / 1e9 / pk["hbm_gbs"], 5)
         if tr else None,
         "note": "one cooperative launch runs every timed iteration; per iteration it sweeps K and G^-1 K twice "
                 "(algorithmic on-chip bytes, own rows from tensor memory, the rest from L2) behind 3 grid barriers. "
                 "DRAM traffic (ncu) is only the first-touch load, so HBM is not the bound; the kernel is bound by "
                 "barrier and L2/TMEM row latency (profiles/r02/README.md: phase timing)"}
    return r


def xspace_roofline(G, lib, dp, ccfg, n, d, nnz, pk):
    """The X-space SMW2 kernels (passes over the 320 MB X) on the same data:
    the streaming matvecs' HBM roofline."""
    from paper_2305_12019_b200 import _lib

    ccfg_x = _lib.GdwdConfig.from_buffer_copy(ccfg)
    ccfg_x.smw_gram_space = 0
    ks = kernel_profile(lib, dp, ccfg_x, 16, n, d, nnz)
    xs = [k for k in ks if k["tag"].startswith(("zmv_", "ztmv_")) and k["gbs"]]
    if not xs:
        return None
    best = max(xs, key=lambda k: k["gbs"])
    tr = traffic_of("c2:" + best["tag"])
    return {"bound": "hbm", "best_kernel": best["tag"], "achieved": best["gbs"], "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": round(best["gbs"] / pk["hbm_gbs"], 4), "traffic": tr["bytes"] if tr else None,
            "kernels": {k["tag"]: k["gbs"] for k in xs},
            "algorithmic_bytes_per_launch": kernel_bytes(best["tag"], n, d, nnz),
            "note": "X-space SMW2 (smw_gram_space=0): each kernel streams X = %.0f MB" % (8 * n * d / 1e6)}


def gram_roofline(lib, dp, n, d, pk):
    """The one-time FP64 tensor-core Gram (DMMA SYRK) of the resident X:
    2 * min(n,d)^2 * max(n,d) / 2 flops (one triangle), device time."""
    from paper_2305_12019_b200 import _lib
    from paper_2305_12019_b200.solver import _check

    ms = C.c_double()
    rc = lib.gdwd_time_gram(dp.ctx, 3, C.byref(ms))
    if rc != _lib.OK:
        return None
    m, k = min(n, d), max(n, d)
    flop = 1.0 * m * m * k  # SYRK: the lower triangle incl. diagonal blocks ~ m^2 k
    tf = flop / (ms.value * 1e-3) / 1e12
    peak = pk.get("fp64_tflops")
    return {"bound": "tensor", "kernel": "gemm_dmma (SYRK, DMMA.8x8x4)", "achieved": round(tf, 2), "peak": peak,
            "unit": "TFLOP/s", "frac": round(tf / peak, 4) if peak else None, "ms": round(ms.value, 3),
            "flop": flop, "peak_source": pk.get("probe_source", "unmeasured")}


def measure_e2e(G, synth, cfg_syn, args, device, dist, K, n, d, nnz):
    # one untimed end-to-end call first (a warm process: allocator pool,
    # module loading), on its own copy that is then released
    prob_w = pinned_problem(G, synth.make_problem(cfg_syn, args.seed))
    G.sgs_admm_solve(prob_w, G.SolverConfig(q=prob_w.q, max_iter=min(K, 20)), device=device)
    G.solver.device_problem(prob_w, device).close()
    buf = prob_w._pinned_values  # one page-locked input buffer, refilled with fresh data before every call
    del prob_w
    # three timed calls, each on freshly generated host data with a new device
    # context (nothing resident, no cached factor); the median call is reported
    runs = []
    reps = 3 if 8.0 * n * d < 4e9 else 1
    for _ in range(reps):
        prob2 = pinned_problem(G, synth.make_problem(cfg_syn, args.seed), buf)
        dist.barrier()
        t1 = time.perf_counter()
        out = G.sgs_admm_solve(prob2, G.SolverConfig(q=prob2.q, max_iter=K), device=device)
        runs.append((dist.max(time.perf_counter() - t1), out))
        G.solver.device_problem(prob2, device).close()
        del prob2
    e2e_s, out = sorted(runs, key=lambda r: r[0])[len(runs) // 2]
    h2d = (8.0 * n * d if nnz is None else 16.0 * nnz + 8.0 * (n + 1)) + 8.0 * 3 * n
    d2h = 8.0 * (4 * n + 3 * d + 1 + 16 * out.iterations)
    return {"value": round(dist.world * out.iterations / e2e_s, 3), "unit": UNIT,
            "h2d_bytes_per_step": round(h2d / out.iterations), "d2h_bytes_per_step": round(d2h / out.iterations),
            "seconds": round(e2e_s, 4), "iterations": out.iterations,
            "runs_s": [round(r[0], 4) for r in runs],
            "breakdown": {k: round(v, 5) for k, v in (out.timings or {}).items()},
            "note": "sgs_admm_solve from host numpy buffers (X in pinned host memory): X upload, factorisation, "
                    "iterations, state download; median of %d calls, each on fresh host data and a new context. "
                    "Sample-space regimes: the Gram, its Cholesky factor and inverse advance block by block "
                    "during the copy (DESIGN.md section 6)" % len(runs)}


def time_to_kkt(G, prob, args, device):
    """One solve on a FRESH device copy (no cached factorisation): setup (Gram
    + factor) + iterations until max(eta_P, eta_D) < 1e-5, device time; and
    the same through the public API from host buffers (upload included)."""
    # warm process first (memory-pool growth for the Gram's split-K workspace is a
    # one-time driver cost): a short solve on its own fresh copy, then released
    warm = G.ProblemData(prob.z_tilde, prob.y, prob.e, prob.weights, prob.C, prob.q, prob.z_scale)
    G.sgs_admm_solve(warm, G.SolverConfig(q=prob.q, max_iter=3), device=device)
    G.solver.device_problem(warm, device).close()
    fresh = G.ProblemData(prob.z_tilde, prob.y, prob.e, prob.weights, prob.C, prob.q, prob.z_scale)
    t0 = time.perf_counter()
    out = G.sgs_admm_solve(fresh, G.SolverConfig(q=prob.q, max_iter=args.kkt_iters), device=device)
    wall = time.perf_counter() - t0
    G.solver.device_problem(fresh, device).close()
    h = out.history
    feas = np.maximum(h[:, 3:6].max(axis=1), h[:, 6:8].max(axis=1))
    hit = np.flatnonzero(feas < 1e-5)
    per_it = out.loop_ms / max(out.iterations, 1)
    up = (out.timings or {}).get("upload_s", 0.0)
    return {"first_feas_1e-5_iter": int(hit[0] + 1) if hit.size else None,
            "first_feas_1e-5_s": round((out.setup_ms + per_it * (hit[0] + 1)) / 1e3, 5) if hit.size else None,
            "first_feas_1e-5_s_with_upload": round(up + (out.setup_ms + per_it * (hit[0] + 1)) / 1e3, 5)
            if hit.size else None,
            "stop_rule_fired": bool(out.converged), "iterations_run": out.iterations,
            "solve_s_device": round((out.setup_ms + out.loop_ms) / 1e3, 4), "solve_s_wall_api": round(wall, 4),
            "setup_ms": round(out.setup_ms, 3), "upload_s": round(up, 5),
            "note": "fresh device copy from pageable host arrays (no cached factor): in the sample-space regimes the "
                    "Gram (FP64 DMMA) and the Cholesky inverse run during the staged upload, so upload_s holds them "
                    "and setup_ms only what is left; elsewhere setup_ms = Gram + factorisation.  first_feas = setup + "
                    "per-iteration loop time x iterations until max(eta_P, eta_D) < 1e-5 (+ upload_s in the "
                    "_with_upload figure)"}


def measure_next_rows(G, prob, device, args):
    """decision_values / train_error (solver.py:610-642) and the penalty-C
    distance statistic (solver.py:193-232) on the workload's matrix: device
    time per call (host buffers in and out) and the oracle's on the host."""
    from oracle import gdwd_oracle as O
    from paper_2305_12019_b200 import ModelFile, identity_meta, scoring

    x, y = prob.z_tilde, prob.y
    w = np.random.default_rng(3).standard_normal(x.nrows) / np.sqrt(x.nrows)
    model = ModelFile(q=prob.q, C=prob.C, z_scale=1.0, mu=1.0, feature_meta=identity_meta(x.nrows), w=w, beta=0.1)
    dm = scoring.device_matrix(x, device)  # upload once (resident, like a served model's inputs)
    scoring.train_error(model, x, y, device)
    reps = 20
    t = time.perf_counter()
    for _ in range(reps):
        scoring.decision_values(model, x, device)
    dev_s = (time.perf_counter() - t) / reps
    t = time.perf_counter()
    for _ in range(reps):
        scoring.train_error(model, x, y, device)
    dev_err_s = (time.perf_counter() - t) / reps
    xs = x.scipy
    t = time.perf_counter()
    O.decision_values(w, 0.1, xs)
    cpu_s = time.perf_counter() - t
    out = {"scoring": {"samples": x.ncols, "device_s_per_call": round(dev_s, 6),
                       "device_samples_per_s": round(x.ncols / dev_s, 1),
                       "train_error_s_per_call": round(dev_err_s, 6),
                       "oracle_s_per_call": round(cpu_s, 6),
                       "note": "matrix resident in HBM; w in and scores out through host buffers"}}
    if x.ncols <= 20000:
        G.compute_penalty_C(x, y, prob.q)
        t = time.perf_counter()
        c, dist_ = G.compute_penalty_C(x, y, prob.q)
        pen_s = time.perf_counter() - t
        pairs = int(min((y > 0).sum(), 2000) * min((y < 0).sum(), 2000))
        pen = {"C": c, "dist": dist_, "device_s": round(pen_s, 5), "pairs": pairs, "oracle_s": None}
        if pairs * x.nrows <= 2e9:  # the oracle's sparse between-class product is slow: bounded
            t = time.perf_counter()
            O.penalty_C(xs, y, prob.q)
            pen["oracle_s"] = round(time.perf_counter() - t, 4)
        out["penalty_C"] = pen
    dm.close()
    return out


# ---------------------------------------------------------------------------
# N > 1: one global problem sharded by samples (strong scaling)
# ---------------------------------------------------------------------------
def _rank_problem(G, synth, parallel, cfg_syn, seed, device, rank, world, allreduce, comm):
    """This rank's shard: two-Gaussian configs are generated in HBM (shard-
    consistent counter-based stream); the others on the host, then uploaded."""
    if cfg_syn.kind == "gauss":
        return synth.make_device_problem(cfg_syn, seed, device, rank, world, allreduce=allreduce, comm=comm)
    prob = synth.make_problem(cfg_syn, seed)
    local = parallel.shard_problem(prob, rank, world)
    if comm is not None:
        parallel.attach(local, comm, prob.n, device)
    else:
        G.device_problem(local, device)
    return local


def run_sharded(args, dist: Dist, world: int):
    """Every rank times its K iterations on its own stream; value = K / max
    over ranks of that time (the global problem's iterations/s)."""
    import paper_2305_12019_b200 as G
    from paper_2305_12019_b200 import _lib, parallel, synth
    from paper_2305_12019_b200.solver import _check

    lib = _lib.load()
    cfg_syn = synth.CONFIGS[args.config]
    K, W = args.steps, args.warmup
    pk = peaks()
    if dist.world > 1:  # torchrun: this process is one rank
        ranks = [dist.rank]
        devices = {dist.rank: dist.local}
        comm_mode = "nccl"
    else:  # one process, one host thread per GPU
        ranks = list(range(world))
        devs = [int(x) for x in args.devices.split(",")] if args.devices else list(range(world))
        if len(devs) != world:
            raise SystemExit("--devices must list --gpus ids")
        devices = dict(enumerate(devs))
        comm_mode = args.comm
    threads_ar = parallel.ThreadRanks(world)
    uid = None
    if comm_mode == "nccl" and dist.world == 1 and world > 1:
        buf = (C.c_uint8 * 128)()
        _check(lib.gdwd_comm_unique_id(buf), None, "nccl unique id")
        uid = bytes(buf)
    res = {}
    errs = []
    t_gen = time.perf_counter()

    def one_rank(r):
        try:
            if dist.world > 1:
                comm = parallel.NcclCommunicator.from_torch()
                ar = dist.sum
            elif world == 1:  # the unsharded single-GPU path (strong-scaling anchor)
                comm, ar = None, None
            else:
                ar = threads_ar.allreduce_for(r)
                comm = (parallel.NcclCommunicator(world, r, lambda _i: uid) if comm_mode == "nccl"
                        else parallel.HostCommunicator(ar, world, r))
            prob = _rank_problem(G, synth, parallel, cfg_syn, args.seed, devices[r], r, world, ar, comm)
            dp = G.device_problem(prob, devices[r])
            ccfg = solver_cfg(_lib, prob, W + K + 1)
            gen = time.perf_counter() - t_gen
            if dist.world > 1:
                dist.barrier()
            ms, it, launches, setup_ms = time_steps(lib, dp, ccfg, W, K)
            # every rank takes part (the instrumented pass all-reduces too); rank 0's is reported
            kern = kernel_profile(lib, dp, ccfg, min(max(4, K // 4), 16), prob.n, prob.d,
                                  None if (prob.z_tilde is None or prob.z_tilde.is_dense) else prob.z_tilde.nnz)
            res[r] = dict(ms=ms, iters=it, launches=launches, setup_ms=setup_ms, n=prob.n, d=prob.d, kernels=kern,
                          gen_s=gen, nnz=None if (prob.z_tilde is None or prob.z_tilde.is_dense) else prob.z_tilde.nnz)
            dp.close()
        except BaseException as exc:
            errs.append(exc)
            threads_ar.barrier.abort()

    dev0 = devices[ranks[0]]
    with Clocks(dev0) as clk:
        if len(ranks) == 1:
            one_rank(ranks[0])
        else:
            th = [threading.Thread(target=one_rank, args=(r,)) for r in ranks]
            for t in th:
                t.start()
            for t in th:
                t.join()
    if errs:
        raise errs[0]
    t_ms = dist.max(max(v["ms"] for v in res.values()))
    iters = res[ranks[0]]["iters"]
    r0 = res.get(0)
    line = {
        "metric": METRIC, "value": round(iters / (t_ms / 1e3), 4), "unit": UNIT, "n_gpus": world, "steps": iters,
        "warmup": W, "ms_per_step": round(t_ms / iters, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded generator with BASELINE %s shapes%s" % (
            args.config, ", each rank generating its shard in HBM" if cfg_syn.kind == "gauss" else ""),
        "config": {"workload": WORKLOADS.get(args.config, args.config), "d": cfg_syn.d, "n": cfg_syn.n,
                   "parallelism": f"dp{world}: samples sharded over {world} GPUs, NCCL all-reduce of the Z~ t "
                                  f"d-partials and n-sums ({'torchrun, one process per GPU' if dist.world > 1 else 'one process, one host thread per GPU'}; comm={comm_mode})",
                   "l2": "inputs larger than L2 (X shard = %.1f GB per GPU)" % (8.0 * cfg_syn.d * cfg_syn.n / world / 1e9),
                   "setup_ms_rank0": round(r0["setup_ms"], 2) if r0 else None,
                   "gen_s": round(r0["gen_s"], 2) if r0 else None},
        "gpu_launches": r0["launches"] if r0 else None,
        "clocks": clk.summary(),
        "e2e": {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "note": "X generated in HBM shard by shard (160 GB exceeds host memory); no host-buffer path"},
    }
    if r0 and r0["kernels"]:
        line["kernels"] = r0["kernels"][:12]
        line["roofline"] = hbm_roofline(r0["kernels"], r0["n"], r0["d"], r0["nnz"], pk, args.config)
    return line


def strong_scaling_anchor(args, dist):
    """Config 5 on ONE GPU (the N = 1 point of the N > 1 strong-scaling runs,
    which shard this same global problem)."""
    import copy

    a = copy.copy(args)
    a.config = "c5"
    a.steps, a.warmup = max(4, min(args.steps, 10)), 3
    line = run_sharded(a, dist, 1)
    return {k: line[k] for k in ("value", "unit", "steps", "warmup", "ms_per_step", "roofline", "kernels")
            if k in line} | {"workload": WORKLOADS["c5"], "n_gpus": 1}


# ---------------------------------------------------------------------------
# CPU legs
# ---------------------------------------------------------------------------
C5_CPU_SAMPLES = 20000


def run_cpu_oracle(args, K: int, W: int):
    """The oracle port on the host cores, bounded sample.  Config 5 (160 GB
    dense; ~320 GB as the reference's int64 CSC) does not fit host memory: the
    port runs on its first 20000 samples (same generator, d, q, C) and the
    per-iteration time is scaled by n / 20000 (every X pass is linear in n)."""
    from oracle import gdwd_oracle as O
    from paper_2305_12019_b200 import synth

    cfg = synth.CONFIGS[args.config]
    scale = 1.0
    if args.config == "c5":
        scale = cfg.n / C5_CPU_SAMPLES
        cfg = cfg.scaled(n=C5_CPU_SAMPLES)
    prob = synth.make_problem(cfg, args.seed)
    t0 = time.perf_counter()
    res = O.solve(prob, O.OracleConfig(max_iter=W + K), operator="csc", gram="dense", record=False,
                  time_after=W)
    per_it = res.timed_s / max(res.timed_iters, 1) * scale
    sample = (f"{res.timed_iters} iterations of config {args.config[1:]} after {W} warm-up iterations "
              f"(oracle port: scipy CSC products = the reference's own operator; the one-time factor built "
              f"with dense BLAS in {res.setup_s:.1f}s instead of the reference's sparse Gram)")
    if scale != 1.0:
        sample += f"; on the first {C5_CPU_SAMPLES} samples, time per iteration x {scale:g} (linear in n)"
    return {"value": round(1.0 / per_it, 5), "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": sample, "setup_s": round(res.setup_s, 2), "total_s": round(time.perf_counter() - t0, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="auto", help="c1..c5; auto = c2 at N = 1, c5 (sharded) at N > 1")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-next", action="store_true", help="skip the scoring / penalty-C measurements")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-anchor", action="store_true", help="skip config 5 on one GPU at N = 1")
    ap.add_argument("--kkt-iters", type=int, default=-1,
                    help="iterations of the time-to-KKT solve (default: the reference's max_iter, 2000, for the "
                         "Gram-space configs c1/c2; 100 elsewhere)")
    ap.add_argument("--cpu-steps", type=int, default=24,
                    help="iterations of the CPU oracle leg (c2: ~0.5 s each on 16 cores, i.e. ~12 s)")
    ap.add_argument("--x-space", action="store_true", help="SMW2 iterations as passes over X (no Gram-space)")
    ap.add_argument("--no-persistent", action="store_true", help="Gram-space SMW2 as a CUDA graph of kernels")
    ap.add_argument("--devices", default=None, help="single-process N > 1: device ids (default 0..N-1)")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "host"],
                    help="single-process N > 1: NCCL, or the host exchange (several ranks may share a GPU)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    dist = Dist()
    world = dist.world if dist.world > 1 else max(1, args.gpus)
    if args.config == "auto":
        args.config = "c2" if world == 1 else "c5"
    if args.impl == "reference":
        # the reference's own CPU path (oracle port) on the host cores, same
        # config / steps / warm-up as the B200 arm; rank 0 only
        if dist.rank == 0:
            K, W = args.steps, args.warmup
            cb = run_cpu_oracle(args, K, W)
            line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world, "steps": K,
                    "warmup": W, "ms_per_step": round(1e3 / cb["value"], 3), "higher_is_better": True,
                    "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "f64",
                    "impl": "reference",
                    "data": "synthetic: seeded generator with BASELINE %s shapes" % args.config,
                    "config": {"workload": WORKLOADS.get(args.config, args.config), "parallelism": "host"},
                    "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                    "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
            print(json.dumps(line), flush=True)
        dist.close()
        return
    if world == 1:
        line = run_single(args, dist)
        if not args.no_cpu and args.config != "c5":
            line["cpu_baseline"] = run_cpu_oracle(args, args.cpu_steps, 1)
        if not args.no_anchor and args.config != "c5":
            line["strong_scaling_anchor"] = strong_scaling_anchor(args, dist)
    else:
        line = run_sharded(args, dist, world)
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
