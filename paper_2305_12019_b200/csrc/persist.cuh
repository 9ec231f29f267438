// Persistent cooperative kernel for the Gram-space SMW2 iteration.
//
// The SMW2 regime (reference subsolvers.py:94-151, chosen when d > 5000,
// 5n < d, n <= 2500) has an n x n working set -- the Gram K = Z~^T Z~ and
// G^{-1} (2 x 32 MB at n = 2000) stay in the 126 MB L2 -- so after the
// one-time DMMA Gram the iteration is latency-bound, not bandwidth-bound.
// One cooperative launch runs many iterations: each iteration is a fixed
// sequence of phases separated by grid barriers; in every phase each CTA
//   * stages the phase's input n-vector in shared memory, computing it
//     elementwise from the previous phase's results (every CTA computes the
//     whole vector, so n-sums over it are available in every CTA without a
//     cross-CTA reduction),
//   * does the GEMV rows it owns (one warp per row) and their epilogue,
//   * writes per-CTA partial sums, which after the barrier every CTA
//     reduces in the same fixed order.
// Scalars (sigma, reuse flag, beta, eps_k ...) are therefore replicated in
// each CTA's shared memory and bit-identical across CTAs; CTA 0 mirrors them
// to the global Scal record and writes the history rows.
//
// Phase map of iteration k (names from solver_ops.cuh / solver.py lines):
//   A  [K alpha_{k-1} ; GK t1]   u, rho of k-1 (needs ||g||_{k-1}, applied while
//                                staging), c_h, g; finish k-1 (obj_d, gap,
//                                stop test)                               :535-542,496-499
//   C  K c_xb                    x_bar, ztw_bar, Newton r+, dr            :501-504
//   D  [K c_res ; GK dr/mu^2]    reuse test; the re-solve g' speculatively
//                                (GK t1 kept from A, linearity)           :506-529
//   H  K [c_x ; c_g ; c_w - c_g] ztw (re-solve only), ||g||, ||w - u||;
//                                Step 3 and the KKT sample terms          :530-545,311-340
// with GK = G^{-1} K precomputed once (DMMA GEMM), so the SMW solve's
// g = G^{-1}(K t1 + y t2) = GK t1 + t2 G^{-1} y needs no separate G^{-1}
// phase (subsolvers.py:138-143, same math, different association).
// 4 grid barriers per iteration (3 with use_sgs = False).
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "solver_ops.cuh"

namespace gdwd {

namespace cg = cooperative_groups;

constexpr int PK_THREADS = 512;
constexpr int PK_WARPS = PK_THREADS / 32;
constexpr int PK_NPART = 14;  // widest cross-CTA sum (norms + KKT terms)
constexpr int PK_TS_ITERS = 64;
constexpr int PK_MAX_OWN = 32;   // samples per CTA, one per lane of warp 0 (host: n <= PK_MAX_OWN * grid)  // diagnostics: iterations timestamped (every CTA)

struct PKArgs {
  Dev D;
  const double* K;     // n x ld
  const double* Ginv;  // n x ld
  const double* GK;    // G^{-1} K, n x ld
  int64_t ld;
  double* part;        // [2][PK_NPART][gridDim] (per value, CTAs contiguous: coalesced cross-CTA reads)
  int count;           // iterations to run in this launch
  int diag;            // diagnostics: 1 = skip the GEMV rows (barrier/staging floor)
  unsigned long long* tstamp;  // diagnostics: CTA-0 %globaltimer at phase boundaries (null: off)
  int use_sgs;
};

// replicated scalar state (shared memory)
struct PKS {
  int k, stopped, converged, reuse, double_count, iters_done, error, pending;
  double sigma, sigma_next, hbot, h2bot, beta_b, beta, coef, s2, gnorm, w2, wu2, ytzw, sdual;
  double sigma_pend;  // sigma of the iteration whose u, rho update is pending
  double cp;          // persist3: t2 |y| - coef of the current SMW solve
  double eta[11];
};

// Cross-CTA reduction of per-CTA partials (slot alternates by phase), the
// same fixed order in every CTA so the totals are bitwise identical
// everywhere.  Small K: thread b loads CTA b's values, a shuffle tree per
// warp, then every thread adds the per-warp sums in warp order.  Wide K
// (the KKT bundle): warp k sums value k over the CTAs (8 loads in flight per
// lane, then a shuffle tree) -- avoids K-wide shuffle trees in 5 warps.
// (The next writer of `red` starts with a __syncthreads.)
template <int K>
GDWD_DEV void pk_cross_sum(const double* part, int slot, double (&out)[K], double* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* p = part + (size_t)slot * PK_NPART * gridDim.x;
  if constexpr (K <= 4) {
    double v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += PK_THREADS) {
#pragma unroll
      for (int k = 0; k < K; ++k) v[k] += ld_cg(p + (size_t)k * gridDim.x + b);
    }
    const int nw = min(PK_WARPS, ((int)gridDim.x + 31) / 32);
    if (warp < nw) {
      warp_sum<K>(v);
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) red[warp * K + k] = v[k];
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double t = 0.0;
      for (int w = 0; w < nw; ++w) t += red[w * K + k];
      out[k] = t;
    }
  } else {
    static_assert(K <= PK_WARPS, "one warp per value");
    if (warp < K) {
      const double* pk = p + (size_t)warp * gridDim.x;
      double v[1] = {0.0};
      for (int b0 = 0; b0 < (int)gridDim.x; b0 += 32 * 8) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int b = b0 + lane + 32 * u;
          x[u] = b < (int)gridDim.x ? ld_cg(pk + b) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) v[0] += x[u];
      }
      warp_sum<1>(v);
      if (lane == 0) red[warp] = v[0];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] = red[k];
  }
}

// This CTA's partials of K values held by lane 0 of each warp (row results):
// per-warp values through shared memory, a shuffle tree in warp 0, stored
// value-major ([slot][k][CTA]) for the coalesced cross-CTA sum.
template <int K>
GDWD_DEV void pk_write_lane0(double* part, int slot, const double (&v)[K], double* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();  // earlier readers of red are done
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) red[warp * K + k] = v[k];
  }
  __syncthreads();
  if (warp == 0) {
    double t[K];
#pragma unroll
    for (int k = 0; k < K; ++k) t[k] = lane < PK_WARPS ? red[lane * K + k] : 0.0;
    warp_sum<K>(t);
    if (lane == 0) {
      double* p = part + (size_t)slot * gridDim.x * PK_NPART + blockIdx.x;
#pragma unroll
      for (int k = 0; k < K; ++k) p[(size_t)k * gridDim.x] = t[k];
    }
  }
}

// dot of K-row i (length n, stride ld) with the staged vector(s); one warp.
// Rows are consumed in batches of U chunks of 64 doubles (one double2 per
// lane per chunk), loads predicated at the ragged end so every batch keeps
// U loads in flight per lane; the pad column of K and of the staged vectors
// is zero.  Two fused multiply-add chains per right-hand side (even / odd
// columns) halve the dependent-add chain; the shuffle tree finishes the sum.
template <int NV>
GDWD_DEV void pk_row_dot(const double* const (&rows)[NV], int64_t n, const double* const (&xs)[NV],
                         double (&out)[NV]) {
  const int lane = threadIdx.x & 31;
  double a0[NV], a1[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) a0[v] = a1[v] = 0.0;
  constexpr int U = 16 / NV;
  for (int64_t j0 = 2 * lane; j0 < n + 2 * lane; j0 += U * 64) {
    double2 z[NV][U];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j = j0 + u * 64;
        z[v][u] = j < n ? __ldg(reinterpret_cast<const double2*>(rows[v] + j)) : make_double2(0.0, 0.0);
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * 64;
      const bool ok = j < n;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const double2 xv = ok ? *reinterpret_cast<const double2*>(xs[v] + j) : make_double2(0.0, 0.0);
        a0[v] = __fma_rn(z[v][u].x, xv.x, a0[v]);
        a1[v] = __fma_rn(z[v][u].y, xv.y, a1[v]);
      }
    }
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) a0[v] += a1[v];
  warp_sum<NV>(a0);
#pragma unroll
  for (int v = 0; v < NV; ++v) out[v] = a0[v];
}

// NV right-hand sides against one K row (row loaded once)
template <int NV>
GDWD_DEV void pk_row_dot_same(const double* row, int64_t n, const double* const (&xs)[NV], double (&out)[NV]) {
  const int lane = threadIdx.x & 31;
  double a0[NV], a1[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) a0[v] = a1[v] = 0.0;
  for (int64_t j0 = 2 * lane; j0 < n + 2 * lane; j0 += 16 * 64) {
    double2 z[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int64_t j = j0 + u * 64;
      z[u] = j < n ? __ldg(reinterpret_cast<const double2*>(row + j)) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int64_t j = j0 + u * 64;
      const bool ok = j < n;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const double2 xv = ok ? *reinterpret_cast<const double2*>(xs[v] + j) : make_double2(0.0, 0.0);
        a0[v] = __fma_rn(z[u].x, xv.x, a0[v]);
        a1[v] = __fma_rn(z[u].y, xv.y, a1[v]);
      }
    }
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) a0[v] += a1[v];
  warp_sum<NV>(a0);
#pragma unroll
  for (int v = 0; v < NV; ++v) out[v] = a0[v];
}

GDWD_DEV unsigned long long pk_now() {  // SM cycle counter (exact intervals within a CTA)
  return clock64();
}

__global__ void __launch_bounds__(PK_THREADS, 1) gram_smw_persistent(PKArgs A) {
  cg::grid_group grid = cg::this_grid();
  const Dev& D = A.D;
  const int64_t n = D.n;
  extern __shared__ double pksm[];
  double* xa = pksm;           // staged vector 1 (n, padded to even)
  const int64_t ns = (n + 3) / 2 * 2;  // buffer stride: > n, even (16-byte aligned double2 reads)
  double* xb = pksm + ns;      // staged vector 2 (phase H stages a third at 2 ns)
  // bulk-copied phase inputs (6 slots) and the constant vectors y, G^{-1} y/|y|
  double* in0 = pksm + 3 * ns;
  auto IN = [&](int v) { return in0 + v * ns; };
  const double* sy = pksm + 9 * ns;
  const double* sjy = pksm + 10 * ns;
  const double* const ysm = sy;    // staged y (names free of the phases' local sums)
  const double* const jysm = sjy;  // staged G^{-1} y / |y|
  __shared__ unsigned long long bar;
  unsigned parity = 0;
  const unsigned vbytes = (unsigned)(((n + 1) / 2 * 2) * sizeof(double));
  // Phase inputs are bulk-copied by thread 0 right after the grid barrier
  // that makes them final (overlapping the cross-CTA sum and the scalar
  // section); every issue is matched by exactly one wait of all threads.
  // issued by lane 0 of the last warp, which takes no part in the cross-CTA
  // sums that follow a barrier
  auto issue = [&](int cnt, const double* const* src, double* const* dst) {
    if (threadIdx.x == PK_THREADS - 32) {
      fence_proxy_async_global();
      mbar_arrive_expect_tx(&bar, cnt * vbytes);
      for (int v = 0; v < cnt; ++v) bulk_g2s(dst[v], src[v], vbytes, &bar);
    }
  };
  auto wait_in = [&]() {
    mbar_wait(&bar, parity);
    parity ^= 1;
  };
  auto fetch = [&](int cnt, const double* const* src, double* const* dst) {
    issue(cnt, src, dst);
    wait_in();
  };
  // phase A inputs: xi, r, alpha, u, rho, x (x only read when an update is pending)
  auto issue_a = [&]() {
    const double* src[6] = {D.xi, D.r, D.al, D.u, D.rho, D.x};
    double* dst[6] = {IN(0), IN(1), IN(2), IN(3), IN(4), IN(5)};
    issue(6, src, dst);
  };
  __shared__ double red[PK_WARPS * PK_NPART];
  __shared__ PKS S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i0 = n * blockIdx.x / gridDim.x, i1 = n * (blockIdx.x + 1) / gridDim.x;
  const int nrows = A.diag == 1 ? 0 : (int)(i1 - i0);
  const double mu = D.mu, mu2 = D.mu2, yty = D.yty, ynorm = D.ynorm;
  const bool mu2_one = mu2 == 1.0;  // x / 1.0 == x exactly: skip the division
  const double ys = D.S->ys;          // SMW scalar, fixed for the solve
  __shared__ double own_u[PK_MAX_OWN], own_rho[PK_MAX_OWN], own_ztw[PK_MAX_OWN];
  int slot = 0;

  if (threadIdx.x == 0) {
    const Scal* G = D.S;
    S.k = G->k; S.stopped = G->stopped; S.converged = G->converged; S.reuse = G->reuse; S.pending = 0;
    S.gnorm = G->gnorm;
    S.double_count = G->double_count; S.iters_done = G->iters_done; S.error = G->error;
    S.sigma = G->sigma; S.sigma_next = G->sigma_next; S.sdual = G->sdual;
    for (int f = 0; f < 11; ++f) S.eta[f] = G->eta[f];
    xa[n] = 0.0;  // pad the odd tail so paired loads read zeros
    xb[n] = 0.0;
    pksm[2 * ns + n] = 0.0;
    mbar_init(&bar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  {
    const double* src[2] = {D.y, D.jy};
    double* dst[2] = {pksm + 9 * ns, pksm + 10 * ns};
    fetch(2, src, dst);
  }

  // Step 2's u, rho update of the previous iteration (solver.py:535-542)
  // needs ||g||, known only after the last barrier of that iteration: phase A
  // applies it on the fly while staging (every CTA, all j) and the owners
  // write it back in phase C, where no CTA reads u or rho.
  auto uv_commit = [&](int64_t j, double& uj, double& rj) {
    const double sp = S.sigma_pend, gn = S.gnorm;
    const double wj = D.x[j];
    const double gj = wj - D.rho[j] / (sp * mu);
    uj = (gn <= D.zscale) ? gj : (D.zscale / gn) * gj;
    rj = D.rho[j] - ((D.tau * sp) * mu) * (wj - uj);
  };

  const int k_end = S.k + A.count;
  const int k_begin = S.k;
  // per-CTA timestamps: slot (iteration, CTA, point); points: 0 top, then per phase
  // 2p+1 = arrival at its barrier, 2p+2 = scalars ready after it
#define PK_TS(pt)                                                                          \
  do {                                                                                     \
    if (A.tstamp && threadIdx.x == 0 && S.k - k_begin < PK_TS_ITERS)                       \
      A.tstamp[((size_t)(S.k - k_begin) * gridDim.x + blockIdx.x) * 32 + (pt)] = pk_now(); \
  } while (0)
  issue_a();
  for (;;) {
    if (S.stopped || S.k >= k_end) {
      wait_in();
      break;
    }
    const int k = S.k;
    const double eps = D.eps_tab[k], tol = D.tol_tab[k];  // issued early, used in C / D
    PK_TS(0);
    const bool pending = S.pending != 0;
    // ---------------- phase A: u, rho (k-1); K alpha; g = GK t1 ---------------
    {
      const double sig = S.sigma_next;
      double yr = 0.0;
      const double sp = S.sigma_pend, gn = S.gnorm;
      wait_in();
      PK_TS(24);
#pragma unroll 1
      for (int64_t j0 = threadIdx.x; j0 < n; j0 += 4 * PK_THREADS)
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // 4 independent elements in flight per thread
        const int64_t j = j0 + u * PK_THREADS;
        if (j >= n) break;
        double uj = IN(3)[j], rj = IN(4)[j];
        if (pending) {  // uv_commit
          const double wj = IN(5)[j];
          const double gj = wj - rj / (sp * mu);
          uj = (gn <= D.zscale) ? gj : (D.zscale / gn) * gj;
          rj = rj - ((D.tau * sp) * mu) * (wj - uj);
        }
        const double alj = IN(2)[j];
        const double rhs = (IN(0)[j] - IN(1)[j]) - alj / sig;
        const double chj = (-rhs + mu2 * uj) + (mu / sig) * rj;
        xa[j] = alj;
        xb[j] = mu2_one ? chj : chj / mu2;
        yr += sy[j] * rhs;
        if (j >= i0 && j < i1) {
          D.h[j] = chj;
          own_u[j - i0] = uj;  // written back in phase C (WAR: other CTAs are still copying u, rho)
          own_rho[j - i0] = rj;
        }
      }
      PK_TS(25);
      double v1[1] = {yr};
      block_sum<1>(v1, red);
      if (threadIdx.x == 0) {
        S.hbot = -v1[0];
        S.s2 = ynorm * (S.hbot / yty);
      }
      __syncthreads();
      PK_TS(26);
      const double t2 = S.hbot / yty;
      double qa = 0.0, sy = 0.0;
      for (int r = warp; r < nrows; r += PK_WARPS) {
        const int64_t i = i0 + r;
        const double* rows[2] = {A.K + i * A.ld, A.GK + i * A.ld};
        const double* xs[2] = {xa, xb};
        const double ali = xa[i];  // alpha (staged)
        double o[2];
        pk_row_dot<2>(rows, n, xs, o);
        if (lane == 0) {
          qa += ali * o[0];
          D.s1[i] = o[1];  // GK t1, reused by phase D's re-solve
          const double gi = o[1] + t2 * (ynorm * jysm[i]);
          D.g[i] = gi;
          sy += (ysm[i] / ynorm) * gi;
        }
      }
      double pv[2] = {qa, sy};
      pk_write_lane0<2>(A.part, slot, pv, red);
      PK_TS(1);
      grid.sync();
      {  // phase C inputs: g (rows of all CTAs), h
        const double* src[2] = {D.g, D.h};
        double* dst[2] = {IN(0), IN(1)};
        issue(2, src, dst);
      }
      double tot[2];
      pk_cross_sum<2>(A.part, slot, tot, red);
      slot ^= 1;
      PK_TS(2);
      if (threadIdx.x == 0) {
        S.coef = (tot[1] + (-S.s2)) / ys;
        if (blockIdx.x == 0) D.h[D.bot] = S.hbot;
        // finish iteration k-1 (solver.py:293-304,334,548-555)
        if (k > 0) {
          const double od = D.kappa * S.sdual - D.zscale * sqrt(tot[0]);
          const double op = S.eta[9];
          const double gap = fabs(op - od) / (1.0 + fabs(op) + fabs(od));
          S.eta[10] = od;
          S.eta[8] = gap;
          if (blockIdx.x == 0) {
            double* hr = D.hist + (int64_t)(k - 1) * HIST_W;
            hr[H_OBJD] = od;
            hr[H_GAP] = gap;
          }
          const double ep = fmax(fmax(S.eta[3], S.eta[4]), S.eta[5]);
          const double ed = fmax(S.eta[6], S.eta[7]);
          const double ec = fmax(fmax(S.eta[0], S.eta[1]), S.eta[2]);
          if (fmax(ep, ed) < D.tol_feas && fmin(ec, gap) < D.tol_cgap && fmax(ec, gap) < D.tol_cap) {
            S.stopped = 1;
            S.converged = 1;
          }
        }
        if (!S.stopped && k >= D.max_iter) S.stopped = 1;
        if (!S.stopped) {
          S.sigma = S.sigma_next;
          if (blockIdx.x == 0) {
            double* hr = D.hist + (int64_t)k * HIST_W;
            hr[H_SIGMA] = S.sigma;
            hr[H_EPS] = D.eps_tab[k];
            hr[H_REUSE] = 1.0;
            hr[H_PSQMR] = 0.0;
          }
        }
      }
      __syncthreads();
      if (S.stopped) {
        wait_in();
        break;
      }
    }
    const double sig = S.sigma;
    PK_TS(16);
    // ---------------- phase C: x_bar, K x_bar -> ztw_bar, Newton -------------
    {
      if (pending) {  // owners write back the u, rho update applied in phase A
        for (int64_t j = i0 + threadIdx.x; j < i1; j += PK_THREADS) {
          D.u[j] = own_u[j - i0];
          D.rho[j] = own_rho[j - i0];
        }
      }
      PK_TS(17);
      double yv = 0.0;
      const double coef = S.coef;
      wait_in();
      PK_TS(18);
#pragma unroll 1
      for (int64_t j0 = threadIdx.x; j0 < n; j0 += 4 * PK_THREADS)
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // 4 independent elements in flight per thread
        const int64_t j = j0 + u * PK_THREADS;
        if (j >= n) break;
        const double v = IN(0)[j] - coef * sjy[j];
        const double x = mu2_one ? IN(1)[j] - v : IN(1)[j] / mu2 - v / mu2;
        xa[j] = x;
        yv += sy[j] * v;
        if (j >= i0 && j < i1) D.xb[j] = x;
      }
      PK_TS(19);
      double v1[1] = {yv};
      block_sum<1>(v1, red);
      if (threadIdx.x == 0) {
        const double vn = (-S.s2) - coef * (-1.0);
        const double p2 = v1[0] + ynorm * vn;
        S.beta_b = S.hbot / yty - p2 / yty;
        if (blockIdx.x == 0) D.xb[D.bot] = S.beta_b;
        S.pending = 0;
      }
      __syncthreads();
      PK_TS(14);
      const double bb = S.beta_b;
      double ydr = 0.0;
      for (int r = warp; r < nrows; r += PK_WARPS) {
        const int64_t i = i0 + r;
        const double* rows[1] = {A.K + i * A.ld};
        const double* xs[1] = {xa};
        // per-sample operands loaded before the sweep (their latency hides under it)
        const double xii = D.xi[i], ali = D.al[i], wli = D.wl[i], ri = D.r[i], yi = ysm[i];
        double o[1];
        pk_row_dot<1>(rows, n, xs, o);
        // every lane holds the same dot (butterfly sums commute bitwise), so
        // the whole warp runs the Newton / bisection solve (warp-parallel
        // bisection levels); lane 0 stores
        const double dot = o[0];
        const double a = ((dot + yi * bb) + xii) - ali / sig;
        const double rn = A.diag == 2 ? ri + 1e-3 * a : newton_margin_warp(a, sig, D.q, wli, ri, tol);
        if (lane == 0) {
          D.ztwb[i] = dot;
          D.rnew[i] = rn;
          const double dri = rn - ri;
          D.dr[i] = dri;
          ydr += yi * dri;
        }
      }
      PK_TS(15);
      double pv[1] = {ydr};
      pk_write_lane0<1>(A.part, slot, pv, red);
      PK_TS(3);
      grid.sync();
      if (A.use_sgs) {  // phase D inputs
        const double* src[4] = {D.h, D.dr, D.ztwb, D.xb};
        double* dst[4] = {IN(0), IN(1), IN(2), IN(3)};
        issue(4, src, dst);
      } else {  // phase H inputs (Step 1c skipped: w = x_bar)
        const double* src[2] = {D.rho, D.xb};
        double* dst[2] = {IN(0), IN(1)};
        issue(2, src, dst);
      }
      double t[1];
      pk_cross_sum<1>(A.part, slot, t, red);
      slot ^= 1;
      PK_TS(4);
      if (threadIdx.x == 0) S.h2bot = S.hbot + t[0];
      __syncthreads();
    }
    // ---------------- phase D: reuse test + speculative re-solve -------------
    // Step 1c's residual q = r^T K r (r = h2 - A x_bar, solver.py:506-524) and,
    // in the same row sweep, the re-solve g' = G^{-1}K (h2/mu^2) + t2' G^{-1}y
    // = [GK t1 (kept from phase A) + GK (dr/mu^2)] + t2' G^{-1}y, used if the
    // test fails (subsolvers.py:138-143 by linearity; one barrier instead of two).
    if (A.use_sgs) {
      const double bb = S.beta_b;
      const double t2 = S.h2bot / yty;
      double ytz = 0.0;
      wait_in();
      PK_TS(20);
#pragma unroll 1
      for (int64_t j0 = threadIdx.x; j0 < n; j0 += 4 * PK_THREADS)
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // 4 independent elements in flight per thread
        const int64_t j = j0 + u * PK_THREADS;
        if (j >= n) break;
        const double h2 = IN(0)[j] + IN(1)[j];
        const double ax = (IN(2)[j] + mu2 * IN(3)[j]) + sy[j] * bb;
        xa[j] = h2 - ax;
        xb[j] = mu2_one ? IN(1)[j] : IN(1)[j] / mu2;
        ytz += sy[j] * IN(2)[j];
        if (j >= i0 && j < i1) D.h2[j] = h2;
      }
      double v1[1] = {ytz};
      block_sum<1>(v1, red);
      if (threadIdx.x == 0) S.ytzw = v1[0];
      __syncthreads();
      PK_TS(21);
      double q = 0.0, syg = 0.0;
      for (int r = warp; r < nrows; r += PK_WARPS) {
        const int64_t i = i0 + r;
        const double* rows[2] = {A.K + i * A.ld, A.GK + i * A.ld};
        const double* xs[2] = {xa, xb};
        const double s1i = D.s1[i];
        double o[2];
        pk_row_dot<2>(rows, n, xs, o);
        if (lane == 0) {
          q += xa[i] * o[0];
          const double gi = (s1i + o[1]) + t2 * (ynorm * jysm[i]);
          D.g[i] = gi;
          syg += (ysm[i] / ynorm) * gi;
        }
      }
      double pv[2] = {q, syg};
      pk_write_lane0<2>(A.part, slot, pv, red);
      PK_TS(5);
      grid.sync();
      {  // H inputs: rho, x_bar (reused) or g' (re-solved) with h, dr
        const double* src[5] = {D.rho, D.xb, D.h, D.dr, D.g};
        double* dst[5] = {IN(0), IN(1), IN(2), IN(3), IN(4)};
        issue(5, src, dst);
      }
      double t[2];
      pk_cross_sum<2>(A.part, slot, t, red);
      slot ^= 1;
      PK_TS(6);
      if (threadIdx.x == 0) {
        const double rb = S.h2bot - (S.ytzw + yty * bb);
        const double rr = hypot(sqrt(t[0] > 0.0 ? t[0] : 0.0), rb);
        S.reuse = rr <= 5.0 * eps;
        if (!S.reuse) {
          S.double_count += 1;
          S.s2 = ynorm * t2;
          S.coef = (t[1] + (-S.s2)) / ys;
        }
        if (blockIdx.x == 0) D.hist[(int64_t)k * HIST_W + H_REUSE] = S.reuse ? 1.0 : 0.0;
      }
      __syncthreads();
    } else {
      if (threadIdx.x == 0) S.reuse = 1;
      __syncthreads();
    }
    const bool reuse = S.reuse != 0;
    // ---------------- phase H: [ztw ;] ||g||, ||w-u||, ||w||; Step 3, KKT --------
    {
      // w coefficients: x_bar when reused, else x = h2/mu^2 - v/mu^2 (GsX)
      double* xw = pksm;              // staged w
      double* xg = pksm + ns;      // staged g
      double* xd = pksm + 2 * ns;  // staged w - g
      double yv = 0.0;
      const double coef = S.coef;
      wait_in();  // slots: rho, x_bar, h, dr, g' (no-sgs: rho, x_bar)
#pragma unroll 1
      for (int64_t j0 = threadIdx.x; j0 < n; j0 += 4 * PK_THREADS)
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // 4 independent elements in flight per thread
        const int64_t j = j0 + u * PK_THREADS;
        if (j >= n) break;
        double wj;
        if (reuse) {
          wj = IN(1)[j];
        } else {
          const double v = IN(4)[j] - coef * sjy[j];
          wj = mu2_one ? (IN(2)[j] + IN(3)[j]) - v : (IN(2)[j] + IN(3)[j]) / mu2 - v / mu2;
          yv += sy[j] * v;
        }
        const double gj = wj - IN(0)[j] / (sig * mu);
        xw[j] = wj;
        xg[j] = gj;
        xd[j] = wj - gj;  // w - u when u = g (no projection)
        if (j >= i0 && j < i1) D.x[j] = wj;
      }
      double v1[1] = {yv};
      block_sum<1>(v1, red);
      if (threadIdx.x == 0) {
        if (reuse) {
          S.beta = S.beta_b;
        } else {
          const double vn = (-S.s2) - coef * (-1.0);
          const double p2 = v1[0] + ynorm * vn;
          S.beta = S.h2bot / yty - p2 / yty;
        }
        if (blockIdx.x == 0) D.x[D.bot] = S.beta;
      }
      __syncthreads();
      PK_TS(11);
      double acc[PK_NPART];
#pragma unroll
      for (int f = 0; f < PK_NPART; ++f) acc[f] = 0.0;
      // Step 3 operands of the CTA's samples (warp 0, one per lane), loaded
      // before the sweep so their latency hides under it
      const int64_t is = i0 + lane;
      const bool has = warp == 0 && is < i1;
      double st_rr = 0.0, st_e = 0.0, st_al = 0.0, st_wl = 0.0;
      if (has) {
        st_rr = D.rnew[is];
        st_e = D.e[is];
        st_al = D.al[is];
        st_wl = D.wl[is];
      }
      for (int r = warp; r < nrows; r += PK_WARPS) {
        const int64_t i = i0 + r;
        const double* Ki = A.K + i * A.ld;
        double o[3];
        if (reuse) {
          const double* xs[2] = {xg, xd};
          double o2[2];
          pk_row_dot_same<2>(Ki, n, xs, o2);
          o[0] = D.ztwb[i];
          o[1] = o2[0];
          o[2] = o2[1];
        } else {
          const double* xs[3] = {xw, xg, xd};
          pk_row_dot_same<3>(Ki, n, xs, o);
        }
        if (lane == 0) {
          D.ztw[i] = o[0];
          own_ztw[r] = o[0];
          acc[10] += xg[i] * o[1];  // g^T K g
          acc[11] += xd[i] * o[2];  // d^T K d
          acc[12] += xd[i] * o[1];  // d^T K g
          acc[13] += xw[i] * o[0];  // w^T K w = ||w||^2
        }
      }
      PK_TS(12);
      __syncthreads();  // ztw of this CTA's rows is visible to its threads
      {
        // Step 3 + KKT sample terms (solver.py:533,538-541,311-333; OpStep3)
        const double bet = S.beta, C = D.C;
        if (has) {  // warp 0: the CTA's samples (at most 32, host-checked)
          const int64_t i = is;
          const double rr = st_rr;
          D.r[i] = rr;
          const double yi = ysm[i], ei = st_e, zt = own_ztw[lane], ali = st_al;
          const double xv = np_max0((((rr - zt) - yi * bet) + ali / sig) - (C / sig) * ei);
          D.xi[i] = xv;
          const double pg = ((zt + yi * bet) + xv) - rr;
          const double an = ali - (D.tau * sig) * pg;
          D.al[i] = an;
          const double wl = st_wl;
          const double s = (D.q * wl) / np_pow(rr, D.qp1);
          const double d2 = an - s;
          const double mn = np_min0(an);
          const double mx = np_max0(an - C * ei);
          acc[0] += yi * an;
          acc[1] += xv * (C * ei - an);
          acc[2] += d2 * d2;
          acc[3] += pg * pg;
          acc[4] += mn * mn;
          acc[5] += mx * mx;
          acc[6] += wl / np_pow(rr, D.q);
          acc[7] += ei * xv;
          acc[8] += np_pow(wl, D.e1) * np_pow(np_max0(an), D.e2);
          acc[9] += (rr <= 0.0) ? 1.0 : 0.0;
        }
      }
      PK_TS(13);
      // partials: KKT sample terms from warp 0 (the CTA's <= 32 samples),
      // row terms from lane 0 of every warp
      __syncthreads();
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) red[warp * 4 + q] = acc[10 + q];
      }
      __syncthreads();
      if (warp == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[10 + q] = lane < PK_WARPS ? red[lane * 4 + q] : 0.0;
        warp_sum<PK_NPART>(acc);
        if (lane == 0) {
          double* p = A.part + (size_t)slot * gridDim.x * PK_NPART + blockIdx.x;
#pragma unroll
          for (int f = 0; f < PK_NPART; ++f) p[(size_t)f * gridDim.x] = acc[f];
        }
      }
      PK_TS(9);
      grid.sync();
      issue_a();  // next iteration's phase A inputs (waited at the loop top or in A)
      double t[PK_NPART];
      pk_cross_sum<PK_NPART>(A.part, slot, t, red);
      slot ^= 1;
      PK_TS(10);
      if (threadIdx.x == 0) {
        const double gg = t[10] > 0.0 ? t[10] : 0.0;
        S.gnorm = sqrt(gg);
        if (S.gnorm <= D.zscale) {
          S.wu2 = t[11] > 0.0 ? t[11] : 0.0;
        } else {  // w - u = d + (1 - s) g with s = z_scale / ||g||
          const double om = 1.0 - D.zscale / S.gnorm;
          const double v = t[11] + 2.0 * om * t[12] + om * om * gg;
          S.wu2 = v > 0.0 ? v : 0.0;
        }
        S.w2 = t[13];
        S.pending = 1;
        S.sigma_pend = S.sigma;
        const double oc = D.one_c;
        if (t[9] > 0.0 && A.diag == 0) {
          S.error = 6;
          S.stopped = 1;
        } else {
          double* e = S.eta;
          e[0] = fabs(t[0]) / oc;
          e[1] = fabs(t[1]) / oc;
          e[2] = t[2] / oc;
          e[3] = sqrt(t[3]) / oc;
          e[4] = (D.mu * sqrt(S.wu2)) / oc;
          e[5] = fmax(sqrt(S.w2) - D.zscale, 0.0) / oc;
          e[6] = sqrt(t[4]) / oc;
          e[7] = sqrt(t[5]) / oc;
          e[9] = t[6] + D.C * t[7];
          S.sdual = t[8];
          if (blockIdx.x == 0) {
            double* hr = D.hist + (int64_t)k * HIST_W;
            for (int f = 0; f < 8; ++f) hr[f] = e[f];
            hr[H_OBJP] = e[9];
            hr[H_BETA] = S.beta;
          }
          const double ep = fmax(fmax(e[3], e[4]), e[5]);
          const double ed = fmax(e[6], e[7]);
          if (D.sched && k + 1 < D.sched_len) S.sigma_next = D.sched[k + 1];
          else S.sigma_next = sigma_rule(S.sigma, ep, ed);
          S.iters_done = k + 1;
          S.k = k + 1;
        }
      }
      __syncthreads();
    }
  }
  // a pending u, rho update is committed before the launch returns
  if (S.pending) {
    for (int64_t j = i0 + threadIdx.x; j < i1; j += PK_THREADS) {
      double uj, rj;
      uv_commit(j, uj, rj);
      D.u[j] = uj;
      D.rho[j] = rj;
    }
    __syncthreads();
    if (threadIdx.x == 0) S.pending = 0;
    __syncthreads();
  }
  // mirror the replicated scalars to the global record
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Scal* G = D.S;
    G->k = S.k; G->stopped = S.stopped; G->converged = S.converged; G->reuse = S.reuse;
    G->double_count = S.double_count; G->iters_done = S.iters_done; G->error = S.error;
    G->sigma = S.sigma; G->sigma_next = S.sigma_next; G->sdual = S.sdual; G->gnorm = S.gnorm;
    G->wu2 = S.wu2; G->w2 = S.w2;
    for (int f = 0; f < 11; ++f) G->eta[f] = S.eta[f];
  }
}

}  // namespace gdwd
