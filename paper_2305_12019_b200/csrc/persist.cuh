// Shared machinery of the persistent cooperative Gram-space kernel
// (persist3.cuh): launch geometry, the replicated scalar record, the
// fixed-order cross-CTA sums and the warp row dots over n x n matrices.
//
// The Gram-space iteration (reference subsolvers.py:94-151 SMW2, and DIRECT
// with 2n <= d) has an n x n working set -- the Gram K = Z~^T Z~ and
// G^{-1} K (2 x 32 MB at n = 2000) stay on chip -- so after the one-time DMMA
// Gram the loop is latency-bound.  In every phase each CTA stages the phase's
// input n-vector in shared memory (every CTA computes the whole vector, so
// n-sums over it need no cross-CTA reduction), does the rows it owns (one
// warp per row) and their epilogue, and writes per-CTA partials that every
// CTA reduces in the same fixed order after the grid barrier: scalars are
// replicated bitwise and every CTA takes the same decisions.
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

}  // namespace gdwd
