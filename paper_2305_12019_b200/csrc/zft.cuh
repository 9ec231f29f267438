// Fused "dot -> per-sample epilogue -> axpy" pass over the sample-major X
// (one HBM read where the unfused loop makes two):
//
//   for every sample i:   dot_i = x_i . w            (optional, device flag)
//                         t_i   = Op::input(i, dot_i) (per-sample update)
//   v = sum_i x_i t_i     (R right-hand sides, then a per-feature epilogue)
//
// Used for the tail of an X-space ADMM iteration (solver.py:530-541 plus the
// next iteration's Z~ [xi - r, alpha], SURVEY App. C fusion P2): Z~^T w after
// a re-solve, Step 3 and the KKT sample sums, then the two products the next
// right-hand side and the dual objective need.
//
// Layout.  A cluster of `cs` CTAs (one per SM) owns a contiguous range of
// samples; CTA rank q of the cluster owns the feature slice [q dw, (q+1) dw).
// Rows of the slice are staged in shared memory by bulk copies (TMA engine,
// mbarrier completion), `tr` rows per stage, `ns` stages in flight.  Column
// warps (15) hold their slice's w entries and the R accumulators of their
// columns in registers: a thread owns columns tid, tid + 480, ...  A 16th
// "sample warp" prefetches the per-sample inputs one tile ahead, combines the
// row dots of the cluster's CTAs (partials exchanged through distributed
// shared memory, one cluster barrier per tile) and runs the epilogue.  Sums
// that need powers (the KKT terms) are left to a separate map over the
// per-sample outputs: a pow on the sample warp would sit on every tile's
// critical path.
//
// Determinism: each row dot is a fixed shuffle tree per warp, a fixed-order
// sum over warps and then over the cluster's ranks; the axpy accumulates in
// row order; per-cluster partials are summed in cluster order by
// zft_reduce_kernel.  Every CTA of a cluster computes the same epilogue from
// the same inputs; only rank 0 writes per-sample outputs and sums (the
// inputs are read before the tile's cluster barrier, the outputs written
// after it, so an overwritten input is never read).
#pragma once
#include "zops.cuh"

namespace gdwd {

constexpr int FT_CW = 480;              // column threads (15 warps)
constexpr int FT_THREADS = FT_CW + 32;  // + the sample warp: 16 warps, 4 per SM sub-partition (128 registers)
constexpr int FT_TRMAX = 8;             // rows per stage
// rows per stage the column loops unroll for: wide slices (many columns per
// thread) stage few rows, and fewer row registers keep the accumulators resident
__host__ __device__ constexpr int ft_trm(int cpt) { return cpt >= 12 ? 2 : (cpt >= 8 ? 4 : FT_TRMAX); }
constexpr int FT_CSMAX = 8;             // CTAs per cluster
constexpr int FT_RED = 16;              // per-warp slots per row / per sum

struct FtGeom {
  int cs;        // CTAs per cluster (feature slices)
  int clusters;  // co-resident clusters (exactly one wave)
  int dw;        // slice width (even)
  int tr;        // rows per stage
  int ns;        // stages
  int64_t ldp;   // stride of the per-cluster partial rows (>= d, even)
};

GDWD_DEV unsigned ft_cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
GDWD_DEV unsigned ft_cluster_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
GDWD_DEV void ft_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// store v at the same shared-memory offset in cluster CTA `rank`
GDWD_DEV void ft_st_cluster(double* local, unsigned rank, double v) {
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}
GDWD_DEV void ft_cw_sync() { asm volatile("bar.sync 1, %0;" ::"n"(FT_CW) : "memory"); }

inline size_t ft_smem_bytes(const FtGeom& g, int R) {
  return ((size_t)(g.ns * g.tr + 1) * g.dw + (size_t)FT_TRMAX * R + 2 * FT_CSMAX * FT_TRMAX + FT_RED * FT_TRMAX) *
             sizeof(double) +
         8 * sizeof(unsigned long long);
}

template <class Op, int CPT>
__global__ void __launch_bounds__(FT_THREADS, 1) zft_kernel(Op op, MatView X, FtGeom g, Scratch s) {
  constexpr int R = Op::R, NN = Op::NN;
  if (op.skip()) return;  // grid-uniform (a flag no CTA of this kernel writes)
  extern __shared__ __align__(16) double fsm[];
  const int dw = g.dw;
  double* stage = fsm;                                          // [ns][tr][dw]
  double* ws = stage + (size_t)g.ns * g.tr * dw;                // [dw] this slice of w
  double* ts = ws + dw;                                         // [FT_TRMAX][R]
  double* xch = ts + FT_TRMAX * R;                              // [2][FT_CSMAX][FT_TRMAX]
  double* red = xch + 2 * FT_CSMAX * FT_TRMAX;                  // [FT_RED][FT_TRMAX]
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(red + FT_RED * FT_TRMAX);
  const int cs = g.cs;
  const unsigned q = cs > 1 ? ft_cluster_rank() : 0u;
  const int cl = cs > 1 ? (int)ft_cluster_id() : (int)blockIdx.x;
  const int64_t c0 = (int64_t)q * dw;
  const int64_t len = c0 < X.cols ? (X.cols - c0 < dw ? X.cols - c0 : dw) : 0;
  const unsigned rowbytes = (unsigned)(((len + 1) & ~(int64_t)1) * sizeof(double));  // even: inside ld's padding
  const int64_t i0 = X.rows * cl / g.clusters, i1 = X.rows * (cl + 1) / g.clusters;
  const int64_t T = (i1 - i0 + g.tr - 1) / g.tr;
  const bool dot = op.need_dot();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool sw = warp == FT_CW / 32;  // the sample warp
  const bool writer = q == 0;

  if (tid == 0) {
    for (int k = 0; k < g.ns; ++k) mbar_init(&bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  // producer (thread 0): stage tile t into slot t % ns
  auto issue = [&](int64_t t) {
    const int k = (int)(t % g.ns);
    const int64_t r0 = i0 + t * g.tr;
    const int nr = (int)(i1 - r0 < g.tr ? i1 - r0 : g.tr);
    double* dst = stage + (size_t)k * g.tr * dw;
    mbar_arrive_expect_tx(&bar[k], (unsigned)nr * rowbytes);
    if (rowbytes)
      for (int r = 0; r < nr; ++r) bulk_g2s(dst + (size_t)r * dw, X.a + (r0 + r) * X.ld + c0, rowbytes, &bar[k]);
  };
  if (tid == 0)
    for (int64_t t = 0; t < T && t < g.ns; ++t) issue(t);

  double acc[R][CPT];
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    const int64_t col = tid + (int64_t)FT_CW * j;
    if (!sw && col < dw) ws[col] = (dot && col < len) ? op.wval(c0 + col) : 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r][j] = 0.0;
  }
  // (each thread reads back only the w entries it stored)
  double na[NN];
#pragma unroll
  for (int k = 0; k < NN; ++k) na[k] = 0.0;
  // launch-uniform scalars once (sigma, beta, ...), and the first tile's
  // per-sample inputs; later tiles' inputs are prefetched one tile ahead
  const typename Op::U u = op.uniform();
  typename Op::Pf pf, pfn;
  if (sw && T > 0 && lane < (i1 - i0 < g.tr ? i1 - i0 : g.tr)) op.prefetch(i0 + lane, pf);

  for (int64_t t = 0; t < T; ++t) {
    const int k = (int)(t % g.ns);
    const unsigned par = (unsigned)((t / g.ns) & 1);
    const int64_t r0 = i0 + t * g.tr;
    const int nr = (int)(i1 - r0 < g.tr ? i1 - r0 : g.tr);
    const double* st = stage + (size_t)k * g.tr * dw;
    double* xb = xch + (t & 1) * (FT_CSMAX * FT_TRMAX);
    if (!sw) {
      mbar_wait(&bar[k], par);
      if (dot) {
        constexpr int TRM = ft_trm(CPT);
        double p[TRM];
#pragma unroll
        for (int r = 0; r < TRM; ++r) p[r] = 0.0;
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
          const int col = tid + FT_CW * j;
          if (col < len) {
            const double wj = ws[col];
#pragma unroll
            for (int r = 0; r < TRM; ++r)
              if (r < nr) p[r] += st[(size_t)r * dw + col] * wj;
          }
        }
        warp_sum<TRM>(p);
        if (lane == 0) {
#pragma unroll
          for (int r = 0; r < TRM; ++r) red[warp * FT_TRMAX + r] = p[r];
        }
      }
    }
    __syncthreads();
    if (sw && dot && lane < nr) {
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < FT_CW / 32; ++w) v += red[w * FT_TRMAX + lane];
      if (cs > 1) {
        for (int rk = 0; rk < cs; ++rk) ft_st_cluster(&xb[q * FT_TRMAX + lane], (unsigned)rk, v);
      } else {
        xb[lane] = v;
      }
    }
    // cluster: every rank's partial row dots are in place, and every rank has
    // read this tile's per-sample inputs (prefetched before arriving)
    if (cs > 1) ft_cluster_sync();
    else __syncthreads();
    if (sw) {
      if (lane < nr) {
        double tv[R];
        double dv = 0.0;
        if (dot)
          for (int rk = 0; rk < cs; ++rk) dv += xb[rk * FT_TRMAX + lane];
        op.input(r0 + lane, dv, pf, u, tv, writer, na);
#pragma unroll
        for (int r = 0; r < R; ++r) ts[lane * R + r] = tv[r];
      }
      const int64_t rn0 = r0 + g.tr;
      if (t + 1 < T && lane < (i1 - rn0 < g.tr ? i1 - rn0 : g.tr)) op.prefetch(rn0 + lane, pfn);
    }
    __syncthreads();
    if (!sw) {
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const int col = tid + FT_CW * j;
        if (col < len) {
#pragma unroll
          for (int r = 0; r < ft_trm(CPT); ++r)
            if (r < nr) {
              const double x = st[(size_t)r * dw + col];
#pragma unroll
              for (int rr = 0; rr < R; ++rr) acc[rr][j] += x * ts[r * R + rr];
            }
        }
      }
      ft_cw_sync();  // the column warps are done with slot k and ts
      if (tid == 0 && t + g.ns < T) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(t + g.ns);
      }
    } else {
      pf = pfn;
    }
  }

  // per-cluster partials of the R products (this CTA's slice)
  if (!sw) {
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int64_t col = tid + (int64_t)FT_CW * j;
      if (col < len) {
#pragma unroll
        for (int rr = 0; rr < R; ++rr) s.part[((int64_t)cl * R + rr) * g.ldp + c0 + col] = acc[rr][j];
      }
    }
  } else if (writer) {
    warp_sum<NN>(na);
    if (lane == 0) {
#pragma unroll
      for (int kk = 0; kk < NN; ++kk) s.npart[(int64_t)cl * NN + kk] = na[kk];
    }
  }
}

// Sum of the per-cluster partials, the per-feature epilogue and the final
// scalar logic; sharded mode publishes [v | n-sums] to the bundle instead
// (all-reduce, then zmv_epi_kernel on every rank).  A CTA covers 32
// features: warp w sums the clusters c = w, w + 8, ... in increasing order,
// then the 8 warp sums are added in warp order (fixed tree: deterministic).
constexpr int FTR_THREADS = 256;
template <class Op>
__global__ void __launch_bounds__(FTR_THREADS) zft_reduce_kernel(Op op, int64_t d, int nparts, int64_t ldp, Scratch s) {
  constexpr int R = Op::R, NN = Op::NN, ND = Op::ND;
  constexpr int NW = FTR_THREADS / 32;
  if (op.skip()) return;
  __shared__ double pw[NW][R][32];
  __shared__ double red[NW * (NN > ND ? NN : ND)];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  double v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = 0.0;
  if (j < d) {
    for (int c = warp; c < nparts; c += NW) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] += ld_cg(s.part + ((int64_t)c * R + r) * ldp + j);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) pw[warp][r][lane] = v[r];
  __syncthreads();
  double dacc[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) dacc[k] = 0.0;
  if (warp == 0 && j < d) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double a = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) a += pw[w][r][lane];
      v[r] = a;
    }
    if (s.bundle) {
#pragma unroll
      for (int r = 0; r < R; ++r) s.bundle[(int64_t)r * d + j] = v[r];
    } else {
      op.epi(j, v, dacc);
    }
  }
  if (!s.bundle) {
    block_sum<ND>(dacc, red);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < ND; ++k) s.tpart[(int64_t)blockIdx.x * ND + k] = dacc[k];
    }
  }
  if (!last_arrival(&s.tickets[0], gridDim.x)) return;
  double nsum[NN];
  block_sum_partials<NN>(s.npart, nparts, nsum, red);
  if (s.bundle) {
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < NN; ++k) s.bundle[(int64_t)R * d + k] = nsum[k];
    }
    return;
  }
  double dsum[ND];
  block_sum_partials<ND>(s.tpart, gridDim.x, dsum, red);
  if (threadIdx.x == 0) op.fin(nsum, dsum);
}

}  // namespace gdwd
