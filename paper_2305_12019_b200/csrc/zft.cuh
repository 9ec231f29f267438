// Fused "dot -> per-sample epilogue -> axpy" pass over the sample-major X
// (one HBM read where the unfused loop makes two):
//
//   for every sample i:   dot_i = x_i . w            (optional, device flag)
//                         t_i   = Op::input(i, dot_i) (per-sample update)
//   v = sum_i x_i t_i     (R right-hand sides, then a per-feature epilogue)
//
// Used for the tail of an X-space ADMM iteration (solver.py:530-541 plus the
// next iteration's Z~ [xi - r, alpha], SURVEY App. C fusion P2): Z~^T w after
// a re-solve, Step 3, then the two products the next right-hand side and
// the dual objective need.
//
// Layout.  A cluster of `cs` CTAs (one per SM) owns a contiguous range of
// samples; CTA rank q of the cluster owns the feature slice [q dw, (q+1) dw).
// Tiles of `tr` rows of the slice are staged in shared memory by bulk copies
// (TMA engine, mbarrier transaction counts), `ns` stages deep.  The CTA is
// warp-specialised and every hand-off is an mbarrier, so the roles overlap
// across tiles instead of meeting at block barriers:
//
//   producer warp  issues a stage's copies once every consumer released it
//   dot warps (6)  each owns a sixth of the slice's columns: reads a w pair
//                  once per tile and applies it to every row (double2 smem
//                  reads, FMA chains), one shuffle tree per row; partials
//                  published to every rank (DSMEM + remote arrive)
//   sample warp    one lane per row: combines the warps' and ranks' partial
//                  dots (fixed order), runs the per-sample epilogue (inputs
//                  staged FT_PFD tiles ahead by cp.async), writes t (R
//                  values per row) for the axpy
//   axpy warps (8) own column pairs of the slice; accumulate x * t over rows
//                  in registers (row order)
//
// Measured (B200, scratch harness): the pass streams at the HBM rate without
// the dot (6.6 TB/s); with it each tile carries ~1.5-2 us of dot-warp work
// and hand-off latency, so tiles of >= 48 KB per SM are needed to stay near
// the HBM rate -- the plan only enables the pass where such tiles fit.
// Determinism: the row dot is a fixed chain/shuffle tree, then a fixed sum
// over ranks; the axpy accumulates in row order; per-cluster partials are
// summed in a fixed order by zft_reduce_kernel.  Every rank of a cluster
// computes the same epilogue from the same inputs; only rank 0 writes the
// per-sample outputs (Op::input must not overwrite an array it reads).
#pragma once
#include "zops.cuh"

namespace gdwd {

constexpr int FT_THREADS = 512;
// 6 dot + 8 axpy warps: at d = 1000 (c3) eight axpy warps still hold two
// column pairs per thread, and the dot warps -- the longer chain per tile --
// each get 84 instead of 125 pairs: 388 -> 368 us per pass (4 + 10: 388,
// 5 + 9: 410, 7 + 7: four-row tiles, slower)
#ifndef FT_NDW_V
#define FT_NDW_V 6
#endif
constexpr int FT_NDW = FT_NDW_V;                    // dot warps 0..NDW-1
constexpr int FT_AW0 = FT_NDW, FT_NAW = 14 - FT_NDW;  // axpy warps NDW..13
constexpr int FT_NA = FT_NAW * 32;        // axpy threads
constexpr int FT_PW = 14, FT_SW = 15;     // producer warp, sample warp
constexpr int FT_TRMAX = 8;               // rows per stage
constexpr int FT_CSMAX = 8;               // CTAs per cluster
constexpr int FT_NSMAX = 8;               // stages
constexpr int FT_RING = 4;                // depth of the dot / t hand-off rings (tiles in flight between roles)
constexpr int FT_PFD = 6;                 // tiles of per-sample inputs in flight (cp.async ring)
constexpr int FT_NPF = 8;                 // max per-sample input fields

struct FtGeom {
  int cs;        // CTAs per cluster (feature slices)
  int clusters;  // co-resident clusters (exactly one wave)
  int dw;        // slice width (even)
  int tr;        // rows per stage
  int ns;        // stages
  int64_t ldp;   // stride of the per-cluster partial rows (>= d, even)
};

// rows per stage the row loops unroll for: wide slices (many column pairs per
// axpy thread) stage few rows, which keeps the accumulators in registers
__host__ __device__ constexpr int ft_tra(int p2) { return p2 >= 8 ? 2 : (p2 >= 4 ? 4 : FT_TRMAX); }
// column pairs per axpy thread for a slice of dw columns
__host__ __device__ constexpr int ft_pairs(int dw) { return (dw / 2 + FT_NA - 1) / FT_NA; }

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
GDWD_DEV unsigned ft_mapa(const void* local, unsigned rank) {
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  return ra;
}
GDWD_DEV void ft_st_remote(unsigned addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
// arrive on an mbarrier of cluster CTA `rank` (release at cluster scope:
// this thread's earlier shared::cluster writes are visible to the waiter)
GDWD_DEV void ft_arrive_remote(unsigned long long* local_bar, unsigned rank) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ft_mapa(local_bar, rank))
               : "memory");
}
GDWD_DEV void ft_arrive_remote_relaxed(unsigned long long* local_bar, unsigned rank) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(ft_mapa(local_bar, rank))
               : "memory");
}
GDWD_DEV void ft_cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
GDWD_DEV void ft_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
GDWD_DEV void ft_cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
#ifndef FT_WAIT_MODE
#define FT_WAIT_MODE 0
#endif
// wait for the phase of parity `par` (CTA scope)
GDWD_DEV void ft_wait(unsigned long long* bar, unsigned par) {
#if FT_WAIT_MODE == 1
  asm volatile(
      "{\n .reg .pred p;\n W_%=:\n mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(par)
      : "memory");
#else
  mbar_wait(bar, par);
#endif
}
GDWD_DEV void ft_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// wait for the phase of parity `par`; cluster scope when remote arrivals feed it
GDWD_DEV void ft_wait_cluster(unsigned long long* bar, unsigned par) {
  asm volatile(
      "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(par)
      : "memory");
}

// diagnostics (build with -DGDWD_FT_TIMING, run with GDWD_FT_TIMING=1):
// globaltimer stamps per tile of CTA 0 (each stamp costs a global load, so
// the stamped build is slower than the production one)
__device__ unsigned long long* g_ft_ts = nullptr;
constexpr int FT_TS_TILES = 512, FT_TS_PTS = 16;
GDWD_DEV unsigned long long ft_now() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}
#ifdef GDWD_FT_TIMING
#define FTS(slot)                                                                                  \
  do {                                                                                             \
    if (g_ft_ts && blockIdx.x == 0 && t < FT_TS_TILES) g_ft_ts[t * FT_TS_PTS + (slot)] = ft_now(); \
  } while (0)
#else
#define FTS(slot) \
  do {            \
  } while (0)
#endif

inline size_t ft_smem_bytes(const FtGeom& g, int R) {
  return ((size_t)(g.ns * g.tr + 1) * g.dw + (size_t)FT_RING * FT_TRMAX * R + FT_RING * (size_t)g.cs * FT_NDW * FT_TRMAX +
          FT_PFD * FT_TRMAX * FT_NPF) *
             sizeof(double) +
         (2 * FT_NSMAX + 4 * FT_RING) * sizeof(unsigned long long);
}

template <class Op, int P2>
__global__ void __launch_bounds__(FT_THREADS, 1) zft_kernel(Op op, MatView X, FtGeom g, Scratch s) {
  constexpr int R = Op::R, NN = Op::NN;
  if (op.skip()) return;  // grid-uniform (a flag no CTA of this kernel writes)
  extern __shared__ __align__(16) double fsm[];
  const int dw = g.dw, ns = g.ns, cs = g.cs;
  double* stage = fsm;                                      // [ns][tr][dw]
  double* ws = stage + (size_t)ns * g.tr * dw;              // [dw]      this slice of w
  double* ts = ws + dw;                                     // [RING][FT_TRMAX][R]
  double* xch = ts + FT_RING * FT_TRMAX * R;                // [RING][cs][FT_NDW][FT_TRMAX] partial row dots
  double* pfr = xch + FT_RING * cs * FT_NDW * FT_TRMAX;  // [PFD][FT_TRMAX][NPF] per-sample inputs
  unsigned long long* full = reinterpret_cast<unsigned long long*>(pfr + FT_PFD * FT_TRMAX * FT_NPF);
  unsigned long long* empty = full + FT_NSMAX;
  unsigned long long* dotd = empty + FT_NSMAX;  // [RING] row dots of every rank in place
  unsigned long long* xfree = dotd + FT_RING;   // [RING] every rank's sample warp has read them
  unsigned long long* tsr = xfree + FT_RING;    // [RING] t of the tile written
  unsigned long long* tsfree = tsr + FT_RING;   // [RING] every axpy warp has read it
  const unsigned q = cs > 1 ? ft_cluster_rank() : 0u;
  const int cl = cs > 1 ? (int)ft_cluster_id() : (int)blockIdx.x;
  const int64_t c0 = (int64_t)q * dw;
  const int64_t len = c0 < X.cols ? (X.cols - c0 < dw ? X.cols - c0 : dw) : 0;
  const int64_t lenp = (len + 1) & ~(int64_t)1;  // even: inside ld's zero padding
  const int64_t i0 = X.rows * cl / g.clusters, i1 = X.rows * (cl + 1) / g.clusters;
  const int64_t T = (i1 - i0 + g.tr - 1) / g.tr;
  const bool dot = op.need_dot();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto rows_of = [&](int64_t t) -> int { return (int)(i1 - (i0 + t * g.tr) < g.tr ? i1 - (i0 + t * g.tr) : g.tr); };

  if (tid == 0) {
    for (int k = 0; k < ns; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], FT_NDW + FT_NAW);
    }
    for (int b = 0; b < FT_RING; ++b) {
      mbar_init(&dotd[b], FT_NDW * cs);
      mbar_init(&xfree[b], cs);
      mbar_init(&tsr[b], 1);
      mbar_init(&tsfree[b], FT_NAW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  for (int64_t j = tid; j < lenp; j += FT_THREADS) ws[j] = (dot && j < len) ? op.wval(c0 + j) : 0.0;
  __syncthreads();
  if (cs > 1) ft_cluster_sync();  // peers' barriers initialised before any remote arrive

  if (warp == FT_PW) {
    // ---- producer ----------------------------------------------------------
    if (lane == 0) {
      const unsigned rowbytes = (unsigned)(lenp * sizeof(double));
      for (int64_t t = 0; t < T; ++t) {
        const int k = (int)(t % ns);
        FTS(0);
        ft_wait(&empty[k], (unsigned)(((t / ns) & 1) ^ 1));
        FTS(1);
        const int nr = rows_of(t);
        const int64_t r0 = i0 + t * g.tr;
        double* dst = stage + (size_t)k * g.tr * dw;
        mbar_arrive_expect_tx(&full[k], (unsigned)nr * rowbytes);
        if (rowbytes)
          for (int r = 0; r < nr; ++r) bulk_g2s(dst + (size_t)r * dw, X.a + (r0 + r) * X.ld + c0, rowbytes, &full[k]);
      }
    }
  } else if (warp < FT_NDW) {
    // ---- dot warps: warp w owns a quarter of the slice's column pairs; per
    // tile it reads each w pair once and applies it to every row --------------
    const int np2 = (int)(lenp >> 1);
    const int cw = (np2 + FT_NDW - 1) / FT_NDW;
    const int pa = warp * cw, pb = pa + cw < np2 ? pa + cw : np2;
    const double2* wr = reinterpret_cast<const double2*>(ws);
    constexpr int TRA = ft_tra(P2);
    for (int64_t t = 0; t < T; ++t) {
      const int k = (int)(t % ns), b = (int)(t % FT_RING);
      const int nr = rows_of(t);
      ft_wait(&full[k], (unsigned)((t / ns) & 1));
      if (dot) {
        ft_wait(&xfree[b], (unsigned)(((t / FT_RING) & 1) ^ 1));
        const double2* st = reinterpret_cast<const double2*>(stage + (size_t)k * g.tr * dw);
        const int dw2 = dw >> 1;
        double a0[FT_TRMAX], a1[FT_TRMAX];
#pragma unroll
        for (int r = 0; r < FT_TRMAX; ++r) a0[r] = a1[r] = 0.0;
#pragma unroll 2
        for (int p = pa + lane; p < pb; p += 32) {
          const double2 w2 = wr[p];
          double2 x[TRA];
#pragma unroll
          for (int r = 0; r < TRA; ++r)
            if (r < nr) x[r] = st[r * dw2 + p];
#pragma unroll
          for (int r = 0; r < TRA; ++r)
            if (r < nr) {
              a0[r] = __fma_rn(x[r].x, w2.x, a0[r]);
              a1[r] = __fma_rn(x[r].y, w2.y, a1[r]);
            }
        }
#pragma unroll
        for (int r = 0; r < FT_TRMAX; ++r) a0[r] += a1[r];
        if (TRA > 4 && nr > 4) warp_sum<8>(a0);
        else if (TRA > 2 && nr > 2) warp_sum<4>(reinterpret_cast<double(&)[4]>(a0));
        else if (TRA > 1 && nr > 1) warp_sum<2>(reinterpret_cast<double(&)[2]>(a0));
        else warp_sum<1>(reinterpret_cast<double(&)[1]>(a0));
        if (lane == 0) {
          // this warp's partial row dots -> every rank's xch[b][q][warp][r]
          double* dst = xch + ((b * cs + q) * FT_NDW + warp) * FT_TRMAX;
#pragma unroll
          for (int r = 0; r < TRA; ++r)
            if (r < nr) {
              if (cs > 1) {
                for (int rk = 0; rk < cs; ++rk) ft_st_remote(ft_mapa(dst + r, (unsigned)rk), a0[r]);
              } else {
                dst[r] = a0[r];
              }
            }
          if (cs > 1) {
            for (int rk = 0; rk < cs; ++rk) ft_arrive_remote(&dotd[b], (unsigned)rk);
          } else {
            ft_arrive(&dotd[b]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) ft_arrive(&empty[k]);  // done with the stage
    }
  } else if (warp < FT_AW0 + FT_NAW) {
    // ---- axpy warps: column pairs ta, ta + FT_NA, ... ------------------------
    const int ta = tid - FT_AW0 * 32;
    constexpr int TRA = ft_tra(P2);
    double acc[R][2 * P2];
#pragma unroll
    for (int j = 0; j < 2 * P2; ++j)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r][j] = 0.0;
    const int np2 = (int)(lenp >> 1);
    for (int64_t t = 0; t < T; ++t) {
      const int k = (int)(t % ns), b = (int)(t % FT_RING);
      const int nr = rows_of(t);
      ft_wait(&full[k], (unsigned)((t / ns) & 1));
      ft_wait(&tsr[b], (unsigned)((t / FT_RING) & 1));
      double tv[TRA][R];
#pragma unroll
      for (int r = 0; r < TRA; ++r)
#pragma unroll
        for (int rr = 0; rr < R; ++rr) tv[r][rr] = r < nr ? ts[(b * FT_TRMAX + r) * R + rr] : 0.0;
      __syncwarp();
      if (lane == 0) ft_arrive(&tsfree[b]);
      const double* st = stage + (size_t)k * g.tr * dw;
#pragma unroll
      for (int j = 0; j < P2; ++j) {
        const int p = ta + FT_NA * j;
        if (p < np2) {
          double2 x[TRA];  // all rows' loads in flight before the FMAs
#pragma unroll
          for (int r = 0; r < TRA; ++r)
            if (r < nr) x[r] = reinterpret_cast<const double2*>(st + (size_t)r * dw)[p];
#pragma unroll
          for (int r = 0; r < TRA; ++r)
            if (r < nr) {
#pragma unroll
              for (int rr = 0; rr < R; ++rr) {
                acc[rr][2 * j] = __fma_rn(x[r].x, tv[r][rr], acc[rr][2 * j]);
                acc[rr][2 * j + 1] = __fma_rn(x[r].y, tv[r][rr], acc[rr][2 * j + 1]);
              }
            }
        }
      }
      __syncwarp();
      if (lane == 0) ft_arrive(&empty[k]);
    }
    // per-cluster partials of the R products (this CTA's slice)
#pragma unroll
    for (int j = 0; j < P2; ++j) {
      const int64_t col = 2 * (int64_t)(ta + FT_NA * j);
      if (col < len) {
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          double* o = s.part + ((int64_t)cl * R + rr) * g.ldp + c0 + col;
          o[0] = acc[rr][2 * j];
          if (col + 1 < len) o[1] = acc[rr][2 * j + 1];
        }
      }
    }
  } else {
    // ---- sample warp: one lane per row ---------------------------------------
    double na[NN];
#pragma unroll
    for (int kk = 0; kk < NN; ++kk) na[kk] = 0.0;
    const typename Op::U u = op.uniform();
    // per-sample inputs FT_PFD tiles ahead by cp.async (loads under a
    // saturated HBM take microseconds: one tile of lead is not enough)
    auto pf_issue = [&](int64_t tt) {
      if (tt < T && lane < rows_of(tt)) {
        double* slot = pfr + ((int)(tt % FT_PFD) * FT_TRMAX + lane) * FT_NPF;
#pragma unroll
        for (int f = 0; f < Op::NPF; ++f) ft_cp_async8(slot + f, op.pf_src(f, i0 + tt * g.tr + lane));
      }
      ft_cp_commit();  // one group per tile, empty or not
    };
#pragma unroll 1
    for (int tt = 0; tt < FT_PFD; ++tt) pf_issue(tt);
    for (int64_t t = 0; t < T; ++t) {
      const int b = (int)(t % FT_RING);
      const int nr = rows_of(t);
      const int64_t r0 = i0 + t * g.tr;
      double dv = 0.0;
      if (dot) {
        if (lane == 0) FTS(8);
        if (cs > 1) ft_wait_cluster(&dotd[b], (unsigned)((t / FT_RING) & 1));  // remote arrivals
        else ft_wait(&dotd[b], (unsigned)((t / FT_RING) & 1));
        if (lane == 0) FTS(9);
        if (lane < nr)
          for (int rk = 0; rk < cs; ++rk)
#pragma unroll
            for (int w = 0; w < FT_NDW; ++w) dv += xch[((b * cs + rk) * FT_NDW + w) * FT_TRMAX + lane];
        __syncwarp();
        if (lane == 0) {
          if (cs > 1) {
            // relaxed: the values read are consumed (dv) before the arrive, and a
            // release here would wait for this warp's global output stores
            for (int rk = 0; rk < cs; ++rk) ft_arrive_remote_relaxed(&xfree[b], (unsigned)rk);
          } else {
            ft_arrive(&xfree[b]);
          }
        }
      }
      double tv[R];
      if (lane == 0) FTS(10);
      ft_cp_wait<FT_PFD - 1>();  // this thread's copies of tile t have landed
      if (lane < nr) {
        typename Op::Pf pf;
        op.load_pf(pfr + ((int)(t % FT_PFD) * FT_TRMAX + lane) * FT_NPF, pf);
        op.input(r0 + lane, dv, pf, u, tv, q == 0, na);
      }
      pf_issue(t + FT_PFD);  // into the slot just read (same lane)
      if (lane == 0) FTS(11);
      ft_wait(&tsfree[b], (unsigned)(((t / FT_RING) & 1) ^ 1));
      if (lane < nr) {
#pragma unroll
        for (int rr = 0; rr < R; ++rr) ts[(b * FT_TRMAX + lane) * R + rr] = tv[rr];
      }
      __syncwarp();
      if (lane == 0) FTS(12);
      if (lane == 0) ft_arrive(&tsr[b]);
    }
    if (q == 0) {
      warp_sum<NN>(na);
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < NN; ++kk) s.npart[(int64_t)cl * NN + kk] = na[kk];
      }
    }
  }
  // no CTA leaves while a peer may still arrive on its barriers
  if (cs > 1) {
    __syncthreads();
    ft_cluster_sync();
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
