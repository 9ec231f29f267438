// Sparse counterparts of zmv / ztmv (zops.cuh) for Z~ stored in both
// orientations (reference linalg/sparse.py: the scipy CSC view and its .T):
//
//   CSR by feature (rowptr[d+1], colidx, val): Z~ t   -- one warp per feature
//   CSC by sample  (colptr[n+1], rowidx, val): Z~^T w -- G lanes per sample
//
// Both use the same Op functors as the dense kernels, so every fused
// epilogue (Newton prox, h/h2/residual updates, PSQMR scalars) is shared.
// Z~ t needs its inputs materialised first (each sample appears in many
// feature rows): sp_prep writes t_r[i] = op.input(i) and the n-sum partials.
// Indices are int32 (nnz < 2^31 per shard), row pointers int64.  Summation
// order is fixed (lane-strided, fixed shuffle tree, fixed partial order), so
// results are deterministic.
#pragma once
#include "common.cuh"
#include "zops.cuh"

namespace gdwd {

struct SpView {
  const int64_t* ptr;  // rows+1 (CSR: features; CSC: samples)
  const int* idx;
  const double* val;
  int64_t rows;   // number of compressed rows (d for CSR, n for CSC)
  int64_t other;  // length of the gathered vector (n for CSR, d for CSC)
};

constexpr int SP_THREADS = 256;
constexpr int SPU = 4;  // nonzeros per lane in flight in the gather loops

// t_r[i] for all samples + n-sum partials (one partial per CTA)
template <class Op>
__global__ void __launch_bounds__(SP_THREADS) sp_prep_kernel(Op op, int64_t n, double* tbuf, Scratch s) {
  constexpr int R = Op::R, NN = Op::NN;
  if (op.skip()) return;
  __shared__ double red[(SP_THREADS / 32) * NN];
  double nacc[NN];
#pragma unroll
  for (int k = 0; k < NN; ++k) nacc[k] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)SP_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * SP_THREADS) {
    double tv[R];
    op.input(i, tv, nacc);
#pragma unroll
    for (int r = 0; r < R; ++r) tbuf[i * R + r] = tv[r];  // interleaved: one gather per nnz
  }
  block_sum<NN>(nacc, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NN; ++k) s.npart[(int64_t)blockIdx.x * NN + k] = nacc[k];
  }
}

// v_j = sum_i Z[j,i] t_i (CSR rows = features), epilogue per feature, then
// the global finaliser sums the prep kernel's nprep n-partials and the
// per-CTA d-partials.
template <class Op>
__global__ void __launch_bounds__(SP_THREADS) sp_zmv_kernel(Op op, SpView A, const double* tbuf, int nprep,
                                                            Scratch s) {
  constexpr int R = Op::R, NN = Op::NN, ND = Op::ND;
  if (op.skip()) return;
  __shared__ double red[(SP_THREADS / 32) * ND];
  __shared__ double red2[(SP_THREADS / 32) * (NN > ND ? NN : ND)];
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)SP_THREADS + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * SP_THREADS) >> 5;
  double dacc[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) dacc[k] = 0.0;
  for (int64_t j = warp; j < A.rows; j += nwarps) {
    const int64_t b = A.ptr[j], e = A.ptr[j + 1];
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    // SPU nnz per lane in flight: all index / value loads of a batch, then
    // all gathers, then the accumulation (lane order k, k+32, ... as before)
    for (int64_t k0 = b + lane; k0 < e; k0 += 32 * SPU) {
      double v[SPU];
      int c[SPU];
#pragma unroll
      for (int u = 0; u < SPU; ++u) {  // clamped, not predicated: never past the row's end
        const int64_t k = k0 + 32 * u, kk = k < e ? k : e - 1;
        const double vv = __ldg(A.val + kk);
        v[u] = k < e ? vv : 0.0;
        c[u] = __ldg(A.idx + kk);
      }
      double tg[SPU][R];
#pragma unroll
      for (int u = 0; u < SPU; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r) tg[u][r] = tbuf[(int64_t)c[u] * R + r];
#pragma unroll
      for (int u = 0; u < SPU; ++u)
        if (k0 + 32 * u < e) {
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] += v[u] * tg[u][r];
        }
    }
    warp_sum<R>(acc);
    if (lane == 0) {
      if (s.bundle) {
#pragma unroll
        for (int r = 0; r < R; ++r) s.bundle[(int64_t)r * A.rows + j] = acc[r];
      } else {
        op.epi(j, acc, dacc);
      }
    }
  }
  block_sum<ND>(dacc, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < ND; ++k) s.tpart[(int64_t)blockIdx.x * ND + k] = dacc[k];
  }
  if (!last_arrival(&s.tickets[0], gridDim.x)) return;
  double nsum[NN], dsum[ND];
  block_sum_partials<NN>(s.npart, nprep, nsum, red2);
  block_sum_partials<ND>(s.tpart, gridDim.x, dsum, red2);
  if (threadIdx.x == 0) {
    if (s.bundle) {
#pragma unroll
      for (int k = 0; k < NN; ++k) s.bundle[(int64_t)R * A.rows + k] = nsum[k];
    } else {
      op.fin(nsum, dsum);
    }
  }
}

// ---------------------------------------------------------------------------
// Z~ t on a sample-blocked sliced ELL (built at upload, gdwd.cu).  The CSR
// gather kernel above is bound by the L1TEX pipe: every nonzero is its own
// 8-byte gather of t from L2.  Here the samples are cut into blocks of
// SB_S = 12288 (t's block, R values per sample, fits shared memory); within a
// block the features are sorted by entry count and cut into 32-wide slices
// stored column-major (entry e of lane l at base + 32 e + l: coalesced value
// and 16-bit block-local index loads), so each lane sums one feature's
// entries of the block in sample order, gathering t from shared memory.
// Every (block, feature) partial is written (zero when empty); a second
// kernel sums them over the blocks in block order and runs the epilogue --
// per feature the entries are still summed in sample order, blocks in order.
// CTAs take equal shares of the entries (chunks of consecutive slices, at
// most a block boundary or two inside a chunk: t is restaged there).
// ---------------------------------------------------------------------------
constexpr int SB_S = 12288;       // samples per block
constexpr int SB_THREADS = 512;
constexpr int SB_CHUNKS = 2 * 148;  // chunk boundaries: 2 per SM (R = 1), pairs for R = 2
#ifndef SB_U_V
#define SB_U_V 8
#endif
constexpr int SB_U = SB_U_V;      // entries per lane in flight

struct SbView {
  const double* val;
  const unsigned short* idx;
  const int64_t* base;  // per slice: first entry
  const int* h;         // per slice: entries per lane
  const int* perm;      // per slice and lane: feature (-1: pad lane)
  const int* chunk;     // SB_CHUNKS + 1 slice boundaries
  int nslpb;            // slices per block (ceil(d / 32))
  int nb;               // blocks
  int64_t n, d;
};

// threads per CTA: R = 1 stages 96 KB of t (2 CTAs of 512 per SM), R = 2
// stages 192 KB (one CTA of 1024 per SM): 32 warps per SM either way
template <int R>
__host__ __device__ constexpr int sb_threads() { return R == 1 ? SB_THREADS : 2 * SB_THREADS; }

template <class Op>
__global__ void __launch_bounds__(sb_threads<Op::R>()) sp_zmv_sb_kernel(Op op, SbView A, const double* tbuf,
                                                                       double* part) {
  constexpr int R = Op::R;
  constexpr int NT = sb_threads<R>();
  if (op.skip()) return;
  extern __shared__ __align__(16) double tsm[];  // [SB_S][R]
  constexpr int PER = R == 1 ? 1 : 2;           // chunks per CTA (grid SB_CHUNKS / PER)
  const int s0 = A.chunk[blockIdx.x * PER], s1 = A.chunk[blockIdx.x * PER + PER];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = NT >> 5;
  for (int s = s0; s < s1;) {
    const int b = s / A.nslpb;
    const int se = s1 < (b + 1) * A.nslpb ? s1 : (b + 1) * A.nslpb;
    const int64_t i0 = (int64_t)b * SB_S;
    const int cnt = (int)(A.n - i0 < SB_S ? A.n - i0 : SB_S);
    __syncthreads();  // the previous block's gathers are done
    {
      const double2* src = reinterpret_cast<const double2*>(tbuf + i0 * R);
      double2* dst = reinterpret_cast<double2*>(tsm);
      for (int k = threadIdx.x; k < (cnt * R + 1) / 2; k += NT) dst[k] = __ldcg(src + k);
    }
    __syncthreads();
    for (int ss = s + warp; ss < se; ss += nw) {
      const int h = A.h[ss];
      const int64_t base = A.base[ss] + lane;
      const int j = A.perm[(int64_t)ss * 32 + lane];
      double acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = 0.0;
      int e = 0;
      for (; e + SB_U <= h; e += SB_U) {
        double v[SB_U];
        int ix[SB_U];
#pragma unroll
        for (int u = 0; u < SB_U; ++u) {
          v[u] = __ldcs(A.val + base + 32 * (int64_t)(e + u));
          ix[u] = __ldcs(A.idx + base + 32 * (int64_t)(e + u));
        }
#pragma unroll
        for (int u = 0; u < SB_U; ++u)
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] += v[u] * tsm[ix[u] * R + r];
      }
      // (a predicated whole-batch tail instead of this loop measured slower: 80.6 vs 74.5 us at c4)
      for (; e < h; ++e) {
        const double v = __ldcs(A.val + base + 32 * (int64_t)e);
        const int ix = __ldcs(A.idx + base + 32 * (int64_t)e);
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] += v * tsm[ix * R + r];
      }
      if (j >= 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) part[((int64_t)b * A.d + j) * R + r] = acc[r];
      }
    }
    s = se;
  }
}

// v_j = sum of the per-block partials; per-feature epilogue, then the
// finaliser (the prep kernel's n-partials and the d-partials) -- the tail of
// sp_zmv_kernel.  Per feature: warp w sums blocks w, w + 8, ... in order,
// then the 8 warp sums are added in warp order (fixed tree).
// SBR_F features per lane (a CTA covers 32 SBR_F features): one wave of CTAs
// at c4 (782 for d = 50000) instead of two waves of 1563 latency-bound ones.
constexpr int SBR_F = 2;
template <class Op>
__global__ void __launch_bounds__(SP_THREADS) sp_zmv_sb_reduce_kernel(Op op, const double* part, int nb, int64_t d,
                                                                    int nprep, Scratch s) {
  constexpr int R = Op::R, NN = Op::NN, ND = Op::ND;
  constexpr int NW = SP_THREADS / 32;
  if (op.skip()) return;
  __shared__ double pw[NW][SBR_F][R][32];
  __shared__ double red2[NW * (NN > ND ? NN : ND)];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j0 = (int64_t)blockIdx.x * (32 * SBR_F) + lane;
  double v[SBR_F][R];
#pragma unroll
  for (int f = 0; f < SBR_F; ++f)
#pragma unroll
    for (int r = 0; r < R; ++r) v[f][r] = 0.0;
#pragma unroll 2
  for (int b = warp; b < nb; b += NW) {
#pragma unroll
    for (int f = 0; f < SBR_F; ++f) {
      const int64_t j = j0 + 32 * f;
      if (j < d) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[f][r] += __ldcg(part + ((int64_t)b * d + j) * R + r);
      }
    }
  }
#pragma unroll
  for (int f = 0; f < SBR_F; ++f)
#pragma unroll
    for (int r = 0; r < R; ++r) pw[warp][f][r][lane] = v[f][r];
  __syncthreads();
  double dacc[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) dacc[k] = 0.0;
  if (warp < SBR_F) {  // warp f finishes the CTA's f-th group of 32 features
    const int f = warp;
    const int64_t j = j0 + 32 * f;
    if (j < d) {
      double vv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double a = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) a += pw[w][f][r][lane];
        vv[r] = a;
      }
      if (s.bundle) {
#pragma unroll
        for (int r = 0; r < R; ++r) s.bundle[(int64_t)r * d + j] = vv[r];
      } else {
        op.epi(j, vv, dacc);
      }
    }
  }
  block_sum<ND>(dacc, red2);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < ND; ++k) s.tpart[(int64_t)blockIdx.x * ND + k] = dacc[k];
  }
  if (!last_arrival(&s.tickets[0], gridDim.x)) return;
  double nsum[NN], dsum[ND];
  block_sum_partials<NN>(s.npart, nprep, nsum, red2);
  block_sum_partials<ND>(s.tpart, gridDim.x, dsum, red2);
  if (threadIdx.x == 0) {
    if (s.bundle) {
#pragma unroll
      for (int k = 0; k < NN; ++k) s.bundle[(int64_t)R * d + k] = nsum[k];
    } else {
      op.fin(nsum, dsum);
    }
  }
}

// dot_i = sum_j Z[j,i] w_j (CSC columns = samples).  A warp takes 32
// consecutive samples: in 32/G rounds each group of G lanes reduces one
// sample's dot, which is parked in the lane with that sample's index; then
// all 32 lanes run the per-sample epilogue (Newton etc.) together.
template <class Op, int G>
__global__ void __launch_bounds__(SP_THREADS) sp_ztmv_kernel(Op op, SpView A, Scratch s) {
  constexpr int NN = Op::NN;
  constexpr int GROUPS = 32 / G;
  if (op.skip()) return;
  __shared__ double red[(SP_THREADS / 32) * NN];
  const int lane = threadIdx.x & 31, sub = lane & (G - 1), grp = lane / G;
  const int64_t warp = (blockIdx.x * (int64_t)SP_THREADS + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * SP_THREADS) >> 5;
  double nacc[NN];
#pragma unroll
  for (int k = 0; k < NN; ++k) nacc[k] = 0.0;
  for (int64_t base = warp * 32; base < A.rows; base += nwarps * 32) {
    double mine = 0.0;
#pragma unroll
    for (int t = 0; t < G; ++t) {
      const int64_t i = base + grp * G + t;  // sample handled by this group in round t
      double acc = 0.0;
      if (i < A.rows) {
        const int64_t b = A.ptr[i], e = A.ptr[i + 1];
        // SPU entries per lane in flight: index / value loads, then gathers
        for (int64_t k0 = b + sub; k0 < e; k0 += (int64_t)G * SPU) {
          double v[SPU];
          int c[SPU];
#pragma unroll
          for (int u = 0; u < SPU; ++u) {  // clamped, not predicated: never past the sample's end
            const int64_t k = k0 + (int64_t)G * u, kk = k < e ? k : e - 1;
            const double vv = __ldg(A.val + kk);
            v[u] = k < e ? vv : 0.0;
            c[u] = __ldg(A.idx + kk);
          }
          double wg[SPU];
#pragma unroll
          for (int u = 0; u < SPU; ++u) wg[u] = op.wval(c[u]);
#pragma unroll
          for (int u = 0; u < SPU; ++u)
            if (k0 + (int64_t)G * u < e) acc += v[u] * wg[u];
        }
      }
#pragma unroll
      for (int off = G / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (sub == t) mine = acc;  // lane grp*G + t owns sample base + grp*G + t
    }
    const int64_t i = base + lane;
    if (i < A.rows) op.row(i, mine, nacc);
  }
  (void)GROUPS;
  if (!Op::HAS_FIN) return;
  block_sum<NN>(nacc, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NN; ++k) s.npart[(int64_t)blockIdx.x * NN + k] = nacc[k];
  }
  if (!last_arrival(&s.tickets[0], gridDim.x)) return;
  double nsum[NN];
  block_sum_partials<NN>(s.npart, gridDim.x, nsum, red);
  if (threadIdx.x == 0) {
    if (s.bundle) {
#pragma unroll
      for (int k = 0; k < NN; ++k) s.bundle[k] = nsum[k];
    } else {
      op.fin(nsum);
    }
  }
}

// ---------------------------------------------------------------------------
// Feature-blocked, sliced-ELL storage for Z~^T w.  The plain CSC kernel is
// bound by its gathers of w (random 8-byte reads of a d-vector, one L1TEX
// tag lookup each).  Here the samples are split into `parts` contiguous
// ranges (one CTA each) and the features into blocks of `fb` (<= 65535):
// the CTA stages w's block in shared memory (op.wval, the values the CSC
// kernel gathers) and gathers from there.  Within (part, block) the samples
// are ordered by their entry count (descending) and cut into slices of 32;
// slice q stores its entries column-major (entry j of the slice's lane l at
// base_q + 32 j + l), padded to the slice's longest sample, so a warp reads
// 32 consecutive values and 16-bit block-local indices per step -- fully
// coalesced -- and each lane sums its own sample's entries in CSC order.
// Each sample's running dot stays in shared memory across the blocks (block
// order fixed: deterministic); the per-sample epilogue runs at the end.
//   sbase[(p*nb + f)*(Q+1) + q]: first padded entry of slice q (Q = S/32 slices)
//   perm / cnt[((p*nb + f)*Q + q)*32 + l]: local sample (0xffff: none) and entry count of lane l
// ---------------------------------------------------------------------------
struct FbView {
  const int* sbase;
  const unsigned short* perm;
  const unsigned short* cnt;
  const unsigned short* idx;
  const double* val;
  int64_t n, d;
  int nb, fb, parts, S, Q;
};

// 512 threads, two CTAs per SM (<= 64 registers), one slice per warp and
// four of its rows in flight (FB_H = 1, FB_U = 4 in gdwd.cu): c4 77.8 us per
// pass.  Measured alternatives: 256 threads with H = 2, U = 8 (round 1) 98.7;
// 512 threads with H = 2, U = 8 / 4 91.2 / 80.4, H = 1, U = 8 / 2 82.8 / 81.6;
// 448-1024 threads with H = 1, U = 4 76.3-80.8 (a plateau).
#ifndef FB_THREADS_V
#define FB_THREADS_V 512
#endif
constexpr int FB_THREADS = FB_THREADS_V;
template <class Op, int H, int U>
#ifndef FB_MINB
#define FB_MINB 2
#endif
__global__ void __launch_bounds__(FB_THREADS, FB_MINB) sp_ztmv_fb_kernel(Op op, FbView A, Scratch s) {
  constexpr int NN = Op::NN;
  if (op.skip()) return;
  extern __shared__ double fbsm[];
  double* wsm = fbsm;          // [fb] staged w block
  double* dot = fbsm + A.fb;   // [S] running dots of the part's samples
  __shared__ double red[(FB_THREADS / 32) * NN];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int p = blockIdx.x;
  const int64_t s0 = (int64_t)p * A.S;
  const int ns = s0 < A.n ? (int)min((int64_t)A.S, A.n - s0) : 0;
  for (int f = 0; f < A.nb; ++f) {
    const int64_t j0 = (int64_t)f * A.fb;
    const int jn = (int)min((int64_t)A.fb, A.d - j0);
    __syncthreads();  // the previous block's gathers are done
    for (int j = threadIdx.x; j < jn; j += FB_THREADS) wsm[j] = op.wval(j0 + j);
    __syncthreads();
    const int64_t pf = (int64_t)p * A.nb + f;
    const int* sb = A.sbase + pf * (A.Q + 1);
    // H slices per warp at a time (H*U rows in flight per lane)
    for (int q0 = H * warp; q0 < A.Q; q0 += H * (FB_THREADS / 32)) {
      int b[H], len[H], ls[H], c[H];
      double acc[H];
#pragma unroll
      for (int h = 0; h < H; ++h) {
        acc[h] = 0.0;
        const int q = q0 + h < A.Q ? q0 + h : q0;
        b[h] = sb[q];
        len[h] = q0 + h < A.Q ? (sb[q + 1] - b[h]) >> 5 : 0;
        const int64_t pl = (pf * A.Q + q) * 32 + lane;
        ls[h] = q0 + h < A.Q ? A.perm[pl] : 0xffff;
        c[h] = A.cnt[pl];
      }
      int lmax = 0;
#pragma unroll
      for (int h = 0; h < H; ++h) lmax = len[h] > lmax ? len[h] : lmax;
      for (int j0 = 0; j0 < lmax; j0 += U) {
        double v[H][U];
        int ix[H][U];
#pragma unroll
        for (int h = 0; h < H; ++h)
#pragma unroll
          for (int u = 0; u < U; ++u) {  // clamped rows of the slice: never past its end
            const int j = j0 + u < len[h] ? j0 + u : (len[h] > 0 ? len[h] - 1 : 0);
            const int64_t at = (int64_t)b[h] + 32 * j + lane;
            v[h][u] = len[h] > 0 ? __ldg(A.val + at) : 0.0;
            ix[h][u] = len[h] > 0 ? __ldg(A.idx + at) : 0;
          }
#pragma unroll
        for (int h = 0; h < H; ++h)
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (j0 + u < c[h]) acc[h] += v[h][u] * wsm[ix[h][u]];
      }
#pragma unroll
      for (int h = 0; h < H; ++h)
        if (ls[h] < ns) dot[ls[h]] = (f == 0) ? acc[h] : dot[ls[h]] + acc[h];  // pad lanes: ls = 0xffff
    }
  }
  __syncthreads();
  double nacc[NN];
#pragma unroll
  for (int k = 0; k < NN; ++k) nacc[k] = 0.0;
  for (int ls = threadIdx.x; ls < ns; ls += FB_THREADS) op.row(s0 + ls, dot[ls], nacc);
  if (!Op::HAS_FIN) return;
  block_sum<NN>(nacc, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NN; ++k) s.npart[(int64_t)blockIdx.x * NN + k] = nacc[k];
  }
  if (!last_arrival(&s.tickets[0], gridDim.x)) return;
  double nsum[NN];
  block_sum_partials<NN>(s.npart, gridDim.x, nsum, red);
  if (threadIdx.x == 0) {
    if (s.bundle) {
#pragma unroll
      for (int k = 0; k < NN; ++k) s.bundle[k] = nsum[k];
    } else {
      op.fin(nsum);
    }
  }
}

// row sums of squares of CSR rows in stored (sample) order: the same
// sequential order as the reference's np.bincount (sparse.py:66-70)
__global__ void sp_rowsq_kernel(SpView A, double* out) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= A.rows) return;
  double s = 0.0;
  for (int64_t k = A.ptr[j]; k < A.ptr[j + 1]; ++k) {
    const double v = A.val[k];
    s += v * v;
  }
  out[j] = s;
}

// scatter a CSC matrix into the dense sample-major layout [n][ld]
__global__ void sp_densify_kernel(SpView csc, double* Zs, int64_t ld) {
  const int64_t i = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  if (i >= csc.rows) return;
  for (int64_t k = csc.ptr[i] + (threadIdx.x & 31); k < csc.ptr[i + 1]; k += 32)
    Zs[i * ld + csc.idx[k]] = csc.val[k];
}

}  // namespace gdwd
