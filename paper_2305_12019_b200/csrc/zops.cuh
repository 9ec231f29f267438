// Streaming fp64 matvec kernels over a row-major [rows x cols] matrix X
// whose rows are samples (X = Z~^T stored sample-major, i.e. the CSC values
// array of a fully dense Z~), plus a generic fused map-reduce.
//
//   zmv  : v = X^T t   (n -> d, "Z~ t";   reference scipy csc_matvec)
//   ztmv : v = X w     (d -> n, "Z~^T w"; reference scipy csr_matvec)
//   vmap : elementwise update + K fused sums
//
// Each kernel is a template over an Op functor that supplies the input
// vector on the fly (no materialised temporaries), consumes the result in an
// epilogue (the per-feature or per-sample update the reference does next),
// and contributes to fused reductions.  Reductions are deterministic
// (common.cuh); the final scalar logic runs in the last-arriving CTA.
//
// HBM layout: rows are padded to ld (multiple of 2 doubles, zero-filled) so
// every thread streams 16-byte double2 loads with L1::no_allocate.
#pragma once
#include <type_traits>

#include "common.cuh"

namespace gdwd {

struct MatView {
  const double* a;
  int64_t rows, cols, ld;
};

struct Scratch {
  double* part;       // per-segment vector partials
  double* npart;      // per-CTA n-sum partials
  double* tpart;      // per-tile d-sum partials
  unsigned* tickets;  // zero-initialised ticket counters
  double* bundle;     // sharded mode: local [R*d vector | n-sums] for the all-reduce (null: fused)
};

// ---------------------------------------------------------------------------
// zmv: grid (tiles, segs); CTA of 256 threads covers 512 columns (2 per
// thread) and a contiguous segment of rows.  Input t is staged in shared
// memory STAGE rows at a time.
// ---------------------------------------------------------------------------
constexpr int ZMV_THREADS = 256;
constexpr int ZMV_TILE = 2 * ZMV_THREADS;
constexpr int ZMV_STAGE = 512;

struct ZmvGeom {
  int tiles, segs;
  int64_t seg_len;
  int64_t ldp;  // leading dim of partial rows (>= cols, even)
};

// Ops may declare SQ = true to accumulate z*z (column sums of squares)
template <class Op, class = void>
struct op_sq : std::false_type {};
template <class Op>
struct op_sq<Op, std::void_t<decltype(Op::SQ)>> : std::integral_constant<bool, Op::SQ> {};

// (forcing >= 5 CTAs per SM spills the 8-row load batch: c3's Z~ [dr, z~tw] pass
// 291 -> 337 us; the kernel's natural 64 registers, 4 CTAs per SM, stand)
#ifndef ZMV_MINB
#define ZMV_MINB 1
#endif
template <class Op>
__global__ void __launch_bounds__(ZMV_THREADS, ZMV_MINB) zmv_kernel(Op op, MatView X, ZmvGeom g, Scratch s) {
  constexpr int R = Op::R, NN = Op::NN, ND = Op::ND;
  if (op.skip()) return;
  __shared__ double ts[R][ZMV_STAGE];
  __shared__ double red[(ZMV_THREADS / 32) * (NN > ND ? NN : ND)];
  const int tile = blockIdx.x, seg = blockIdx.y;
  const int64_t s0 = (int64_t)seg * g.seg_len;
  const int64_t s1 = (s0 + g.seg_len < X.rows) ? s0 + g.seg_len : X.rows;
  const int64_t j0 = (int64_t)tile * ZMV_TILE + 2 * threadIdx.x;
  const bool colok = j0 < X.cols;

  double acc[R][2];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r][0] = acc[r][1] = 0.0;
  double nacc[NN];
#pragma unroll
  for (int k = 0; k < NN; ++k) nacc[k] = 0.0;

  for (int64_t c0 = s0; c0 < s1; c0 += ZMV_STAGE) {
    const int cn = (int)((c0 + ZMV_STAGE < s1) ? ZMV_STAGE : s1 - c0);
    __syncthreads();
    for (int ii = threadIdx.x; ii < cn; ii += ZMV_THREADS) {
      double tv[R];
      double na[NN];
#pragma unroll
      for (int k = 0; k < NN; ++k) na[k] = 0.0;
      op.input(c0 + ii, tv, na);
#pragma unroll
      for (int r = 0; r < R; ++r) ts[r][ii] = tv[r];
#pragma unroll
      for (int k = 0; k < NN; ++k) nacc[k] += na[k];
    }
    __syncthreads();
    if (colok) {
      const double* p = X.a + c0 * X.ld + j0;
      int ii = 0;
      for (; ii + 8 <= cn; ii += 8) {  // 8 rows x 16 B in flight per thread
        double2 z[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) z[u] = ld_stream2(p + (int64_t)(ii + u) * X.ld);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const double t = op_sq<Op>::value ? 1.0 : ts[r][ii + u];
            acc[r][0] += z[u].x * (op_sq<Op>::value ? z[u].x : t);
            acc[r][1] += z[u].y * (op_sq<Op>::value ? z[u].y : t);
          }
        }
      }
      for (; ii < cn; ++ii) {
        const double2 z = ld_stream2(p + (int64_t)ii * X.ld);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double t = ts[r][ii];
          acc[r][0] += z.x * (op_sq<Op>::value ? z.x : t);
          acc[r][1] += z.y * (op_sq<Op>::value ? z.y : t);
        }
      }
    }
  }
  if (colok) {
#pragma unroll
    for (int r = 0; r < R; ++r)
      *reinterpret_cast<double2*>(s.part + ((int64_t)seg * R + r) * g.ldp + j0) = make_double2(acc[r][0], acc[r][1]);
  }
  if (tile == 0) {
    block_sum<NN>(nacc, red);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < NN; ++k) s.npart[(int64_t)seg * NN + k] = nacc[k];
    }
  }
  if (!last_arrival(&s.tickets[tile], gridDim.y)) return;

  if (s.bundle) {
    // sharded: publish the local Z~ t (this tile) and the n-sums, no epilogue
    if (colok) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double v0 = 0.0, v1 = 0.0;
        const int S = (int)gridDim.y;
        for (int sg0 = 0; sg0 < S; sg0 += 8) {  // segment order, 8 loads in flight
          double2 pv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            pv[u] = sg0 + u < S ? __ldcg(reinterpret_cast<const double2*>(s.part + ((int64_t)(sg0 + u) * R + r) * g.ldp + j0))
                                : make_double2(0.0, 0.0);
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (sg0 + u < S) {
              v0 += pv[u].x;
              v1 += pv[u].y;
            }
        }
        s.bundle[(int64_t)r * X.cols + j0] = v0;
        if (j0 + 1 < X.cols) s.bundle[(int64_t)r * X.cols + j0 + 1] = v1;
      }
    }
    if (!last_arrival(&s.tickets[gridDim.x], gridDim.x)) return;
    double nsum[NN];
    block_sum_partials<NN>(s.npart, gridDim.y, nsum, red);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < NN; ++k) s.bundle[(int64_t)R * X.cols + k] = nsum[k];
    }
    return;
  }

  double dacc[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) dacc[k] = 0.0;
  if (colok) {
    double v0[R], v1[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v0[r] = v1[r] = 0.0;
    // segment partials summed in segment order, 8 loads in flight
    const int S = (int)gridDim.y;
    for (int sg0 = 0; sg0 < S; sg0 += 8) {
      double2 pv[8][R];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r)
          pv[u][r] = sg0 + u < S ? __ldcg(reinterpret_cast<const double2*>(s.part + ((int64_t)(sg0 + u) * R + r) * g.ldp + j0))
                                 : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (sg0 + u < S) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            v0[r] += pv[u][r].x;
            v1[r] += pv[u][r].y;
          }
        }
    }
    op.epi(j0, v0, dacc);
    if (j0 + 1 < X.cols) op.epi(j0 + 1, v1, dacc);
  }
  block_sum<ND>(dacc, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < ND; ++k) s.tpart[(int64_t)tile * ND + k] = dacc[k];
  }
  if (!last_arrival(&s.tickets[gridDim.x], gridDim.x)) return;
  double nsum[NN], dsum[ND];
  block_sum_partials<NN>(s.npart, gridDim.y, nsum, red);
  block_sum_partials<ND>(s.tpart, gridDim.x, dsum, red);
  if (threadIdx.x == 0) op.fin(nsum, dsum);
}

// ---------------------------------------------------------------------------
// ztmv: grid (chunks, ranges).  Rows are split into `ranges` contiguous,
// evenly sized row ranges (one full wave of CTAs, sized from the occupancy
// calculator); the chunk of w (<= ZT_CW columns) is staged in shared memory
// and each warp computes row dots over the chunk.  With several chunks the
// last-arriving CTA of a row range sums the chunk partials in fixed order.
// The per-sample epilogue runs one sample per thread, ZT_BATCH rows at a time.
// ---------------------------------------------------------------------------
constexpr int ZT_THREADS = 256;
constexpr int ZT_CW = 4096;
constexpr int ZT_BATCH = 256;

struct ZtGeom {
  int chunks, ranges;
  int cw;  // chunk width (even)
};

// An Op with a heavy per-sample epilogue (the Newton prox) declares
// ZT_MINB: the minimum CTAs per SM the kernel is compiled for, so that the
// epilogue's registers (run once per CTA) do not cut the streaming loop's
// occupancy -- the rows' loads in flight are what the pass lives on.
#ifndef ZT_MINB_OVERRIDE
#define ZT_MINB_OVERRIDE 0
#endif
template <class Op, class = void>
struct ZtMinB {
  static constexpr int v = 1;
};
template <class Op>
struct ZtMinB<Op, decltype((void)Op::ZT_MINB)> {
  static constexpr int v = ZT_MINB_OVERRIDE ? ZT_MINB_OVERRIDE : Op::ZT_MINB;
};

template <class Op>
__global__ void __launch_bounds__(ZT_THREADS, ZtMinB<Op>::v) ztmv_kernel(Op op, MatView X, ZtGeom g, Scratch s) {
  constexpr int NN = Op::NN;
  if (op.skip()) return;
  extern __shared__ double zsm[];
  double* ws = zsm;           // cw
  double* sdot = zsm + g.cw;  // ZT_BATCH
  __shared__ double red[(ZT_THREADS / 32) * NN];
  const int c = blockIdx.x, rg = blockIdx.y;
  const int64_t c0 = (int64_t)c * g.cw;
  const int64_t clen = (c0 + g.cw < X.ld) ? g.cw : X.ld - c0;
  const int64_t i0 = X.rows * rg / g.ranges, i1 = X.rows * (rg + 1) / g.ranges;
  for (int jj = threadIdx.x; jj < clen; jj += ZT_THREADS) {
    const int64_t j = c0 + jj;
    ws[jj] = (j < X.cols) ? op.wval(j) : 0.0;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool single = gridDim.x == 1;
  double nacc[NN];
#pragma unroll
  for (int k = 0; k < NN; ++k) nacc[k] = 0.0;
  for (int64_t b0 = i0; b0 < i1; b0 += ZT_BATCH) {
    const int nb = (int)((b0 + ZT_BATCH < i1) ? ZT_BATCH : i1 - b0);
    __syncthreads();
    for (int li = warp; li < nb; li += ZT_THREADS / 32) {
      const double* p = X.a + (b0 + li) * X.ld + c0;
      double acc = 0.0;
      int64_t jj = 2 * lane;
      for (; jj + 7 * 64 < clen; jj += 8 * 64) {
        double2 z[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) z[u] = ld_stream2(p + jj + u * 64);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc += z[u].x * ws[jj + u * 64];
          acc += z[u].y * ws[jj + u * 64 + 1];
        }
      }
      for (; jj < clen; jj += 64) {
        const double2 z = ld_stream2(p + jj);
        acc += z.x * ws[jj];
        acc += z.y * ws[jj + 1];
      }
      double a1[1] = {acc};
      warp_sum<1>(a1);
      if (lane == 0) {
        if (single) sdot[li] = a1[0];
        else s.part[(int64_t)c * X.rows + b0 + li] = a1[0];
      }
    }
    if (single) {
      __syncthreads();
      if (threadIdx.x < nb) op.row(b0 + threadIdx.x, sdot[threadIdx.x], nacc);
    }
  }
  if (!single) {
    if (!last_arrival(&s.tickets[rg], gridDim.x)) return;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += ZT_THREADS) {
      double dot = 0.0;
      for (int cc = 0; cc < (int)gridDim.x; ++cc) dot += ld_cg(s.part + (int64_t)cc * X.rows + i);
      op.row(i, dot, nacc);
    }
  }
  if (!Op::HAS_FIN) return;
  block_sum<NN>(nacc, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NN; ++k) s.npart[(int64_t)rg * NN + k] = nacc[k];
  }
  // global ticket lives after the per-range slots
  if (!last_arrival(&s.tickets[single ? 0 : gridDim.y], gridDim.y)) return;
  double nsum[NN];
  block_sum_partials<NN>(s.npart, gridDim.y, nsum, red);
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
// vmap: grid-stride elementwise pass with NR fused sums.
// ---------------------------------------------------------------------------
constexpr int VM_THREADS = 256;

template <class Op>
__global__ void __launch_bounds__(VM_THREADS) vmap_kernel(Op op, int64_t len, Scratch s) {
  constexpr int NR = Op::NR;
  if (op.skip()) return;
  __shared__ double red[(VM_THREADS / 32) * NR];
  double acc[NR];
#pragma unroll
  for (int k = 0; k < NR; ++k) acc[k] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)VM_THREADS + threadIdx.x; i < len; i += (int64_t)gridDim.x * VM_THREADS)
    op.elem(i, acc);
  if (!Op::HAS_FIN) return;
  block_sum<NR>(acc, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NR; ++k) s.npart[(int64_t)blockIdx.x * NR + k] = acc[k];
  }
  if (!last_arrival(&s.tickets[0], gridDim.x)) return;
  double sum[NR];
  block_sum_partials<NR>(s.npart, gridDim.x, sum, red);
  if (threadIdx.x == 0) {
    if (s.bundle) {
#pragma unroll
      for (int k = 0; k < NR; ++k) s.bundle[k] = sum[k];
    } else {
      op.fin(sum);
    }
  }
}

// ---------------------------------------------------------------------------
// Sharded mode: after the all-reduce of the bundle, every rank runs the
// epilogue on identical data (so replicated d-space state stays identical).
// ---------------------------------------------------------------------------
template <class Op>
__global__ void __launch_bounds__(VM_THREADS) zmv_epi_kernel(Op op, const double* bundle, int64_t d, Scratch s) {
  constexpr int R = Op::R, NN = Op::NN, ND = Op::ND;
  if (op.skip()) return;
  __shared__ double red[(VM_THREADS / 32) * (NN > ND ? NN : ND)];
  double dacc[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) dacc[k] = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)VM_THREADS + threadIdx.x; j < d; j += (int64_t)gridDim.x * VM_THREADS) {
    double v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = bundle[(int64_t)r * d + j];
    op.epi(j, v, dacc);
  }
  block_sum<ND>(dacc, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < ND; ++k) s.tpart[(int64_t)blockIdx.x * ND + k] = dacc[k];
  }
  if (!last_arrival(&s.tickets[0], gridDim.x)) return;
  double dsum[ND];
  block_sum_partials<ND>(s.tpart, gridDim.x, dsum, red);
  if (threadIdx.x == 0) {
    double nsum[NN];
#pragma unroll
    for (int k = 0; k < NN; ++k) nsum[k] = bundle[(int64_t)R * d + k];
    op.fin(nsum, dsum);
  }
}

// fin of an n-reducing ztmv / vmap op with the all-reduced sums
template <class Op, int K>
__global__ void fin_kernel(Op op, const double* bundle) {
  if (op.skip()) return;
  double sum[K];
#pragma unroll
  for (int k = 0; k < K; ++k) sum[k] = bundle[k];
  op.fin(sum);
}

}  // namespace gdwd
