// FP64 tensor-core (DMMA) GEMM, Gram (SYRK) and the one-time dense
// Cholesky + explicit inverse used by the DIRECT and SMW regimes.
//
// Reference call sites replaced:
//   subsolvers.py:76   (Z Z^T).toarray()        -> gram_syrk(TN)  [DIRECT]
//   subsolvers.py:109  (Z^T Z).toarray()/mu^2   -> gram_syrk(NT)  [SMW]
//   cholesky.py:46     scipy.linalg.cholesky    -> chol_inverse (recursive
//                      blocked potrf+trtri on DMMA GEMMs)
//   cholesky.py:60-61  two solve_triangular     -> replaced per iteration by
//                      one GEMV with the explicit inverse (solver kernels).
//
// tcgen05 has no f64 kind; the FP64 tensor path on sm_100a is the legacy
// warp-level mma.sync m8n8k4 (SASS: DMMA.8x8x4).  Tiles: CTA 64x64, BK=16,
// 8 warps as 2(m) x 4(n), each warp 32x16 = 4x2 DMMA tiles; register-staged
// double buffering of the next K-slab; split-K over grid.z writes
// deterministic per-slice partials that a fixed-order reduction sums.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

#include "common.cuh"
#include "gram.cuh"

namespace gdwd {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, GT = 256;

// operand element (row r in [0,R), k) with strides (sr, sk)
struct Opnd {
  const double* p;
  int64_t sr, sk;
};

GDWD_DEV void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Load a BK x 64 slab of operand op (rows r0.., k0..) into registers.
// kfast: the k index varies fastest across threads (for operands whose k
// stride is 1) so that the warp's loads coalesce; otherwise r is fastest.
template <bool KFAST>
GDWD_DEV void load_slab(const Opnd& op, int64_t R, int64_t K, int64_t r0, int64_t k0, double (&reg)[4]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    int idx = threadIdx.x + e * GT;  // 0..1023
    int kk, rr;
    if (KFAST) { kk = idx & (BK - 1); rr = idx >> 4; }
    else       { rr = idx & 63;       kk = idx >> 6; }
    int64_t r = r0 + rr, k = k0 + kk;
    reg[e] = (r < R && k < K) ? op.p[r * op.sr + k * op.sk] : 0.0;
  }
}

// Shared tiles: operands whose k stride is 1 (KFAST) are kept [r][k] so the
// coalesced global rows store without bank conflicts; the others [k][r].
// Both are padded so the DMMA fragment reads (lanes g = lane/4 along r,
// t4 = lane%4 along k) are conflict-free.
constexpr int KPAD = 4, RPAD = 8;
constexpr int TILE_DOUBLES = (BM * (BK + KPAD) > BK * (BM + RPAD)) ? BM * (BK + KPAD) : BK * (BM + RPAD);

template <bool KFAST>
GDWD_DEV void store_slab(double* s, const double (&reg)[4]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    int idx = threadIdx.x + e * GT;
    int kk, rr;
    if (KFAST) { kk = idx & (BK - 1); rr = idx >> 4; s[rr * (BK + KPAD) + kk] = reg[e]; }
    else       { rr = idx & 63;       kk = idx >> 6; s[kk * (BM + RPAD) + rr] = reg[e]; }
  }
}

template <bool KFAST>
GDWD_DEV double frag(const double* s, int k, int r) {
  return KFAST ? s[r * (BK + KPAD) + k] : s[k * (BM + RPAD) + r];
}

// C-tile partial: Cw[m][n] = sum_{k in slice} A(m,k) B(n,k)
template <bool AK, bool BKF>
__global__ void __launch_bounds__(GT) gemm_dmma_kernel(Opnd A, Opnd B, int64_t M, int64_t N, int64_t K,
                                                       int64_t kslice, double* W, int64_t ldw,
                                                       int64_t wslice, bool upper_only, double alpha,
                                                       double beta, double* C, int64_t ldc, int tri = 0) {
  const int bm = blockIdx.y, bn = blockIdx.x;
  if (upper_only && bn < bm) return;
  if ((tri & GEMM_C_LOWER) && bn > bm) return;
  __shared__ double As[2][TILE_DOUBLES];
  __shared__ double Bs[2][TILE_DOUBLES];
  const int64_t m0 = (int64_t)bm * BM, n0 = (int64_t)bn * BN;
  int64_t kb = (int64_t)blockIdx.z * kslice;
  int64_t ke = (kb + kslice < K) ? kb + kslice : K;
  // k ranges where a triangular operand is zero for every row of the tile
  // (tile origins are multiples of BK, so kb stays slab-aligned)
  if ((tri & GEMM_B_KLE_N) && n0 + BN < ke) ke = n0 + BN;
  if ((tri & GEMM_A_KLE_M) && m0 + BM < ke) ke = m0 + BM;
  if ((tri & GEMM_B_KGE_N) && n0 > kb) kb = n0;
  if ((tri & GEMM_A_KGE_M) && m0 > kb) kb = m0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t4 = lane & 3;

  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double ra[4], rb[4];
  int buf = 0;
  if (kb < ke) {
    load_slab<AK>(A, M, ke, m0, kb, ra);
    load_slab<BKF>(B, N, ke, n0, kb, rb);
    store_slab<AK>(As[0], ra);
    store_slab<BKF>(Bs[0], rb);
  }
  __syncthreads();
  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
    const bool more = k0 + BK < ke;
    if (more) {
      load_slab<AK>(A, M, ke, m0, k0 + BK, ra);
      load_slab<BKF>(B, N, ke, n0, k0 + BK, rb);
    }
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = frag<AK>(As[buf], kk + t4, wm * 32 + i * 8 + g);
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = frag<BKF>(Bs[buf], kk + t4, wn * 16 + j * 8 + g);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
    if (more) {
      store_slab<AK>(As[buf ^ 1], ra);
      store_slab<BKF>(Bs[buf ^ 1], rb);
    }
    __syncthreads();
    buf ^= 1;
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + wm * 32 + i * 8 + g;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t nn = n0 + wn * 16 + j * 8 + t4 * 2 + h;
        if (nn >= N) continue;
        if (W) {
          W[(int64_t)blockIdx.z * wslice + m * ldw + nn] = acc[i][j][h];
        } else {
          double* cp = C + m * ldc + nn;
          *cp = (beta == 0.0) ? alpha * acc[i][j][h] : beta * *cp + alpha * acc[i][j][h];
        }
      }
    }
  }
}

// Sum split-K partials in slice order, symmetric fill from the upper
// triangle, C[i][j] = S[min][max] / div + (i==j ? shift : 0).
__global__ void syrk_finish_kernel(const double* W, int64_t ldw, int64_t wslice, int nslice, int64_t M,
                                   double div, double shift, double* C, int64_t ldc, bool accumulate) {
  const int64_t tot = M * M;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx / M, j = idx % M;
    int64_t a = i < j ? i : j, b = i < j ? j : i;
    double s = 0.0;
    for (int z = 0; z < nslice; ++z) s += W[z * wslice + a * ldw + b];
    double v = (div == 1.0) ? s : s / div;
    if (i == j) v += shift;
    C[i * ldc + j] = accumulate ? C[i * ldc + j] + v : v;
  }
}

// Dense factor + inverse of one diagonal block (m <= LEAF_MAX) in shared
// memory: A = L L^T (L lower), Linv = L^{-1}.  Upper parts are written as
// zeros.  Factor: 8-column panels; inverse: forward substitution, 8 columns
// per warp (below).  blockDim = 256.
constexpr int LEAF_MAX = 64;  // three (LEAF_MAX x LEAF_MAX+1) doubles in dynamic shared memory
constexpr size_t LEAF_SMEM = (size_t)3 * LEAF_MAX * (LEAF_MAX + 1) * sizeof(double);
__global__ void potrf_trtri_small(double* A, int64_t lda, double* Linv, int64_t ldl, int m, int* info,
                                  int64_t offset) {
  extern __shared__ double leaf_sm[];
  auto L = reinterpret_cast<double (*)[LEAF_MAX + 1]>(leaf_sm);
  auto Li = reinterpret_cast<double (*)[LEAF_MAX + 1]>(leaf_sm + LEAF_MAX * (LEAF_MAX + 1));
  auto Tm = reinterpret_cast<double (*)[LEAF_MAX + 1]>(leaf_sm + 2 * LEAF_MAX * (LEAF_MAX + 1));
  __shared__ int bad;
  const int t = threadIdx.x;
  if (t == 0) bad = 0;
  for (int idx = t; idx < LEAF_MAX * LEAF_MAX; idx += blockDim.x) {
    const int i = idx / LEAF_MAX, j = idx % LEAF_MAX;
    L[i][j] = (i < m && j <= i) ? A[i * lda + j] : 0.0;
    Li[i][j] = 0.0;
  }
  __syncthreads();
#ifdef LEAF_TIMING
  const long long lt0 = clock64();
#endif
  // Factor in 8-column panels.  Warp 0 factors a panel in registers (lane l
  // owns rows p0 + l and p0 + 32 + l; pivots and L[k][j] by shuffles, an
  // rsqrt per pivot (<= 1 ulp) instead of an IEEE sqrt and division, no
  // block barrier per column).  Look-ahead: in round p warp 0 applies panel
  // p's rank-8 update to panel p+1's columns and factors panel p+1 while the
  // other warps apply it to the columns beyond -- one block barrier per
  // panel, the bulk update off the critical path.  Updates subtract the 8
  // products in column order (the roundings of column-by-column rank-1
  // updates).
  auto factor_panel = [&](int p0) {  // warp 0
    const int pw = m - p0 < 8 ? m - p0 : 8;
    const int ra = p0 + t, rb = p0 + 32 + t;
    double Pa[8], Pb[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      Pa[c] = (ra < m && c < pw) ? L[ra][p0 + c] : 0.0;
      Pb[c] = (rb < m && c < pw) ? L[rb][p0 + c] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c < pw) {
        double d = __shfl_sync(0xffffffffu, Pa[c], c);
        if (!(d > 0.0)) {
          if (t == 0) bad = 1;
          d = 1.0;
        }
        const double rinv = rsqrt(d), r = d * rinv;
        const double sc = Pa[c] * rinv;  // selects, not branches: no divergence per column
        Pa[c] = t == c ? r : (t > c ? sc : Pa[c]);
        Pb[c] = Pb[c] * rinv;
#pragma unroll
        for (int c2 = c + 1; c2 < 8; ++c2) {
          const double lk = __shfl_sync(0xffffffffu, Pa[c], c2);  // L[p0+c2][p0+c]
          Pa[c2] = __fma_rn(-Pa[c], lk, Pa[c2]);
          Pb[c2] = __fma_rn(-Pb[c], lk, Pb[c2]);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c < pw) {
        if (ra < m && t >= c) L[ra][p0 + c] = Pa[c];
        if (rb < m) L[rb][p0 + c] = Pb[c];
      }
    }
  };
  // panel (p0, pw) applied to columns [kb, ke): worker u of nthr owns column
  // k = kb + u % ncol (its 8 multipliers in registers) and rows
  // i = kb + u / ncol + 4 s >= k
  auto update_cols = [&](int p0, int pw, int kb, int ke, int u, int nthr) {
    const int ncol = ke - kb;
    for (int idx = u; idx < 4 * ncol; idx += nthr) {
      const int kk = idx % ncol, ph = idx / ncol, k = kb + kk;
      double lk[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) lk[c] = c < pw ? L[k][p0 + c] : 0.0;
#pragma unroll 4
      for (int ii = ph; ii < m - kb; ii += 4) {
        if (ii >= kk) {
          const int i = kb + ii;
          double acc = L[i][k];
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (c < pw) acc = __fma_rn(-L[i][p0 + c], lk[c], acc);
          L[i][k] = acc;
        }
      }
    }
  };
  if (t < 32) factor_panel(0);
  __syncthreads();
  for (int p0 = 0; p0 + 8 < m; p0 += 8) {  // panel p0 is factored; q0 = p0 + 8 < m
    const int q0 = p0 + 8;
    const int q1 = q0 + 8 < m ? q0 + 8 : m;
    if (t < 32) {
      update_cols(p0, 8, q0, q1, t, 32);
      __syncwarp();
      factor_panel(q0);
    } else if (q1 < m) {
      update_cols(p0, 8, q1, m, t - 32, blockDim.x - 32);
    }
    __syncthreads();
  }
#ifdef LEAF_TIMING
  const long long lt1 = clock64();
#endif
  // Inverse by forward substitution, L X = I: each warp solves 8 columns
  // c0 .. c0+7 (lane l holds rows l and l + 32 of each); step j turns b_j
  // into x_j = b_j / L_jj (one shuffle per column) and subtracts
  // L[i][j] x_j from the rows below -- no block barrier, m - c0 steps.
  if (t < m) Tm[0][t] = 1.0 / L[t][t];
  __syncthreads();
  {
    // column blocks paired long/short per SM sub-partition (warps w, w + 4)
    const int w = t >> 5, l = t & 31, c0 = 8 * (w < 4 ? w : 11 - w);
    if (c0 < m) {
      double Xa[8], Xb[8];
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        Xa[cc] = l == c0 + cc ? 1.0 : 0.0;
        Xb[cc] = l + 32 == c0 + cc ? 1.0 : 0.0;
      }
      // rows <= j have la = lb = 0 (x - 0 * y == x): selects only, no branch
      for (int j = c0; j < (m < 32 ? m : 32); ++j) {
        const double dj = Tm[0][j];
        const double la = l > j ? L[l][j] : 0.0;
        const double lb = l + 32 < m ? L[l + 32][j] : 0.0;
        const bool own = l == j;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const double xj = __shfl_sync(0xffffffffu, Xa[cc], j) * dj;
          const double ua = __fma_rn(-la, xj, Xa[cc]);
          Xb[cc] = __fma_rn(-lb, xj, Xb[cc]);
          Xa[cc] = own ? xj : ua;
        }
      }
      for (int j = c0 > 32 ? c0 : 32; j < m; ++j) {  // rows < 32 are final
        const double dj = Tm[0][j];
        const double lb = l + 32 > j && l + 32 < m ? L[l + 32][j] : 0.0;
        const bool own = l == j - 32;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const double xj = __shfl_sync(0xffffffffu, Xb[cc], j - 32) * dj;
          const double ub = __fma_rn(-lb, xj, Xb[cc]);
          Xb[cc] = own ? xj : ub;
        }
      }
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        if (c0 + cc < m) {
          if (l < m) Li[l][c0 + cc] = Xa[cc];
          if (l + 32 < m) Li[l + 32][c0 + cc] = Xb[cc];
        }
      }
    }
  }
  __syncthreads();
#ifdef LEAF_TIMING
  if (t == 0 && offset == 0) printf("[leaf] m=%d factor %lld inverse %lld cycles\n", m, lt1 - lt0, clock64() - lt1);
#endif
  for (int idx = t; idx < m * m; idx += blockDim.x) {
    const int i = idx / m, j = idx % m;
    A[i * lda + j] = (j <= i) ? L[i][j] : 0.0;
    Linv[i * ldl + j] = (j <= i) ? Li[i][j] : 0.0;
  }
  if (t == 0 && bad && info) atomicCAS(info, 0, (int)offset + 1);
}

__global__ void zero_kernel(double* p, int64_t rows, int64_t cols, int64_t ld) {
  const int64_t tot = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
       idx += (int64_t)gridDim.x * blockDim.x)
    p[(idx / cols) * ld + idx % cols] = 0.0;
}

__global__ void copy2d_kernel(const double* s, int64_t lds, double* d, int64_t ldd, int64_t rows,
                              int64_t cols) {
  const int64_t tot = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
       idx += (int64_t)gridDim.x * blockDim.x)
    d[(idx / cols) * ldd + idx % cols] = s[(idx / cols) * lds + idx % cols];
}

int grid_for(int64_t tot) {
  int64_t b = (tot + 255) / 256;
  return (int)(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

}  // namespace

// C (M x N) = alpha * sum_k A(m,k) B(n,k) + beta * C.
// A(m,k) = a[m*sam + k*sak]; B(n,k) = b[n*sbn + k*sbk].
cudaError_t gemm_f64(const double* a, int64_t sam, int64_t sak, const double* b, int64_t sbn,
                     int64_t sbk, int64_t M, int64_t N, int64_t K, double alpha, double beta, double* C,
                     int64_t ldc, cudaStream_t st, int tri) {
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), 1);
  Opnd A{a, sam, sak}, B{b, sbn, sbk};
  const bool ak = (sak == 1), bk = (sbk == 1);
  if (ak && bk)
    gemm_dmma_kernel<true, true><<<grid, GT, 0, st>>>(A, B, M, N, K, K, nullptr, 0, 0, false, alpha, beta, C, ldc, tri);
  else if (ak)
    gemm_dmma_kernel<true, false><<<grid, GT, 0, st>>>(A, B, M, N, K, K, nullptr, 0, 0, false, alpha, beta, C, ldc, tri);
  else if (bk)
    gemm_dmma_kernel<false, true><<<grid, GT, 0, st>>>(A, B, M, N, K, K, nullptr, 0, 0, false, alpha, beta, C, ldc, tri);
  else
    gemm_dmma_kernel<false, false><<<grid, GT, 0, st>>>(A, B, M, N, K, K, nullptr, 0, 0, false, alpha, beta, C, ldc,
                                                        tri);
  return cudaGetLastError();
}

int64_t gram_workspace_doubles(int64_t M, int64_t K) {
  int nslice = gram_slices(M, K);
  return (int64_t)nslice * M * M;
}

int gram_slices(int64_t M, int64_t K) {
  const int64_t tiles = ((M + BM - 1) / BM) * ((M + BM - 1) / BM + 1) / 2;
  int64_t s = (148 * 3 + tiles - 1) / tiles;  // aim for >= 3 CTAs per SM
  int64_t kmax = (K + 255) / 256;             // keep >= 256 K per slice
  if (s > kmax) s = kmax;
  if (s > 64) s = 64;
  if (s < 1) s = 1;
  return (int)s;
}

// Symmetric Gram of the rows/columns of a row-major [R x L] matrix Zs:
//   trans_k = true : C (L x L) = Zs^T Zs   (sum over rows,   "DIRECT": Z Z^T)
//   trans_k = false: C (R x R) = Zs Zs^T   (sum over columns, "SMW":   Z^T Z)
// then C = C / div + shift * I.  W: workspace of gram_workspace_doubles.
cudaError_t gram_syrk(const double* Zs, int64_t R, int64_t Lc, int64_t ldz, bool sum_over_rows, double div,
                      double shift, double* C, int64_t ldc, double* W, cudaStream_t st, bool accumulate) {
  const int64_t M = sum_over_rows ? Lc : R;
  const int64_t K = sum_over_rows ? R : Lc;
  const int ns = gram_slices(M, K);
  int64_t kslice = (K + ns - 1) / ns;
  kslice = (kslice + BK - 1) / BK * BK;
  dim3 grid((unsigned)((M + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)ns);
  if (sum_over_rows) {
    // A(m,k) = Zs[k][m]: m stride 1, k stride ldz (r fastest)
    Opnd A{Zs, 1, ldz};
    gemm_dmma_kernel<false, false><<<grid, GT, 0, st>>>(A, A, M, M, K, kslice, W, M, M * M, true, 1.0, 0.0,
                                                        nullptr, 0);
  } else {
    Opnd A{Zs, ldz, 1};
    gemm_dmma_kernel<true, true><<<grid, GT, 0, st>>>(A, A, M, M, K, kslice, W, M, M * M, true, 1.0, 0.0,
                                                      nullptr, 0);
  }
  syrk_finish_kernel<<<grid_for(M * M), 256, 0, st>>>(W, M, M * M, ns, M, div, shift, C, ldc, accumulate);
  return cudaGetLastError();
}

namespace {

#ifndef CHOL_LEAF
#define CHOL_LEAF 64  // diagonal blocks factored by one CTA; the recursion's critical path
#endif
static_assert(CHOL_LEAF <= LEAF_MAX, "leaf larger than potrf_trtri_small's shared arrays");
// Recursive blocked Cholesky + triangular inverse (lower):
//   A (m x m, ld) is overwritten by L; Li (ld) receives L^{-1}; T scratch.
// Side stream of the recursion (per thread and device): L21 L11^{-1}, the
// first factor of the off-diagonal inverse block, does not depend on the
// lower-right factorisation and runs beside it.
struct CholAux {
  cudaStream_t side = nullptr;
  int dev = -1;
};
static cudaStream_t chol_side_stream() {
  static thread_local CholAux aux[8];
  int dev = 0;
  cudaGetDevice(&dev);
  CholAux& a = aux[dev & 7];
  if (!a.side || a.dev != dev) {
    cudaStreamCreateWithFlags(&a.side, cudaStreamNonBlocking);
    a.dev = dev;
  }
  return a.side;
}

// Recursive blocked Cholesky + triangular inverse (lower):
//   Li (ld) receives L^{-1}; A's diagonal leaf blocks receive L, its other
//   blocks are scratch afterwards; T (m x m, ld) holds L's off-diagonal
//   blocks in place (block (2,1) of this level at T + m1 ld, the lower-right
//   recursion in T's lower-right block), so no copy back is needed.
cudaError_t chol_rec(double* A, double* Li, double* T, int64_t ld, int64_t m, int64_t off, int* info,
                     cudaStream_t st, cudaStream_t side, std::vector<cudaEvent_t>& evs) {
  if (m <= CHOL_LEAF) {
    static unsigned long long attr = 0;
    if (once_per_device(attr))
      cudaFuncSetAttribute(potrf_trtri_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LEAF_SMEM);
    potrf_trtri_small<<<1, 256, LEAF_SMEM, st>>>(A, ld, Li, ld, (int)m, info, off);
    return cudaGetLastError();
  }
  int64_t m1 = ((m / 2) + CHOL_LEAF - 1) / CHOL_LEAF * CHOL_LEAF;
  if (m1 >= m) m1 = m - CHOL_LEAF;
  const int64_t m2 = m - m1;
  double* A11 = A;
  double* A21 = A + m1 * ld;
  double* A22 = A + m1 * ld + m1;
  double* L11i = Li;
  double* L21i = Li + m1 * ld;
  double* L22i = Li + m1 * ld + m1;
  double* L21 = T + m1 * ld;
  cudaError_t e = chol_rec(A11, L11i, T, ld, m1, off, info, st, side, evs);
  if (e != cudaSuccess) return e;
  // L21 = A21 * L11i^T   (m2 x m1): A(i,k)=A21[i][k], B(j,k)=L11i[j][k]
  e = gemm_f64(A21, ld, 1, L11i, ld, 1, m2, m1, m1, 1.0, 0.0, L21, ld, st, GEMM_B_KLE_N);
  if (e != cudaSuccess) return e;
  // A22 -= L21 L21^T (lower tiles: the recursion reads only A22's lower triangle)
  e = gemm_f64(L21, ld, 1, L21, ld, 1, m2, m2, m1, -1.0, 1.0, A22, ld, st, GEMM_C_LOWER);
  if (e != cudaSuccess) return e;
  // beside the lower-right recursion: A21 <- L21 * L11i (A(i,k)=L21[i][k], B(j,k)=L11i[k][j])
  cudaEvent_t ev_fork, ev_join;
  cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming);
  evs.push_back(ev_fork);
  evs.push_back(ev_join);
  if ((e = cudaEventRecord(ev_fork, st)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(side, ev_fork, 0)) != cudaSuccess) return e;
  e = gemm_f64(L21, ld, 1, L11i, 1, ld, m2, m1, m1, 1.0, 0.0, A21, ld, side, GEMM_B_KGE_N);
  if (e != cudaSuccess) return e;
  if ((e = cudaEventRecord(ev_join, side)) != cudaSuccess) return e;
  e = chol_rec(A22, L22i, T + m1 * ld + m1, ld, m2, off + m1, info, st, side, evs);
  if (e != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(st, ev_join, 0)) != cudaSuccess) return e;
  // L21i = -L22i * (L21 L11i) : A(i,k)=L22i[i][k], B(j,k)=A21[k][j]
  e = gemm_f64(L22i, ld, 1, A21, 1, ld, m2, m1, m2, -1.0, 0.0, L21i, ld, st, GEMM_A_KLE_M);
  return e;
}

}  // namespace

// In place: A (m x m SPD, row-major ld) -> A^{-1}.  Li, T: m x m scratch
// (ld).  *info (device int) receives 1 + index of the first non-positive
// pivot block, 0 on success.  Returns launch errors only.
cudaError_t chol_inverse(double* A, double* Li, double* T, int64_t ld, int64_t m, int* info, cudaStream_t st) {
  zero_kernel<<<grid_for(m * m), 256, 0, st>>>(Li, m, m, ld);
  std::vector<cudaEvent_t> evs;
  cudaError_t e = chol_rec(A, Li, T, ld, m, 0, info, st, chol_side_stream(), evs);
  for (cudaEvent_t ev : evs) cudaEventDestroy(ev);  // released once the recorded work completes
  if (e != cudaSuccess) return e;
  // A^{-1} = Li^T Li : C(i,j) = sum_k Li[k][i] Li[k][j] -- symmetric: upper
  // tiles on the DMMA SYRK path, mirrored (T is the workspace)
  if (gram_slices(m, m) == 1) return gram_syrk(Li, m, m, ld, true, 1.0, 0.0, A, ld, T, st);
  return gemm_f64(Li, 1, ld, Li, 1, ld, m, m, m, 1.0, 0.0, A, ld, st, GEMM_A_KGE_M | GEMM_B_KGE_N);
}

}  // namespace gdwd
