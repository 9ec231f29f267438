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
// warp-level mma.sync m8n8k4 (SASS: DMMA.8x8x4).  Two kernels:
//   gram_tile_kernel  the Gram-shaped products (both operands with the same
//                     fast axis): 64x128 CTA tile, 4 warps of 64x32, 16-byte
//                     cp.async into a 3-stage ring, two CTAs per SM
//   gemm_dmma_kernel  general strides and triangular-operand skips (the
//                     Cholesky recursion and chain): CTA 64x64, BK=16, 8
//                     warps as 2(m) x 4(n), each warp 32x16 = 4x2 DMMA tiles,
//                     register-staged double buffering of the next K-slab
// Split-K over grid.z writes deterministic per-slice partials that a
// fixed-order reduction sums.  The row-block (bordered) forms at the end of
// the file advance the Gram, the Cholesky factor and the inverse one block
// of samples at a time, under the host-to-device copy (gdwd.cu).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

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
    const int64_t i = idx / M, j = idx % M;
    if (j < i) continue;  // each upper entry is summed once and stored to both halves
    double s = 0.0;
    for (int z = 0; z < nslice; ++z) s += W[z * wslice + i * ldw + j];
    double v = (div == 1.0) ? s : s / div;
    if (i == j) v += shift;
    C[i * ldc + j] = accumulate ? C[i * ldc + j] + v : v;
    if (i != j) C[j * ldc + i] = accumulate ? C[j * ldc + i] + v : v;
  }
}

// ---------------------------------------------------------------------------
// Gram-shaped products (both operands with the same fast axis, 16-byte
// aligned rows): 64 x 128 CTA tile, 4 warps side by side, each warp
// 64 x 32 = 8 x 4 DMMA tiles (32 DMMAs per 12 fragment loads), operands
// brought global -> shared by 16-byte cp.async in a 3-stage ring (no register
// staging).  Two CTAs per SM (192 registers x 128 threads, 90 KB of shared
// memory each): one CTA's barrier / fragment-load bubble at a K step is
// covered by the other's DMMAs.  K tails and rows beyond M / N are
// zero-filled by the copy's source size.
// ---------------------------------------------------------------------------
constexpr int TMA = 64, TNB = 128, TK = 16, TSTAGES = 3, TT = 128;
constexpr int T_KSTRIDE = TK + 4;    // k-fast tiles [r][k]: fragment reads conflict-free
constexpr int T_RSTRIDE_A = TMA + 8;  // r-fast tiles [k][r]
constexpr int T_RSTRIDE_B = TNB + 8;
constexpr int T_TILE_A = (TMA * T_KSTRIDE > TK * T_RSTRIDE_A) ? TMA * T_KSTRIDE : TK * T_RSTRIDE_A;
constexpr int T_TILE_B = (TNB * T_KSTRIDE > TK * T_RSTRIDE_B) ? TNB * T_KSTRIDE : TK * T_RSTRIDE_B;
constexpr int T_STAGE = T_TILE_A + T_TILE_B;
constexpr size_t T_SMEM = (size_t)TSTAGES * T_STAGE * sizeof(double);

GDWD_DEV void cp_async16(double* smem, const double* g, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(g), "r"(src_bytes) : "memory");
}

// one ROWS x 16 operand tile in chunks of two doubles
template <bool KF, int ROWS>
GDWD_DEV void tile_load(double* sm, const Opnd& op, int64_t R, int64_t r0, int64_t k0, int64_t ke) {
  constexpr int RSTRIDE = ROWS + 8;
#pragma unroll
  for (int e = 0; e < ROWS * 8 / TT; ++e) {
    const int c = threadIdx.x + e * TT;
    if (KF) {
      const int rr = c >> 3, kc = (c & 7) * 2;
      const int64_t r = r0 + rr, k = k0 + kc;
      const int v = (r < R && k < ke) ? (ke - k >= 2 ? 2 : 1) : 0;
      cp_async16(sm + rr * T_KSTRIDE + kc, op.p + (v ? r * op.sr + k : 0), v * 8);
    } else {
      const int kk = c / (ROWS / 2), rc = (c % (ROWS / 2)) * 2;
      const int64_t r = r0 + rc, k = k0 + kk;
      const int v = (k < ke && r < R) ? (R - r >= 2 ? 2 : 1) : 0;
      cp_async16(sm + kk * RSTRIDE + rc, op.p + (v ? k * op.sk + r : 0), v * 8);
    }
  }
}

template <bool KF>
__global__ void __launch_bounds__(TT, 2) gram_tile_kernel(Opnd A, Opnd B, int64_t M, int64_t N, int64_t K,
                                                          int64_t kslice, double* W, int64_t ldw, int64_t wslice,
                                                          bool upper_only, double alpha, double beta, double* C,
                                                          int64_t ldc) {
  const int bm = blockIdx.y, bn = blockIdx.x;
  const int64_t m0 = (int64_t)bm * TMA, n0 = (int64_t)bn * TNB;
  if (upper_only && n0 + TNB <= m0) return;  // every entry below the diagonal
  extern __shared__ __align__(16) double tsm[];
  const int64_t kb = (int64_t)blockIdx.z * kslice;
  const int64_t ke = (kb + kslice < K) ? kb + kslice : K;
  const int nk = kb < ke ? (int)((ke - kb + TK - 1) / TK) : 0;
  const int lane = threadIdx.x & 31, wn = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < TSTAGES - 1; ++s) {
    if (s < nk) {
      tile_load<KF, TMA>(tsm + (size_t)s * T_STAGE, A, M, m0, kb + (int64_t)s * TK, ke);
      tile_load<KF, TNB>(tsm + (size_t)s * T_STAGE + T_TILE_A, B, N, n0, kb + (int64_t)s * TK, ke);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int it = 0; it < nk; ++it) {
    asm volatile("cp.async.wait_group %0;" ::"n"(TSTAGES - 2) : "memory");
    __syncthreads();  // stage `it` landed for everyone; stage it-1 is free again
    {
      const int nx = it + TSTAGES - 1;
      if (nx < nk) {
        double* st = tsm + (size_t)(nx % TSTAGES) * T_STAGE;
        tile_load<KF, TMA>(st, A, M, m0, kb + (int64_t)nx * TK, ke);
        tile_load<KF, TNB>(st + T_TILE_A, B, N, n0, kb + (int64_t)nx * TK, ke);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const double* as = tsm + (size_t)(it % TSTAGES) * T_STAGE;
    const double* bs = as + T_TILE_A;
#pragma unroll
    for (int kk = 0; kk < TK; kk += 4) {
      double af[8], bf[4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        af[i] = KF ? as[(i * 8 + g) * T_KSTRIDE + kk + t4] : as[(kk + t4) * T_RSTRIDE_A + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        bf[j] = KF ? bs[(wn * 32 + j * 8 + g) * T_KSTRIDE + kk + t4] : bs[(kk + t4) * T_RSTRIDE_B + wn * 32 + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t m = m0 + i * 8 + g;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t nn = n0 + wn * 32 + j * 8 + t4 * 2 + h;
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

// the tiled kernel needs 16-byte aligned rows along the fast axis
static bool tile_ok(const double* p, int64_t ld) { return ((uintptr_t)p & 15) == 0 && (ld & 1) == 0; }

template <bool KF>
static cudaError_t launch_tile(Opnd A, Opnd B, int64_t M, int64_t N, int64_t K, int64_t kslice, int ns, double* W,
                               int64_t ldw, int64_t wslice, bool upper_only, cudaStream_t st) {
  static unsigned long long attr = 0;
  if (once_per_device(attr))
    cudaFuncSetAttribute(gram_tile_kernel<KF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T_SMEM);
  dim3 grid((unsigned)((N + TNB - 1) / TNB), (unsigned)((M + TMA - 1) / TMA), (unsigned)ns);
  gram_tile_kernel<KF><<<grid, TT, T_SMEM, st>>>(A, B, M, N, K, kslice, W, ldw, wslice, upper_only, 1.0, 0.0, nullptr,
                                                 0);
  return cudaGetLastError();
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

namespace {
// C = beta C + alpha sum_z W[z] (slice order), tiles above the diagonal
// untouched when only the lower ones were computed
__global__ void splitk_finish_kernel(const double* W, int64_t wslice, int nslice, int64_t M, int64_t N, double alpha,
                                     double beta, double* C, int64_t ldc, int lower) {
  const int64_t tot = M * N;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / N, j = idx % N;
    if (lower && j / BN > i / BM) continue;
    double s = 0.0;
    for (int z = 0; z < nslice; ++z) s += W[z * wslice + idx];
    double* cp = C + i * ldc + j;
    *cp = (beta == 0.0) ? alpha * s : beta * *cp + alpha * s;
  }
}
}  // namespace

// gemm_f64 for few output tiles and a long K (the bordered chain's products):
// K is split over grid.z so that the GPU fills, partials go to W (capacity
// wcap doubles) and are summed in slice order.  Falls back to one slice.
cudaError_t gemm_f64_splitk(const double* a, int64_t sam, int64_t sak, const double* b, int64_t sbn, int64_t sbk,
                            int64_t M, int64_t N, int64_t K, double alpha, double beta, double* C, int64_t ldc,
                            cudaStream_t st, int tri, double* W, int64_t wcap) {
  const int64_t tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
  const int64_t tiles = (tri & GEMM_C_LOWER) ? tm * (tm + 1) / 2 : tm * tn;
  int64_t ns = (148 * 2 + tiles - 1) / tiles;
  const int64_t kmax = (K + 63) / 64;  // >= 64 of K per slice
  if (ns > kmax) ns = kmax;
  if (ns > 32) ns = 32;
  if (W == nullptr || ns * M * N > wcap) ns = wcap / (M * N);
  if (ns <= 1 || W == nullptr) return gemm_f64(a, sam, sak, b, sbn, sbk, M, N, K, alpha, beta, C, ldc, st, tri);
  int64_t kslice = (K + ns - 1) / ns;
  kslice = (kslice + BK - 1) / BK * BK;
  ns = (K + kslice - 1) / kslice;
  dim3 grid((unsigned)tn, (unsigned)tm, (unsigned)ns);
  Opnd A{a, sam, sak}, B{b, sbn, sbk};
  const bool ak = (sak == 1), bk = (sbk == 1);
  if (ak && bk)
    gemm_dmma_kernel<true, true><<<grid, GT, 0, st>>>(A, B, M, N, K, kslice, W, N, M * N, false, 1.0, 0.0, nullptr, 0, tri);
  else if (ak)
    gemm_dmma_kernel<true, false><<<grid, GT, 0, st>>>(A, B, M, N, K, kslice, W, N, M * N, false, 1.0, 0.0, nullptr, 0, tri);
  else if (bk)
    gemm_dmma_kernel<false, true><<<grid, GT, 0, st>>>(A, B, M, N, K, kslice, W, N, M * N, false, 1.0, 0.0, nullptr, 0, tri);
  else
    gemm_dmma_kernel<false, false><<<grid, GT, 0, st>>>(A, B, M, N, K, kslice, W, N, M * N, false, 1.0, 0.0, nullptr, 0,
                                                        tri);
  splitk_finish_kernel<<<grid_for(M * N), 256, 0, st>>>(W, M * N, (int)ns, M, N, alpha, beta, C, ldc,
                                                        (tri & GEMM_C_LOWER) != 0);
  return cudaGetLastError();
}

int64_t gram_workspace_doubles(int64_t M, int64_t K) {
  int nslice = gram_slices(M, K);
  return (int64_t)nslice * M * M;
}

// Split-K factor for `tiles` output tiles: the kernel is resident at 2 CTAs
// per SM (120 registers x 256 threads), i.e. 296 at once; pick the slice
// count whose CTA total fills whole waves best (>= kmin of K per slice, at
// least ~2 waves when K allows so the tail wave is a small share), smallest
// such count on ties.
static int pick_slices(int64_t tiles, int64_t K, int64_t kmin, int smax, int64_t slots = 2 * 148) {
  int64_t kmax = (K + kmin - 1) / kmin;
  if (kmax > smax) kmax = smax;
  if (kmax < 1) kmax = 1;
  int best = 1;
  double best_eff = -1.0;
  for (int64_t s = 1; s <= kmax; ++s) {
    const int64_t ctas = tiles * s, waves = (ctas + slots - 1) / slots;
    double eff = (double)ctas / (double)(waves * slots);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = (int)s;
    }
  }
  return best;
}

int gram_slices(int64_t M, int64_t K) {  // 64 x 128 tiles on or above the diagonal, two CTAs per SM
  int64_t tiles = 0;
  for (int64_t m0 = 0; m0 < M; m0 += TMA) tiles += (M + TNB - 1) / TNB - m0 / TNB;
  return pick_slices(tiles, K, 512, 32, 2 * 148);
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
  if (tile_ok(Zs, ldz)) {
    cudaError_t e = sum_over_rows
                        ? launch_tile<false>(Opnd{Zs, 1, ldz}, Opnd{Zs, 1, ldz}, M, M, K, kslice, ns, W, M, M * M, true, st)
                        : launch_tile<true>(Opnd{Zs, ldz, 1}, Opnd{Zs, ldz, 1}, M, M, K, kslice, ns, W, M, M * M, true, st);
    if (e != cudaSuccess) return e;
    syrk_finish_kernel<<<grid_for(M * M), 256, 0, st>>>(W, M, M * M, ns, M, div, shift, C, ldc, accumulate);
    return cudaGetLastError();
  }
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

// ---------------------------------------------------------------------------
// Row-block (bordered) forms: the n x n sample-space Gram, its Cholesky
// factor and the explicit inverse advance one block of samples at a time, so
// they run while the remaining samples are still being copied to the device
// (gdwd.cu: upload_dense_pipelined).  Same quantities as gram_syrk +
// chol_inverse (subsolvers.py:109, cholesky.py:46,60-61), other association.
// ---------------------------------------------------------------------------
namespace {

int rowblock_slices(int64_t mb, int64_t r1, int64_t K) {
  const int64_t tiles = ((mb + TMA - 1) / TMA) * ((r1 + TNB - 1) / TNB);
  // Default: whole waves of many short slices (c2's last block: 37 slices of
  // 544, four exact waves), so Gram CTAs retire every ~70 us and the factor
  // chain's launches (which cannot co-reside with two of them: registers)
  // find a slot quickly.  Measured alternatives at c2, end to end: >= 1024 of
  // K per slice (Gram kernel faster, chain starved) 8.15-8.24 ms; one partial
  // wave of GDWD_RB_CTAS = 288 / 264 / 232 / 200 CTAs (some SMs left with one
  // Gram CTA for the chain) 8.06-8.10 / 8.10-8.24 / 8.15-8.18 / 8.33-8.38 ms;
  // this default 8.02-8.08 ms.
  static const int64_t cap = [] {
    const char* e = getenv("GDWD_RB_CTAS");
    return (int64_t)(e ? atoi(e) : 0);
  }();
  if (cap <= 0) return pick_slices(tiles, K, 256, 64, 2 * 148);  // whole waves of short slices
  int64_t s = cap / tiles;
  const int64_t kmax = (K + 255) / 256;
  if (s > kmax) s = kmax;
  if (s > 64) s = 64;
  if (s < 1) s = 1;
  return (int)s;
}

// Sum the split-K partials of block rows r0..r1 in slice order; the diagonal
// block takes (min, max) so K stays exactly symmetric.  Writes K's rows and
// their mirror, and G = K / mu2 + I on the rows (columns < r1).
__global__ void rowblock_finish_kernel(const double* W, int64_t wslice, int nslice, int64_t r0, int64_t r1,
                                       double* K, int64_t ldk, double* G, int64_t ldg, double mu2) {
  const int64_t mb = r1 - r0, tot = mb * r1;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / r1, j = idx % r1;
    int64_t a = i, b = j;
    if (j >= r0 && j - r0 < i) { a = j - r0; b = r0 + i; }
    double s = 0.0;
    for (int z = 0; z < nslice; ++z) s += W[z * wslice + a * r1 + b];
    K[(r0 + i) * ldk + j] = s;
    if (j < r0) K[j * ldk + r0 + i] = s;
    const double g = (mu2 == 1.0) ? s : s / mu2;
    G[(r0 + i) * ldg + j] = (j == r0 + i) ? g + 1.0 : g;
  }
}

__global__ void mirror_lower_kernel(double* A, int64_t ld, int64_t m) {
  const int64_t tot = m * m;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / m, j = idx % m;
    if (j > i) A[i * ld + j] = A[j * ld + i];
  }
}

}  // namespace

int64_t gram_rowblock_workspace(int64_t n, int64_t d, int64_t mb) {
  int64_t best = 0;
  for (int64_t r0 = 0; r0 < n; r0 += mb) {
    const int64_t r1 = r0 + mb < n ? r0 + mb : n;
    const int64_t need = (int64_t)rowblock_slices(r1 - r0, r1, d) * (r1 - r0) * r1;
    if (need > best) best = need;
  }
  return best;
}

// K[r0:r1, 0:r1] = Zs[r0:r1] Zs[0:r1]^T over the d feature columns (row-major
// samples, ldz), mirrored into K[0:r0, r0:r1]; G rows = K / mu2 + I.
cudaError_t gram_rowblock(const double* Zs, int64_t ldz, int64_t d, int64_t r0, int64_t r1, double* K, int64_t ldk,
                          double* G, int64_t ldg, double mu2, double* W, cudaStream_t st) {
  const int64_t mb = r1 - r0;
  const int ns = rowblock_slices(mb, r1, d);
  int64_t kslice = (d + ns - 1) / ns;
  kslice = (kslice + BK - 1) / BK * BK;
  Opnd A{Zs + r0 * ldz, ldz, 1}, B{Zs, ldz, 1};
  if (tile_ok(Zs, ldz)) {
    cudaError_t e = launch_tile<true>(A, B, mb, r1, d, kslice, ns, W, r1, mb * r1, false, st);
    if (e != cudaSuccess) return e;
  } else {
    dim3 grid((unsigned)((r1 + BN - 1) / BN), (unsigned)((mb + BM - 1) / BM), (unsigned)ns);
    gemm_dmma_kernel<true, true><<<grid, GT, 0, st>>>(A, B, mb, r1, d, kslice, W, r1, mb * r1, false, 1.0, 0.0,
                                                      nullptr, 0);
  }
  rowblock_finish_kernel<<<grid_for(mb * r1), 256, 0, st>>>(W, mb * r1, ns, r0, r1, K, ldk, G, ldg, mu2);
  return cudaGetLastError();
}

// One bordered step: rows r0..r1 of L^{-1} (into Wi) from the block's rows of
// G and the r0 rows of L^{-1} already there, then Ginv's lower triangle
// += Wi[r0:r1, 0:r1]^T Wi[r0:r1, 0:r1].
//   G rows: consumed (scratch afterwards); T rows r0..r1: scratch.
//   chain carries the dependent sequence, side the half of the inverse row
//   that does not need the diagonal factor, acc the rank-mb update.
cudaError_t bordered_chol_step(double* G, double* Wi, double* T, double* Ginv, int64_t ld, int64_t r0, int64_t r1,
                               int* info, cudaStream_t chain, cudaStream_t side, cudaStream_t acc, double* ws,
                               int64_t wcap) {
  // split-K workspaces: one for the chain's products, one for the side stream's
  double* ws_chain = ws;
  double* ws_side = ws ? ws + wcap / 2 : nullptr;
  const int64_t wc = wcap / 2;
  const int64_t mb = r1 - r0, p = r0;
  double* Gc = G + r0 * ld;
  double* Wc = Wi + r0 * ld;
  double* Tc = T + r0 * ld;
  std::vector<cudaEvent_t> evs;
  auto ev = [&]() {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    evs.push_back(e);
    return e;
  };
  cudaError_t e = cudaSuccess;
  auto done = [&](cudaError_t r) {
    for (cudaEvent_t x : evs) cudaEventDestroy(x);  // released once the recorded work completes
    return r;
  };
  cudaEvent_t ev_half = nullptr;
  if (p > 0) {
    // L_c = G[c, 0:p] W^T (W = L^{-1} of the rows before, lower triangular)
    if ((e = gemm_f64_splitk(Gc, ld, 1, Wi, ld, 1, mb, p, p, 1.0, 0.0, Tc, ld, chain, GEMM_B_KLE_N, ws_chain, wc)) !=
        cudaSuccess)
      return done(e);
    cudaEvent_t ev_fork = ev();
    ev_half = ev();
    cudaEventRecord(ev_fork, chain);
    cudaStreamWaitEvent(side, ev_fork, 0);
    // beside the diagonal block's factorisation: G[c, 0:p] <- L_c W
    if ((e = gemm_f64_splitk(Tc, ld, 1, Wi, 1, ld, mb, p, p, 1.0, 0.0, Gc, ld, side, GEMM_B_KGE_N, ws_side, wc)) !=
        cudaSuccess)
      return done(e);
    cudaEventRecord(ev_half, side);
    // S = G[c, c] - L_c L_c^T (lower tiles)
    if ((e = gemm_f64_splitk(Tc, ld, 1, Tc, ld, 1, mb, mb, p, -1.0, 1.0, Gc + r0, ld, chain, GEMM_C_LOWER, ws_chain,
                             wc)) != cudaSuccess)
      return done(e);
  }
  if ((e = chol_rec(Gc + r0, Wc + r0, Tc + r0, ld, mb, r0, info, chain, chol_side_stream(), evs)) != cudaSuccess)
    return done(e);
  if (p > 0) {
    cudaStreamWaitEvent(chain, ev_half, 0);
    // W[c, 0:p] = -W[c, c] (L_c W)
    if ((e = gemm_f64(Wc + r0, ld, 1, Gc, 1, ld, mb, p, mb, -1.0, 0.0, Wc, ld, chain, GEMM_A_KLE_M)) != cudaSuccess)
      return done(e);
  }
  cudaEvent_t ev_row = ev();
  cudaEventRecord(ev_row, chain);
  cudaStreamWaitEvent(acc, ev_row, 0);
  e = gemm_f64(Wc, 1, ld, Wc, 1, ld, r1, r1, mb, 1.0, 1.0, Ginv, ld, acc, GEMM_C_LOWER);
  return done(e);
}

// Ginv's upper triangle from its lower one (after the last bordered step)
cudaError_t mirror_lower(double* A, int64_t ld, int64_t m, cudaStream_t st) {
  mirror_lower_kernel<<<grid_for(m * m), 256, 0, st>>>(A, ld, m);
  return cudaGetLastError();
}

}  // namespace gdwd
