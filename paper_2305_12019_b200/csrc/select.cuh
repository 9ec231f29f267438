// Between-class distance statistic of the penalty-C heuristic
// (reference solver.py:193-232, compute_penalty_C):
//   gather the two (subsampled) classes into dense blocks, squared norms,
//   the between-class Gram A B^T on the FP64 tensor cores (gram.cu),
//   d_ij = sqrt(max(|a_i|^2 + |b_j|^2 - 2 a_i.b_j, 0)), and the exact median
//   of the positive d_ij by radix selection on the IEEE bit patterns
//   (non-negative doubles order like their uint64 patterns).
#pragma once
#include "common.cuh"
#include "spops.cuh"

namespace gdwd {

// rows idx[] of the dense sample-major matrix (stride ldz) -> out [cnt][ldo]
__global__ void gather_rows_kernel(const double* Zs, int64_t ldz, const int64_t* idx, int64_t cnt, int64_t d,
                                   double* out, int64_t ldo) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= cnt) return;
  const double* src = Zs + idx[r] * ldz;
  double* dst = out + r * ldo;
  for (int64_t k = threadIdx.x & 31; k < d; k += 32) dst[k] = src[k];
}

// CSC columns idx[] -> dense rows of out (zeroed by the caller)
__global__ void gather_csc_kernel(SpView csc, const int64_t* idx, int64_t cnt, double* out, int64_t ldo) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= cnt) return;
  const int64_t c = idx[r];
  for (int64_t k = csc.ptr[c] + (threadIdx.x & 31); k < csc.ptr[c + 1]; k += 32) out[r * ldo + csc.idx[k]] = csc.val[k];
}

// squared norm of each row (warp per row, fixed lane-strided order + tree)
__global__ void row_sq_kernel(const double* A, int64_t lda, int64_t rows, int64_t d, double* sq) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= rows) return;
  double v[1] = {0.0};
  for (int64_t k = threadIdx.x & 31; k < d; k += 32) {
    const double a = A[r * lda + k];
    v[0] += a * a;
  }
  warp_sum<1>(v);
  if ((threadIdx.x & 31) == 0) sq[r] = v[0];
}

// d_ij from the Gram; counts exact zeros (duplicated points across classes)
__global__ void between_dist_kernel(const double* G, int64_t ldg, const double* sqa, const double* sqb, int64_t na,
                                    int64_t nb, double* dist, unsigned long long* zeros) {
  const int64_t tot = na * nb;
  unsigned long long z = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / nb, j = t % nb;
    double d2 = (sqa[i] + sqb[j]) - 2.0 * G[i * ldg + j];
    d2 = isnan(d2) ? d2 : (d2 > 0.0 ? d2 : 0.0);  // np.maximum(d2, 0)
    const double dv = sqrt(d2);
    dist[t] = dv;
    z += (dv == 0.0) ? 1ull : 0ull;
  }
  for (int off = 16; off > 0; off >>= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
  if ((threadIdx.x & 31) == 0 && z) atomicAdd(zeros, z);
}

// Radix selection of the k-th smallest (0-based) value: 8 passes of 8 bits
// from the most significant.  state = {prefix, k}; each pass histograms the
// next digit of the values that match the prefix so far, then one thread
// picks the bucket holding rank k.
__global__ void radix_hist_kernel(const double* v, int64_t n, const unsigned long long* state, int shift,
                                  unsigned long long* hist) {
  __shared__ unsigned long long h[256];
  for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const unsigned long long prefix = state[0];
  const unsigned long long hi_mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v[t]);
    if ((bits & hi_mask) == (prefix & hi_mask)) atomicAdd(&h[(bits >> shift) & 255ull], 1ull);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x)
    if (h[b]) atomicAdd(&hist[b], h[b]);
}

__global__ void radix_pick_kernel(unsigned long long* hist, unsigned long long* state, int shift) {
  if (threadIdx.x != 0) return;
  unsigned long long k = state[1], acc = 0;
  int b = 0;
  for (; b < 256; ++b) {
    if (acc + hist[b] > k) break;
    acc += hist[b];
  }
  if (b > 255) b = 255;
  state[0] |= (unsigned long long)b << shift;
  state[1] = k - acc;
  for (int c = 0; c < 256; ++c) hist[c] = 0;
}

}  // namespace gdwd
