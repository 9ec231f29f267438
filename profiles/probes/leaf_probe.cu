// Time the 64 x 64 diagonal-block kernel of chol_inverse in isolation.
#include "../../paper_2305_12019_b200/csrc/gram.cu"
#include <cstdio>
#include <random>
#include <vector>
using namespace gdwd;
// variant: L and V = L^{-1} both in shared memory (dynamic, 2 x 64 x 65)
__global__ void __launch_bounds__(256) leaf_smem(double* A, int64_t lda, double* Linv, int64_t ldl, int m,
                                                 int* info) {
  extern __shared__ double ptsm[];
  double (*L)[65] = reinterpret_cast<double (*)[65]>(ptsm);
  double (*V)[65] = reinterpret_cast<double (*)[65]>(ptsm + 64 * 65);
  const int t = threadIdx.x;
  for (int idx = t; idx < 64 * 64; idx += blockDim.x) {
    const int i = idx >> 6, j = idx & 63;
    L[i][j] = (i < m && j < m && j <= i) ? A[i * lda + j] : 0.0;
    V[i][j] = 0.0;
  }
  __syncthreads();
  for (int j = 0; j < m; ++j) {
    if (t == 0) L[j][j] = sqrt(L[j][j]);
    __syncthreads();
    for (int i = j + 1 + t; i < m; i += blockDim.x) L[i][j] = L[i][j] / L[j][j];
    __syncthreads();
    for (int idx = t; idx < 64 * 64; idx += blockDim.x) {
      const int i = idx >> 6, k = idx & 63;
      if (k > j && i >= k && i < m) L[i][k] -= L[i][j] * L[k][j];
    }
    __syncthreads();
  }
  const int TIMING_SPLIT = 0;
  if (TIMING_SPLIT) return;
  {
    const int c = t >> 2, p = t & 3;
    for (int i = 0; i < m; ++i) {
      double s = 0.0;
      if (c < m && i > c)
        for (int k = c + p; k < i; k += 4) s += L[i][k] * V[k][c];
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (c < m && p == 0 && i >= c) V[i][c] = ((i == c ? 1.0 : 0.0) - s) / L[i][i];
      __syncwarp();
    }
  }
  __syncthreads();
  for (int idx = t; idx < m * m; idx += blockDim.x) {
    const int i = idx / m, j = idx % m;
    A[i * lda + j] = (j <= i) ? L[i][j] : 0.0;
    Linv[i * ldl + j] = (j <= i) ? V[i][j] : 0.0;
  }
}
__global__ void __launch_bounds__(256) leaf_potrf_only(double* A, int64_t lda, int m) {
  __shared__ double L[64][65];
  const int t = threadIdx.x;
  for (int idx = t; idx < 64 * 64; idx += blockDim.x) {
    const int i = idx >> 6, j = idx & 63;
    L[i][j] = (i < m && j < m && j <= i) ? A[i * lda + j] : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < m; ++j) {
    if (t == 0) L[j][j] = sqrt(L[j][j]);
    __syncthreads();
    for (int i = j + 1 + t; i < m; i += blockDim.x) L[i][j] = L[i][j] / L[j][j];
    __syncthreads();
    for (int idx = t; idx < 64 * 64; idx += blockDim.x) {
      const int i = idx >> 6, k = idx & 63;
      if (k > j && i >= k && i < m) L[i][k] -= L[i][j] * L[k][j];
    }
    __syncthreads();
  }
  for (int idx = t; idx < m * m; idx += blockDim.x) A[(idx / m) * lda + idx % m] = L[idx / m][idx % m];
}
int main() {
  const int m = 64, ld = 64;
  std::vector<double> S(m * m);
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  std::vector<double> X(m * 100);
  for (auto& v : X) v = nd(g);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int k = 0; k < 100; ++k) s += X[i * 100 + k] * X[j * 100 + k] / 100.0;
      S[i * m + j] = s;
    }
  double *dS, *dA, *dL;
  int* info;
  cudaMalloc(&dS, m * m * 8);
  cudaMalloc(&dA, m * m * 8);
  cudaMalloc(&dL, m * m * 8);
  cudaMalloc(&info, 4);
  cudaMemcpy(dS, S.data(), m * m * 8, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaFuncSetAttribute(leaf_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 64 * 65 * 8);
  for (int variant = 0; variant < 3; ++variant)
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(dA, dS, m * m * 8, cudaMemcpyDeviceToDevice);
    cudaEventRecord(a);
    for (int k = 0; k < 10; ++k) {
      cudaMemcpyAsync(dA, dS, m * m * 8, cudaMemcpyDeviceToDevice);
      if (variant == 0) potrf_trtri_small<<<1, 256>>>(dA, ld, dL, ld, m, info, 0);
      else if (variant == 1) leaf_smem<<<1, 256, 2 * 64 * 65 * 8>>>(dA, ld, dL, ld, m, info);
      else leaf_potrf_only<<<1, 256>>>(dA, ld, m);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("variant %d: %.1f us per launch incl. a 32 KB d2d copy (%s)\n", variant, ms * 100.0, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
