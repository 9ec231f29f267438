// chol_inverse timing probe: m x m SPD (K/1 + I with K a random Gram), CUDA
// events around each call after warm-up.  Build against gram.cu with
// (built against the library sources, no extension needed).
#include <cstdio>
#include <vector>
#include <random>
#include "../../paper_2305_12019_b200/csrc/gram.cuh"
using namespace gdwd;
int main(int argc, char** argv) {
  const int64_t m = argc > 1 ? atoll(argv[1]) : 2000, ld = (m + 1) / 2 * 2, r = 400;
  std::vector<double> X((size_t)m * r);
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  for (auto& v : X) v = nd(g) / 20.0;
  double *dX, *S, *A, *W;
  int* info;
  cudaMalloc(&dX, X.size() * 8);
  cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&S, m * ld * 8);
  cudaMalloc(&A, m * ld * 8);
  cudaMalloc(&W, 3 * m * ld * 8 + gram_workspace_doubles(m, r) * 8);
  cudaMalloc(&info, 4);
  cudaStream_t st;
  cudaStreamCreate(&st);
  gram_syrk(dX, m, r, r, false, 1.0, 1.0, S, ld, W, st);  // S = X X^T + I
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 6; ++rep) {
    cudaMemcpyAsync(A, S, m * ld * 8, cudaMemcpyDeviceToDevice, st);
    cudaMemsetAsync(info, 0, 4, st);
    cudaEventRecord(a, st);
    chol_inverse(A, W, W + m * ld, ld, m, info, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int inf;
    cudaMemcpy(&inf, info, 4, cudaMemcpyDeviceToHost);
    if (rep) printf("m=%lld chol_inverse %.3f ms (info %d) %s\n", (long long)m, ms, inf, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
