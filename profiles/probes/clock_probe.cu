// Effective SM clock of a single-CTA kernel vs a full-GPU kernel: a chain of
// dependent integer adds of known length, timed with events and clock64.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(long long iters, unsigned long long* out) {
  unsigned long long t0 = clock64();
  unsigned x = threadIdx.x;
  for (long long i = 0; i < iters; ++i) x = x * 1664525u + 1013904223u;
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = x; }
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int grid : {1, 1, 148, 148 * 4, 1}) {
    const long long it = 20000000;
    cudaEventRecord(a);
    chain<<<grid, 128>>>(it, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("grid %4d: %.3f ms, %llu cycles -> %.0f MHz\n", grid, ms, h[0], h[0] / (ms * 1e3));
  }
  return 0;
}
