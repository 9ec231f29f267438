// DMMA throughput vs warps per SM and independent accumulator chains per warp
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(int iters, double* out) {
  double c[CH][2];
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
template <int CH>
void run(int warps, double* out) {
  const int sms = 148, iters = 20000 / CH * 8;
  k<CH><<<sms, warps * 32>>>(100, out);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<CH><<<sms, warps * 32>>>(iters, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flop = 2.0 * 8 * 8 * 4 * CH * (double)iters * warps * sms;
  printf("warps/SM %2d chains %2d: %.2f TF/s\n", warps, CH, flop / (ms * 1e-3) / 1e12);
}
int main() {
  double* out; cudaMalloc(&out, 8);
  for (int w : {4, 8, 12, 16, 24, 32}) { run<8>(w, out); run<16>(w, out); run<32>(w, out); }
  return 0;
}
