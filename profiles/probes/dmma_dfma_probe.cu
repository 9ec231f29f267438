// Do the FP64 tensor pipe (DMMA) and the FP64 CUDA-core pipe (DFMA) run concurrently?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int iters, int mode, double* out) {  // mode 0: all DMMA, 1: all DFMA, 2: even warps DMMA / odd warps DFMA
  const int warp = threadIdx.x >> 5;
  const bool dm = mode == 0 || (mode == 2 && (warp & 1) == 0);
  double s = 0;
  if (dm) {
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else {
    double c[16];
    for (int i = 0; i < 16; ++i) c[i] = i;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) c[i] = __fma_rn(c[i], a, b);
    for (int i = 0; i < 16; ++i) s += c[i];
  }
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* out; cudaMalloc(&out, 8);
  const int sms = 148, warps = 16, iters = 20000;
  for (int mode = 0; mode < 3; ++mode) {
    k<<<sms, warps * 32>>>(100, mode, out);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<sms, warps * 32>>>(iters, mode, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    // flops: DMMA warp: 8 x 512 per iter; DFMA warp: 16 x 32 lanes x 2 per iter = 1024
    double wd = mode == 0 ? warps : (mode == 2 ? warps / 2 : 0), wf = warps - wd;
    double flop = ((double)iters * sms) * (wd * 8 * 512 + wf * 1024);
    printf("mode %d: %.3f ms, %.2f TF/s (DMMA warps %g, DFMA warps %g)\n", mode, ms, flop / (ms * 1e-3) / 1e12, wd, wf);
  }
  return 0;
}
