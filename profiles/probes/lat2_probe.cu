// Clean dependent-chain latency: 1024 unrolled ops, one warp.
#include <cstdio>
template <int W>
__global__ void k(double xd, float xf, double* od, float* of, long long* cyc) {
  double x = xd, y = 1.0000001, z = 1e-300;
  float f = xf, g = 1.0000001f, h = 1e-30f;
  long long t0 = clock64();
  if (W == 0) {
#pragma unroll
    for (int i = 0; i < 1024; ++i) x = __fma_rn(x, y, z);
  } else if (W == 1) {
#pragma unroll
    for (int i = 0; i < 1024; ++i) f = __fmaf_rn(f, g, h);
  } else if (W == 2) {
#pragma unroll
    for (int i = 0; i < 1024; ++i) x = __dadd_rn(x, y);
  } else if (W == 3) {  // 4 independent chains
    double a = x, b = x + 1, c = x + 2, d = x + 3;
#pragma unroll
    for (int i = 0; i < 256; ++i) { a = __fma_rn(a, y, z); b = __fma_rn(b, y, z); c = __fma_rn(c, y, z); d = __fma_rn(d, y, z); }
    x = a + b + c + d;
  }
  long long t1 = clock64();
  od[threadIdx.x] = x; of[threadIdx.x] = f; cyc[threadIdx.x] = t1 - t0;
}
int main() {
  double* od; float* of; long long* c;
  cudaMalloc(&od, 1024 * 8); cudaMalloc(&of, 1024 * 4); cudaMalloc(&c, 1024 * 8);
  long long h;
  const char* nm[] = {"DFMA chain", "FFMA chain", "DADD chain", "4x DFMA chains"};
  for (int w = 0; w < 4; ++w) {
    for (int r = 0; r < 2; ++r) {
      if (w == 0) k<0><<<1, 32>>>(1.5, 1.5f, od, of, c);
      if (w == 1) k<1><<<1, 32>>>(1.5, 1.5f, od, of, c);
      if (w == 2) k<2><<<1, 32>>>(1.5, 1.5f, od, of, c);
      if (w == 3) k<3><<<1, 32>>>(1.5, 1.5f, od, of, c);
    }
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-16s %6.1f cycles/op (1 warp)\n", nm[w], h / 1024.0);
  }
  // throughput-ish: 16 warps on one SM
  k<0><<<1, 512>>>(1.5, 1.5f, od, of, c); k<0><<<1, 512>>>(1.5, 1.5f, od, of, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA chain, 16 warps/SM: %6.1f cycles/op per warp\n", h / 1024.0);
}
