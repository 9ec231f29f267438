// Dependent-chain latency (cycles per op) of the fp64 operations in the Newton prox.
#include <cstdio>
#include "solver_ops.cuh"
using namespace gdwd;
__global__ void k(double x0, int which, double* out, long long* cyc) {
  double x = x0, y = 1.0000001;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
    switch (which) {
      case 0: x = __dmul_rn(x, y); break;
      case 1: x = __fma_rn(x, y, 1e-300); break;
      case 2: x = __ddiv_rn(x, y); break;
      case 3: x = np_pow(x, -2.0) * 1e-300 + 1.5; break;
      case 4: x = pow(x, 0.3333333333333333) + 1.0; break;
      case 5: x = (double)ilogb(x) * 1e-300 + x; break;
      case 6: x = pow_int_dd(x, -2) + 1.0; break;
      case 7: x = newton_margin(x * 1e-300 + 0.3, 10.0, 1.0, 0.7, 1.0, 1e-8) + 1.0; break;
      case 8: x = newton_margin(x * 1e-300 + 0.3, 3e13, 1.0, 0.7, 0.5, 1e-8) + 1.0; break;
      case 9: x = bisect_margin(x * 1e-300 + 0.3, 3e13, 1.0, 0.7, 1e-8) + 1.0; break;
      case 10: x = np_pow(x, 2.0) * 1e-300 + 1.5; break;
      case 11: x = sqrt(x) + 1.0; break;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  cyc[threadIdx.x] = t1 - t0;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 64 * 8);
  const char* nm[] = {"dmul", "dfma", "ddiv", "np_pow(x,-2)", "pow(x,1/3)", "ilogb", "pow_int_dd(-2)",
                      "newton sig=10", "newton sig=3e13", "bisect sig=3e13", "np_pow(x,2)", "sqrt"};
  for (int w = 0; w < 12; ++w) {
    for (int r = 0; r < 2; ++r) k<<<1, 32>>>(1.5, w, o, c);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-18s %8.1f cycles/op\n", nm[w], h / 256.0);
  }
}
