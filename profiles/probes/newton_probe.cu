// Latency of the Newton prox (newton_margin / newton_margin_warp) per sample
// inside one CTA-wave, at the sigma regime config 2 reaches late (3e13):
// cycles per sample (clock64), Newton counts, median / max.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <random>
#include <vector>
#include "solver_ops.cuh"
using namespace gdwd;

__global__ void per_warp(const double* a, const double* w, const double* r0, int n, double sigma, double q, double tol,
                         double* out, long long* cyc, int* its, int warp_form) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; gw < n; gw += nw) {
  long long t0 = clock64();
  int it = 0;
  double r;
  if (warp_form) r = newton_margin_warp(a[gw], sigma, q, w[gw], r0[gw], tol, 50, 0, &it);
  else {
    r = 0.0;
    if (lane == 0) r = newton_margin(a[gw], sigma, q, w[gw], r0[gw], tol, 50, 0, &it);
  }
  long long t1 = clock64();
  if (lane == 0) {
    out[gw] = r;
    cyc[gw] = t1 - t0;
    its[gw] = it;
  }
  }
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  int cfg = -1;
  const int n = 2000;
  std::mt19937_64 g(1);
  std::normal_distribution<double> N(0, 1);
  std::uniform_real_distribution<double> U(0, 1);
  std::vector<double> a(n), w(n), r0(n);
  for (int i = 0; i < n; ++i) {
    a[i] = N(g) * 2;
    w[i] = U(g) + 0.1;
    r0[i] = std::pow(10.0, -3 + 4 * U(g));
  }
  double *da, *dw, *dr, *dout;
  long long* dc;
  int* di;
  cudaMalloc(&da, n * 8); cudaMalloc(&dw, n * 8); cudaMalloc(&dr, n * 8); cudaMalloc(&dout, n * 8);
  cudaMalloc(&dc, n * 8); cudaMalloc(&di, n * 4);
  cudaMemcpy(da, a.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, w.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, r0.data(), n * 8, cudaMemcpyHostToDevice);
  for (double q : {1.0, 2.0})
    for (double sigma : {10.0, 3e13})
      for (int wpb : {1, 4, 16})
      for (int wf = 0; wf < 2; ++wf) {
        ++cfg;
        if (only >= 0 && cfg != only) continue;
        for (int rep = 0; rep < 2; ++rep)
          per_warp<<<148, 32 * wpb>>>(da, dw, dr, n, sigma, q, 1e-8, dout, dc, di, wf);
        cudaDeviceSynchronize();
        std::vector<long long> c(n);
        std::vector<int> it(n);
        cudaMemcpy(c.data(), dc, n * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(it.data(), di, n * 4, cudaMemcpyDeviceToHost);
        std::vector<long long> cs = c;
        std::sort(cs.begin(), cs.end());
        int imax = std::max_element(c.begin(), c.end()) - c.begin();
        printf("q=%g sigma=%g wpb=%2d %s: cycles median %lld p90 %lld max %lld (sample %d: a=%g r0=%g newton its %d)  [%s]\n", q,
               sigma, wpb, wf ? "warp  " : "thread", cs[n / 2], cs[n * 9 / 10], cs[n - 1], imax, a[imax], r0[imax], it[imax],
               cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
