// L2-resident read bandwidth probe (denominator for the persistent SMW2
// kernel, whose K / G^{-1}K sweeps hit L2).  Reads a buffer of S bytes
// repeatedly with 16-byte loads; prints GB/s per size and grid.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const double2* __restrict__ p, size_t n2, int reps, double* out) {
  double2 acc = {0, 0};
  for (int r = 0; r < reps; ++r) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldg(p + i);
      acc.x += v.x;
      acc.y += v.y;
    }
  }
  if (acc.x == 1.2345) out[0] = acc.y;
}

// persistent-style: one warp per row of length L doubles, rows spread over CTAs
__global__ void rows(const double* __restrict__ K, int n, int reps, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int i0 = (long)n * blockIdx.x / gridDim.x, i1 = (long)n * (blockIdx.x + 1) / gridDim.x;
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (int i = i0 + warp; i < i1; i += nw) {
      const double* row = K + (size_t)i * n;
      for (int j = 2 * lane; j < n; j += 64) {
        double2 v = __ldg(reinterpret_cast<const double2*>(row + j));
        acc += v.x + v.y;
      }
    }
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* buf;
  size_t maxb = (size_t)256 << 20;
  cudaMalloc(&buf, maxb);
  cudaMemset(buf, 0, maxb);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t mb : {8, 16, 32, 64, 96, 256}) {
    size_t bytes = mb << 20, n2 = bytes / 16;
    for (int per : {1, 2, 4, 8}) {
      int reps = mb >= 256 ? 5 : 40;
      rd<<<sms * per, 512>>>((const double2*)buf, n2, 1, out);
      cudaEventRecord(a);
      rd<<<sms * per, 512>>>((const double2*)buf, n2, reps, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("stream %4zu MB grid %dx%d: %.0f GB/s\n", mb, sms, per, bytes * (double)reps / (ms * 1e-3) / 1e9);
    }
  }
  for (int n : {2000, 2896}) {
    for (int th : {256, 512, 1024}) {
      int reps = 40;
      rows<<<sms, th>>>(buf, n, 1, out);
      cudaEventRecord(a);
      rows<<<sms, th>>>(buf, n, reps, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double bytes = 8.0 * n * n;
      printf("rows n=%d (%.0f MB) %d thr: %.0f GB/s, %.2f us/sweep\n", n, bytes / 1048576, th,
             bytes * reps / (ms * 1e-3) / 1e9, ms * 1e3 / reps);
    }
  }
  return 0;
}
