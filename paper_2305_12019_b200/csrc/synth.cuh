// On-device generation of the dense synthetic configurations (BASELINE.json
// configs[4]: 160 GB does not fit host memory in the build container, and a
// host generator would take minutes).  Counter-based: the noise of sample i
// (global index), features (2p, 2p+1) is a Box-Muller pair from a splitmix64
// hash of (seed, i, p), so any shard regenerates its columns independently.
// This stream differs from synth.py's numpy Philox stream (which the host
// configs and the golden fixtures use); device-generated proxies are checked
// against the oracle by downloading them.
#pragma once
#include "common.cuh"

namespace gdwd {

GDWD_DEV uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

GDWD_DEV double u01(uint64_t h) {  // (0, 1]
  return ((double)(h >> 11) + 1.0) * (1.0 / 9007199254740992.0);
}

// X[i][j] = ytrue_i * shift * [j < signal_k] + N(0,1)  (kind 0: iid noise)
__global__ void gen_gauss_kernel(double* Zs, int64_t ld, int64_t d, int64_t n, int64_t offset, uint64_t seed,
                                 int64_t signal_k, double shift) {
  const int64_t pairs = (d + 1) / 2;
  const int64_t tot = n * pairs;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / pairs, p = idx % pairs;
    const uint64_t gi = (uint64_t)(offset + i);
    const uint64_t h1 = splitmix64(seed ^ splitmix64(gi * 0x100000001B3ull + (uint64_t)p * 2));
    const uint64_t h2 = splitmix64(h1 ^ 0x5851F42D4C957F2Dull);
    const double r = sqrt(-2.0 * log(u01(h1)));
    double s, c;
    sincospi(2.0 * u01(h2), &s, &c);
    const double yt = (gi & 1) ? -1.0 : 1.0;  // true labels alternate (synth.true_labels)
    const int64_t j = 2 * p;
    double* row = Zs + i * ld;
    row[j] = r * c + (j < signal_k ? yt * shift : 0.0);
    if (j + 1 < d) row[j + 1] = r * s + (j + 1 < signal_k ? yt * shift : 0.0);
  }
}

// Z~ = X diag(y) / z_scale in place (scale_problem, solver.py:269-276:
// values * col_sign / z_scale)
__global__ void scale_rows_kernel(double* Zs, int64_t ld, int64_t d, int64_t n, const double* y, double z_scale) {
  const int64_t tot = n * d;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / d, j = idx % d;
    double* p = Zs + i * ld + j;
    *p = (*p * y[i]) / z_scale;
  }
}

}  // namespace gdwd
