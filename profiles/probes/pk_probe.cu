// Micro-probe for the persistent Gram-space kernel's phase structure:
// 148 CTAs x 512 threads, ~180 KB dynamic smem (same L1 carve-out), phases of
// "sweep an L2-resident n x n matrix with one warp per row, then grid barrier".
// Reports us per phase for: barrier only, sweep + barrier (several load
// shapes), and a hand-rolled barrier.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

struct Args {
  const double* K0;
  const double* K1;
  int n, ld, phases, sweep, custom, rows_split, nred;
  double* part;
  double* out;
  unsigned* bar;
};

__device__ __forceinline__ void my_grid_sync(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned target = (gen + 1) * gridDim.x;
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  gen++;
  __syncthreads();
}

template <int U>
__device__ double rowdot(const double* row, int n, const double* x) {
  const int lane = threadIdx.x & 31;
  double acc = 0;
  for (int j0 = 2 * lane; j0 < n + 2 * lane; j0 += U * 64) {
    double2 z[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int j = j0 + u * 64;
      z[u] = j < n ? __ldg(reinterpret_cast<const double2*>(row + j)) : make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int j = j0 + u * 64;
      if (j < n) {
        double2 xv = *reinterpret_cast<const double2*>(x + j);
        acc += z[u].x * xv.x + z[u].y * xv.y;
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

template <int K>
__device__ void warp_sum(double (&v)[K]) {
#pragma unroll
  for (int o = 16; o; o >>= 1)
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
}
template <int K>
__device__ void block_sum(double (&v)[K], double* scratch) {
  warp_sum<K>(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0)
    for (int k = 0; k < K; ++k) scratch[wid * K + k] = v[k];
  __syncthreads();
  if (wid == 0) {
    for (int k = 0; k < K; ++k) v[k] = lane < nw ? scratch[lane * K + k] : 0.0;
    warp_sum<K>(v);
  }
  __syncthreads();
}
__device__ __forceinline__ double ld_cg(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
template <int K>
__device__ double reduce_phase(double* part, int slot, double x, double* red, cg::grid_group& grid, int custom,
                               unsigned* bar, unsigned& gen) {
  double t[K];
  for (int k = 0; k < K; ++k) t[k] = x * (k + 1);
  block_sum<K>(t, red);
  if (threadIdx.x == 0) {
    double* p = part + (size_t)slot * gridDim.x * 14 + blockIdx.x;
    for (int k = 0; k < K; ++k) p[(size_t)k * gridDim.x] = t[k];
  }
  if (custom) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned target = (gen + 1) * gridDim.x;
      __threadfence();
      atomicAdd(bar, 1u);
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      } while (v < target);
    }
    gen++;
    __syncthreads();
  } else {
    grid.sync();
  }
  const double* p = part + (size_t)slot * gridDim.x * 14;
  double v[K];
  for (int k = 0; k < K; ++k) v[k] = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
    for (int k = 0; k < K; ++k) v[k] += ld_cg(p + (size_t)k * gridDim.x + b);
  const int nw = ((int)gridDim.x + 31) / 32, warp = threadIdx.x >> 5;
  if (warp < nw) {
    warp_sum<K>(v);
    if ((threadIdx.x & 31) == 0)
      for (int k = 0; k < K; ++k) red[warp * K + k] = v[k];
  }
  __syncthreads();
  double o = 0;
  for (int k = 0; k < K; ++k) {
    double tt = 0;
    for (int w = 0; w < nw; ++w) tt += red[w * K + k];
    o += tt;
  }
  return o;
}

// two rows per warp sharing the x loads; NX right-hand sides
template <int U, int NX>
__device__ void rowdot2(const double* r0, const double* r1, int n, const double* x, double* o) {
  const int lane = threadIdx.x & 31;
  double a0[NX], a1[NX];
  for (int v = 0; v < NX; ++v) a0[v] = a1[v] = 0;
  for (int j0 = 2 * lane; j0 < n + 2 * lane; j0 += U * 64) {
    double2 z0[U], z1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int j = j0 + u * 64;
      z0[u] = j < n ? __ldg(reinterpret_cast<const double2*>(r0 + j)) : make_double2(0, 0);
      z1[u] = j < n ? __ldg(reinterpret_cast<const double2*>(r1 + j)) : make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int j = j0 + u * 64;
      if (j < n) {
#pragma unroll
        for (int v = 0; v < NX; ++v) {
          double2 xv = *reinterpret_cast<const double2*>(x + v * 2048 + j);
          a0[v] += z0[u].x * xv.x + z0[u].y * xv.y;
          a1[v] += z1[u].x * xv.x + z1[u].y * xv.y;
        }
      }
    }
  }
  for (int v = 0; v < NX; ++v) {
#pragma unroll
    for (int q = 16; q; q >>= 1) {
      a0[v] += __shfl_xor_sync(0xffffffffu, a0[v], q);
      a1[v] += __shfl_xor_sync(0xffffffffu, a1[v], q);
    }
    o[v] = a0[v] + a1[v];
  }
}
template <int U, int NX>
__device__ void rowdot1(const double* r0, int n, const double* x, double* o) {
  const int lane = threadIdx.x & 31;
  double a0[NX];
  for (int v = 0; v < NX; ++v) a0[v] = 0;
  for (int j0 = 2 * lane; j0 < n + 2 * lane; j0 += U * 64) {
    double2 z0[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int j = j0 + u * 64;
      z0[u] = j < n ? __ldg(reinterpret_cast<const double2*>(r0 + j)) : make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int j = j0 + u * 64;
      if (j < n) {
#pragma unroll
        for (int v = 0; v < NX; ++v) {
          double2 xv = *reinterpret_cast<const double2*>(x + v * 2048 + j);
          a0[v] += z0[u].x * xv.x + z0[u].y * xv.y;
        }
      }
    }
  }
  for (int v = 0; v < NX; ++v) {
#pragma unroll
    for (int q = 16; q; q >>= 1) a0[v] += __shfl_xor_sync(0xffffffffu, a0[v], q);
    o[v] = a0[v];
  }
}

__global__ void __launch_bounds__(512, 1) probe(Args A) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = threadIdx.x; j < 3 * 2048; j += blockDim.x) sm[j] = 1.0;
  __syncthreads();
  const int n = A.n;
  double acc = 0;
  unsigned gen = 0;
  // row partition: rows_split warps per row (each a contiguous column range)
  const int i0 = (long)n * blockIdx.x / gridDim.x, i1 = (long)n * (blockIdx.x + 1) / gridDim.x;
  for (int p = 0; p < A.phases; ++p) {
    const double* K = (p & 1) ? A.K1 : A.K0;
    if (A.sweep >= 100) {  // 100 + 10*pairs + NX
      const int pairs = (A.sweep / 10) % 10, nx = A.sweep % 10;
      double o[3];
      if (pairs) {
        for (int r = 2 * warp; r < i1 - i0; r += 32) {
          const double* r0 = K + (size_t)(i0 + r) * A.ld;
          const double* r1 = r + 1 < i1 - i0 ? r0 + A.ld : r0;
          if (nx == 1) rowdot2<8, 1>(r0, r1, n, sm, o);
          else rowdot2<8, 3>(r0, r1, n, sm, o);
          if (lane == 0) acc += o[0];
        }
      } else {
        for (int r = warp; r < i1 - i0; r += 16) {
          const double* r0 = K + (size_t)(i0 + r) * A.ld;
          if (nx == 1) rowdot1<16, 1>(r0, n, sm, o);
          else rowdot1<16, 3>(r0, n, sm, o);
          if (lane == 0) acc += o[0];
        }
      }
    } else if (A.sweep) {
      if (A.rows_split == 1) {
        for (int r = warp; r < i1 - i0; r += 16) {
          double d = A.sweep == 8 ? rowdot<8>(K + (size_t)(i0 + r) * A.ld, n, sm)
                                 : rowdot<16>(K + (size_t)(i0 + r) * A.ld, n, sm);
          if (lane == 0) acc += d;
        }
      } else {
        // split each row into rows_split column ranges; work items = rows*split
        const int S = A.rows_split, items = (i1 - i0) * S;
        for (int it = warp; it < items; it += 16) {
          const int r = it / S, s = it % S;
          const int c0 = (int)((long)n * s / S) & ~1, c1 = s + 1 == S ? n : (int)((long)n * (s + 1) / S) & ~1;
          double d = rowdot<16>(K + (size_t)(i0 + r) * A.ld + c0, c1 - c0, sm + c0);
          if (lane == 0) acc += d;
        }
      }
    }
    if (A.nred) {
      __shared__ double red[16 * 14];
      const int slot = p & 1;
      double x = acc + 1.0;
      double o = A.nred == 1 ? reduce_phase<1>(A.part, slot, x, red, grid, A.custom, A.bar, gen)
               : A.nred == 2 ? reduce_phase<2>(A.part, slot, x, red, grid, A.custom, A.bar, gen)
                             : reduce_phase<14>(A.part, slot, x, red, grid, A.custom, A.bar, gen);
      acc += o * 1e-30;
    } else if (A.custom) my_grid_sync(A.bar, gen);
    else grid.sync();
  }
  if (acc == 1.2345) A.out[0] = acc;
}

int main() {
  const int n = 2000, ld = 2000;
  double *K0, *K1, *out;
  unsigned* bar;
  cudaMalloc(&K0, (size_t)n * ld * 8);
  cudaMalloc(&K1, (size_t)n * ld * 8);
  cudaMemset(K0, 0, (size_t)n * ld * 8);
  cudaMemset(K1, 0, (size_t)n * ld * 8);
  cudaMalloc(&out, 8);
  cudaMalloc(&bar, 4);
  const size_t smem = 180 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double* part;
  cudaMalloc(&part, 2 * 148 * 14 * 8);
  struct Cfg { const char* name; int sweep, custom, split, nred; } cfgs[] = {
      {"grid.sync only", 0, 0, 1, 0}, {"sweep U16 + grid.sync", 16, 0, 1, 0},
      {"1 row/warp, 1 rhs", 101, 0, 1, 0}, {"2 rows/warp, 1 rhs", 111, 0, 1, 0},
      {"1 row/warp, 3 rhs", 103, 0, 1, 0}, {"2 rows/warp, 3 rhs", 113, 0, 1, 0}};
  for (auto& c : cfgs) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(bar, 0, 4);
      Args A{K0, K1, n, ld, 400, c.sweep, c.custom, c.split, c.nred, part, out, bar};
      void* args[] = {&A};
      cudaEventRecord(a);
      cudaError_t e0 = cudaLaunchCooperativeKernel((void*)probe, 148, 512, args, smem, 0);
      cudaEventRecord(b);
      cudaError_t e = cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("%-28s %7.2f us/phase (%s %s)\n", c.name, ms * 1e3 / 400, cudaGetErrorString(e0), cudaGetErrorString(e));
    }
  }
  return 0;
}
