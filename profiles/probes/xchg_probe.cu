// Exchange-latency probe for the persistent Gram-space kernel: 148 CTAs x 512
// threads, each phase every CTA owns n/148 entries of V n-vectors plus NP
// partial sums, and every CTA needs all of them (vectors in shared memory,
// partials summed in a fixed order) before the next phase.  Modes:
//   0  plain stores + cooperative grid.sync + TMA bulk copy of the vectors
//      (+ ld.cg of the partials)                     -- the current kernel
//   1  "LL" words: each double travels as {lo32, flag, hi32, flag} in one
//      16-byte volatile store; readers poll until both flags carry the phase
//      epoch (8-byte single-copy atomicity), so barrier + data is one trip
//   2  per-CTA flag (release pattern: data, fence, flag store); thread b
//      polls CTA b's flag, fence, then plain loads of the vectors
// Reports microseconds per phase (no GEMV sweep: the exchange floor).
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int T = 512;

struct Args {
  int n, V, NP, phases, mode;
  double* vec;      // mode 0/2: [V][n]
  double* part;     // mode 0/2: [NP][grid]
  uint4* llvec;     // mode 1: [V][n]
  uint4* llpart;    // mode 1: [NP][grid]
  unsigned* flags;  // mode 2: [grid]
  double* out;
  unsigned epoch0;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void st_ll(uint4* p, double v, unsigned f) {
  unsigned long long b = __double_as_longlong(v);
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"((unsigned)b), "r"(f),
               "r"((unsigned)(b >> 32)), "r"(f)
               : "memory");
}
__device__ __forceinline__ uint4 ld_ll(const uint4* p) {
  uint4 r;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}
__device__ __forceinline__ double ll_val(uint4 r) {
  return __longlong_as_double(((unsigned long long)r.z << 32) | r.x);
}

__global__ void __launch_bounds__(T, 1) probe(Args A) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];  // [V][n]
  __shared__ unsigned long long bar;
  __shared__ double red[64];
  const int n = A.n, V = A.V, NP = A.NP;
  const int i0 = (int)((long)n * blockIdx.x / gridDim.x), i1 = (int)((long)n * (blockIdx.x + 1) / gridDim.x);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  for (int j = threadIdx.x; j < V * n; j += T) sm[j] = 1.0;
  __syncthreads();
  unsigned parity = 0;
  double acc = 0.0;
  for (int p = 0; p < A.phases; ++p) {
    const unsigned f = A.epoch0 + p;
    uint4* llvec = A.llvec + (size_t)(p & 1) * 3 * 2048;  // double-buffered: a writer two phases ahead
    uint4* llpart = A.llpart + (size_t)(p & 1) * 16 * 148;  // cannot overwrite what a reader still polls
    // produce: owners' entries depend on what was read last phase
    if (A.mode != 3)
    for (int v = 0; v < V; ++v)
      for (int i = i0 + threadIdx.x; i < i1; i += T) {
        const double x = sm[v * n + (i + 1) % n] * 0.5 + 0.25;
        if (A.mode == 1) st_ll(llvec + (size_t)v * n + i, x, f);
        else A.vec[(size_t)v * n + i] = x;
      }
    if (threadIdx.x < NP && A.mode != 3 && A.mode != 8 && A.mode != 9 && A.mode != 12) {
      const double x = sm[threadIdx.x] + 1.0;
      if (A.mode == 1) st_ll(llpart + (size_t)threadIdx.x * gridDim.x + blockIdx.x, x, f);
      else A.part[(size_t)threadIdx.x * gridDim.x + blockIdx.x] = x;
    }
    if (A.mode == 0 || (A.mode >= 3 && A.mode < 8)) {
      if (A.mode == 7) {
        __syncthreads();
        if (threadIdx.x == 0) { __threadfence(); }
        __syncthreads();
      } else grid.sync();
      if (threadIdx.x == T - 32 && (A.mode == 0 || A.mode == 6)) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        const unsigned bytes = (unsigned)(n * 8);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(V * bytes)
                     : "memory");
        for (int v = 0; v < V; ++v)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(sm + v * n)),
              "l"(A.vec + (size_t)v * n), "r"(bytes), "r"(smem_u32(&bar))
              : "memory");
      }
      // cross-sum of partials: warp k sums value k
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      if (warp < NP && (A.mode == 0 || A.mode == 5)) {
        double s = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) s += __ldcg(A.part + (size_t)warp * gridDim.x + b);
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red[warp] = s;
      }
      if (A.mode == 0 || A.mode == 6) asm volatile(
          "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
              smem_u32(&bar)),
          "r"(parity)
          : "memory");
      if (A.mode == 0 || A.mode == 6) parity ^= 1;
      __syncthreads();
    } else if (A.mode == 11 || A.mode == 12) {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      uint4* lp = llpart;
      if (A.mode == 11) {
        __syncthreads();
        if (threadIdx.x == 0) {
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(A.flags + 0) : "memory");
          unsigned v;
          const unsigned target = (f - A.epoch0 + 1) * gridDim.x;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(A.flags + 0) : "memory");
          } while ((int)(v - target) < 0);
        }
        __syncthreads();
      } else {
        __syncthreads();
        if (threadIdx.x == 0) {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          for (int k = 0; k < NP; ++k) st_ll(lp + (size_t)blockIdx.x * 16 + k, sm[k] + 1.0, f);
        }
        if (threadIdx.x < gridDim.x) {
          const uint4* q = lp + (size_t)threadIdx.x * 16;
          uint4 r[16];
          bool ok;
          do {
            ok = true;
            for (int k = 0; k < NP; ++k) r[k] = ld_ll(q + k);
            for (int k = 0; k < NP; ++k) ok &= (r[k].y == f && r[k].w == f);
          } while (!ok);
          double s = 0.0;
          for (int k = 0; k < NP; ++k) s += ll_val(r[k]);
          acc += s * 1e-300;
        }
        if (lane == 0 && warp * 32 < (int)gridDim.x) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        __syncthreads();
      }
      if (threadIdx.x == T - 32) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        const unsigned bytes = (unsigned)(n * 8);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(V * bytes)
                     : "memory");
        for (int v = 0; v < V; ++v)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(sm + v * n)),
              "l"(A.vec + (size_t)v * n), "r"(bytes), "r"(smem_u32(&bar))
              : "memory");
      }
      if (A.mode == 11 && warp < NP) {
        double s = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) s += __ldcg(A.part + (size_t)warp * gridDim.x + b);
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red[warp] = s;
      }
      asm volatile(
          "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
              smem_u32(&bar)),
          "r"(parity)
          : "memory");
      parity ^= 1;
      __syncthreads();
    } else if (A.mode >= 8) {
      // barrier + partials in one trip: per-CTA LL words (value, epoch) written
      // after a release fence (mode 8) or none (9); mode 10: release/acquire flag + ld.cg partials
      uint4* lp = llpart;
      if (A.mode == 10) {
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(A.flags + blockIdx.x), "r"(f) : "memory");
        if (threadIdx.x < gridDim.x) {
          unsigned g;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(A.flags + threadIdx.x) : "memory");
          } while ((int)(g - f) < 0);
        }
        __syncthreads();
      } else {
        __syncthreads();
        if (threadIdx.x < 32) {
          if (A.mode == 8 && threadIdx.x == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
          __syncwarp();
          if (threadIdx.x < NP) st_ll(lp + (size_t)blockIdx.x * 16 + threadIdx.x, sm[threadIdx.x] + 1.0, f);
        }
        if (threadIdx.x < gridDim.x) {
          const uint4* q = lp + (size_t)threadIdx.x * 16;
          double s = 0.0;
          for (int k = 0; k < NP; ++k) {
            uint4 r;
            do { r = ld_ll(q + k); } while (r.y != f || r.w != f);
            s += ll_val(r);
          }
          if (A.mode == 8) asm volatile("fence.acq_rel.gpu;" ::: "memory");
          acc += s * 1e-300;
        }
        __syncthreads();
      }
      if (threadIdx.x == T - 32) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        const unsigned bytes = (unsigned)(n * 8);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(V * bytes)
                     : "memory");
        for (int v = 0; v < V; ++v)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(sm + v * n)),
              "l"(A.vec + (size_t)v * n), "r"(bytes), "r"(smem_u32(&bar))
              : "memory");
      }
      if (A.mode == 10) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (warp < NP) {
          double s = 0.0;
          for (int b = lane; b < (int)gridDim.x; b += 32) s += __ldcg(A.part + (size_t)warp * gridDim.x + b);
          for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == 0) red[warp] = s;
        }
      }
      asm volatile(
          "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
              smem_u32(&bar)),
          "r"(parity)
          : "memory");
      parity ^= 1;
      __syncthreads();
    } else if (A.mode == 1) {
      // poll all V*n entries + NP*grid partials; up to 16 entries per thread in flight
      const int tot = V * n, totp = NP * gridDim.x;
      constexpr int U = 16;
      for (int base = 0; base < tot + totp; base += U * T) {
        bool need[U];
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) need[u] = base + u * T + (int)threadIdx.x < tot + totp;
        for (;;) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int e = base + u * T + threadIdx.x;
            if (need[u]) r[u] = e < tot ? ld_ll(llvec + e) : ld_ll(llpart + (e - tot));
          }
          bool any = false;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (!need[u]) continue;
            if (r[u].y == f && r[u].w == f) {
              const int e = base + u * T + threadIdx.x;
              if (e < tot) sm[e] = ll_val(r[u]);
              else acc += ll_val(r[u]) * 1e-300;
              need[u] = false;
            } else {
              any = true;
            }
          }
          if (!any) break;
        }
      }
      __syncthreads();
    } else {
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(A.flags + blockIdx.x), "r"(f) : "memory");
      }
      if (threadIdx.x < gridDim.x) {
        unsigned g;
        do {
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(A.flags + threadIdx.x) : "memory");
        } while ((int)(g - f) < 0);
        __threadfence();
      }
      __syncthreads();
      for (int e = threadIdx.x; e < V * n; e += T) sm[e] = __ldcg(A.vec + e);
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      if (warp < NP) {
        double s = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) s += __ldcg(A.part + (size_t)warp * gridDim.x + b);
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red[warp] = s;
      }
      __syncthreads();
    }
    acc += sm[threadIdx.x % n];
  }
  if (acc == 1.2345) A.out[0] = acc;
}

__global__ void chase(const unsigned* nxt, int steps, int vol, unsigned* out, long long* cyc) {
  unsigned j = 0;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    if (vol) asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(j) : "l"(nxt + j) : "memory");
    else j = __ldcg(nxt + j);
  }
  long long t1 = clock64();
  out[0] = j;
  cyc[0] = t1 - t0;
}

int main() {
  {
    const int N = 1 << 22;  // 16 MB of u32, L2-resident
    unsigned* h = new unsigned[N];
    unsigned long long x = 88172645463325252ull;
    for (int i = 0; i < N; ++i) h[i] = 0;
    // random cycle with stride
    for (int i = 0; i < N; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (unsigned)(x % N) & ~31u; }
    unsigned *d, *o; long long* c;
    cudaMalloc(&d, N * 4); cudaMalloc(&o, 4); cudaMalloc(&c, 8);
    cudaMemcpy(d, h, N * 4, cudaMemcpyHostToDevice);
    for (int vol = 0; vol < 2; ++vol) {
      chase<<<1, 1>>>(d, 2000, vol, o, c);
      chase<<<1, 1>>>(d, 2000, vol, o, c);
      long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
      int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      printf("L2 chase (%s): %.0f cycles/load = %.0f ns at %d MHz\n", vol ? "volatile" : "ld.cg", cy / 2000.0, cy / 2000.0 / (clk / 1e6), clk / 1000);
    }
  }
  const int G = 148;
  double *vec, *part, *out;
  uint4 *llvec, *llpart;
  unsigned* flags;
  cudaMalloc(&vec, 3 * 2048 * 8);
  cudaMalloc(&part, 16 * G * 8);
  cudaMalloc(&llvec, 2 * 3 * 2048 * 16);
  cudaMalloc(&llpart, 2 * 16 * G * 16 + 16 * G * 16);
  cudaMalloc(&flags, G * 4);
  cudaMemset(llvec, 0, 2 * 3 * 2048 * 16);
  cudaMemset(llpart, 0, 2 * 16 * G * 16);
  cudaMemset(flags, 0, G * 4);
  cudaMalloc(&out, 8);
  const size_t smem = 3 * 2048 * 8;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  unsigned epoch = 1;
  const char* names[] = {"grid.sync+TMA", "LL poll", "flag+loads", "sync only", "stores+sync", "+partials", "+TMA only", "stores+fence", "LL part+fence", "LL part nofence", "rel/acq flag", "red.rel bar+ldcg", "LL+fence batched"};
  for (int n : {1000, 2000})
    for (int V : {3})
      for (int NP : {3, 14})
        for (int mode : {11, 12}) {
          float best = 1e9;
          for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(flags, 0, G * 4);
            Args A{n, V, NP, 400, mode, vec, part, llvec, llpart, flags, out, epoch};
            epoch += 400;
            void* args[] = {&A};
            cudaEventRecord(a);
            cudaError_t e0 = cudaLaunchCooperativeKernel((void*)probe, G, T, args, smem, 0);
            cudaEventRecord(b);
            cudaError_t e = cudaEventSynchronize(b);
            if (e0 != cudaSuccess || e != cudaSuccess) {
              printf("error %s %s\n", cudaGetErrorString(e0), cudaGetErrorString(e));
              return 1;
            }
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
          }
          printf("n=%d V=%d NP=%2d %-14s %6.2f us/phase\n", n, V, NP, names[mode], best * 1e3 / 400);
        }
  return 0;
}
