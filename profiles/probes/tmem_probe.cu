// TMEM as a resident store for Gram rows: read throughput of
// tcgen05.ld.32x32b.x32 by 16 warps of one CTA per SM (each warp streams its
// lane quarter's 128-column block), vs the same bytes from L2.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void tm_ld32(uint32_t addr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
}
__global__ void __launch_bounds__(512, 1) k(int reps, double* out, long long* cyc) {
  __shared__ uint32_t taddr;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr;
  // warp w: lanes 32*(w%4).., columns 128*(w/4)..+128
  const uint32_t my = base + ((uint32_t)(32 * (warp & 3)) << 16) + 128 * (warp >> 2);
  double acc = 0.0;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t v[32];
      tm_ld32(my + 32 * c, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int q = 0; q < 32; q += 2) acc += __hiloint2double(v[q + 1], v[q]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * 512 + threadIdx.x] = acc;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 148 * 512 * 8); cudaMalloc(&c, 148 * 8);
  for (int rep = 0; rep < 2; ++rep) {
    k<<<148, 512>>>(100, o, c);
    cudaError_t e = cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    // bytes per CTA per rep: 16 warps x 32 lanes x 128 cols x 4 B = 256 KB
    printf("%s: %lld cycles for 100 x 256 KB -> %.1f B/cycle/SM (%.2f us per 256 KB at 1.965 GHz)\n",
           cudaGetErrorString(e), h, 100.0 * 262144 / h, h / 100.0 / 1965.0);
  }
}
