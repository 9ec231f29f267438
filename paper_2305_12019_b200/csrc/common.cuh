// Common device helpers for the gdwd B200 kernels.
//
// Everything here is fp64.  Reductions are deterministic: a fixed
// warp-shuffle tree, then a fixed-order sum over warps, then (across CTAs) a
// fixed-order sum over per-CTA partials performed by whichever CTA arrives
// last at a ticket (the order of the final sum never depends on which CTA
// that is).  SPEC.md:103,109 requires reproducible reductions.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define GDWD_DEV __device__ __forceinline__

namespace gdwd {

// True the first time it is called for the current device with this flag
// word (one bit per device): per-device one-time setup such as
// cudaFuncSetAttribute, which applies to the current device only.
inline bool once_per_device(unsigned long long& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (__atomic_fetch_or(&mask, bit, __ATOMIC_RELAXED) & bit) return false;
  return true;
}

constexpr int WARP = 32;

// ---------------------------------------------------------------------------
// numpy-compatible elementwise helpers.  numpy's ``power`` with a scalar
// exponent takes exact fast paths for 2, 0.5, -1 and 1 (square, sqrt,
// reciprocal, copy); everything else goes to a libm/SIMD pow that is within
// ~1 ulp (on the build host it differs from the correctly rounded value in
// ~5% of cases).  Mirroring the fast paths keeps those exponents bitwise
// identical to the reference.  Other small integer exponents (the Newton
// prox's s^-(q+1) for integer q) are evaluated as a double-double power
// rounded once -- the correctly rounded value in every case tested against
// exact rational arithmetic -- at the cost of one IEEE division instead of a
// CUDA pow (<= 2 ulp, an order of magnitude longer dependency chain).
// ---------------------------------------------------------------------------
GDWD_DEV double pow_int_dd(double x, int m) {  // x^m, 2 <= |m| <= 16
  const int a = m < 0 ? -m : m;
  double hi = x, lo = 0.0;
  for (int i = 1; i < a; ++i) {  // (hi + lo) * x as a double-double
    const double p = __dmul_rn(hi, x);
    double e = __fma_rn(hi, x, -p);
    e = __fma_rn(lo, x, e);
    const double h = __dadd_rn(p, e);
    lo = __dsub_rn(e, __dsub_rn(h, p));
    hi = h;
  }
  if (m > 0) return hi;
  // 1 / (hi + lo): IEEE quotient of hi, then one correction step
  const double q = __ddiv_rn(1.0, hi);
  double r = __fma_rn(-q, hi, 1.0);
  r = __fma_rn(-q, lo, r);
  return __fma_rn(q, r, q);
}

GDWD_DEV double np_pow(double x, double e) {
  if (e == 2.0) return __dmul_rn(x, x);
  if (e == 0.5) return __dsqrt_rn(x);
  if (e == 1.0) return x;
  if (e == -1.0) return __ddiv_rn(1.0, x);
  if (e == 0.0) return 1.0;
  const double ae = fabs(e);
  // x > 0 with x^|e| and its error terms far from overflow / underflow
  // binary exponent from the bits (== ilogb for normal x; a subnormal reads
  // -1023 and fails the bound exactly as ilogb's <= -1023 would)
  const int ex = (int)((__double_as_longlong(x) >> 52) & 0x7ff) - 1023;
  if (ae <= 16.0 && ae == rint(ae) && x > 0.0 && isfinite(x) && (abs(ex) + 1) * (int)ae < 960)
    return pow_int_dd(x, (int)e);
  return pow(x, e);
}

// ---------------------------------------------------------------------------
// Reductions
// ---------------------------------------------------------------------------
template <int K>
GDWD_DEV void warp_sum(double (&v)[K]) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
  }
}

// Block-wide sum of K values; result valid in warp 0 (returned in v).
// ``scratch`` must hold (blockDim.x/32)*K doubles.
template <int K>
GDWD_DEV void block_sum(double (&v)[K], double* scratch) {
  warp_sum<K>(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) scratch[wid * K + k] = v[k];
  }
  __syncthreads();
  if (wid == 0) {  // fixed shuffle tree over the per-warp sums
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = lane < nw ? scratch[lane * K + k] : 0.0;
    warp_sum<K>(v);
  }
  __syncthreads();
}

// Ticket: returns true in exactly one CTA (the last of ``count`` arrivals),
// after a fence that makes every earlier CTA's global writes visible.  The
// counter is reset so the same slot can be reused (CUDA-graph replay).
GDWD_DEV bool last_arrival(unsigned int* ticket, unsigned int count) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned int t = atomicAdd(ticket, 1u);
    s_last = (t == count - 1);
    if (s_last) *ticket = 0u;
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

// load that bypasses L1 (data written by other CTAs of the same grid)
GDWD_DEV double ld_cg(const double* p) { return __ldcg(p); }

// Fixed-order sum of partials[p*stride + k], p in [0, np), for k < K, done by
// thread 0.  Used by the ticket winner.
template <int K>
GDWD_DEV void sum_partials(const double* partials, int np, double (&out)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = 0.0;
  for (int p = 0; p < np; ++p) {
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] += ld_cg(partials + (size_t)p * K + k);
  }
}

// Block-cooperative fixed-order sum of partials[p*K + k], p in [0, np): thread
// t sums p = t, t+blockDim, ... in increasing order, then a fixed tree.  All
// threads must call; the result is valid in thread 0.
template <int K>
GDWD_DEV void block_sum_partials(const double* partials, int np, double (&out)[K], double* scratch) {
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = 0.0;
  for (int p = threadIdx.x; p < np; p += blockDim.x) {
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] += ld_cg(partials + (size_t)p * K + k);
  }
  block_sum<K>(out, scratch);
}

// ---------------------------------------------------------------------------
// Bulk asynchronous copies (TMA engine, non-tensor form) with mbarrier
// completion: one thread arms the barrier with the byte count and issues the
// copies; every thread waits on the barrier's phase parity.
// ---------------------------------------------------------------------------
GDWD_DEV unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

GDWD_DEV void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
GDWD_DEV void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// global -> shared, `bytes` a multiple of 16, both addresses 16-byte aligned
GDWD_DEV void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
GDWD_DEV void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// order this thread's view of generic-proxy global writes (made visible by a
// preceding grid barrier) before its async-proxy (bulk copy) reads
GDWD_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// 128-bit streaming load (no L1 allocation): X is read once per pass.
GDWD_DEV double2 ld_stream2(const double* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p));
  return r;
}

}  // namespace gdwd
