// Shared device helpers for libtnc: complex arithmetic, operand addressing.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/tnc.h"

namespace tnc {

template <typename R> struct cplx;
template <> struct cplx<float>  { using T = float2;  };
template <> struct cplx<double> { using T = double2; };

template <typename R> __device__ __forceinline__ typename cplx<R>::T czero() {
  typename cplx<R>::T v; v.x = R(0); v.y = R(0); return v;
}

// acc += a * b  (4 real FMAs)
__device__ __forceinline__ void cfma(float2& acc, const float2 a, const float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}
__device__ __forceinline__ void cfma(double2& acc, const double2 a, const double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ float2  cconj(float2 v)  { v.y = -v.y; return v; }
__device__ __forceinline__ double2 cconj(double2 v) { v.y = -v.y; return v; }
__device__ __forceinline__ float2  cadd(float2 a, float2 b)   { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

// Element offset of the site operand for batch element z (see tnc_site).
__device__ __forceinline__ int64_t site_offset(const tnc_site& s, int64_t z, int64_t spb, int64_t s0) {
  const int64_t b = z / spb;
  const int64_t sl = s0 + (z - b * spb);
  int64_t off = z * s.zstride;
  if (s.sel) off += (int64_t)s.sel[b] * s.vstride;
  for (int c = 0; c < s.ncut; ++c) off += ((sl / s.cut_div[c]) % s.cut_ext[c]) * s.cut_stride[c];
  return off;
}

}  // namespace tnc

namespace tnc {
// ---- mbarrier + bulk-copy (TMA 1D) helpers --------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// one arrival per warp (lane 0, after the warp has converged)
__device__ __forceinline__ void mbar_arrive_warp(uint64_t* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}
#ifndef TNC_MBAR_HINT
#define TNC_MBAR_HINT 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
#if TNC_MBAR_HINT
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)), "r"(phase), "r"(TNC_MBAR_HINT) : "memory");
#else
  // try_wait + nanosleep backoff: a waiting warp does not steal issue slots
  // from the working warps of its SM sub-partition
  uint32_t done = 0, ns = 8;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}" : "=r"(done) : "r"(smem_u32(bar)), "r"(phase) : "memory");
    if (done) break;
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
  }
#endif
}
// pure try_wait loop (the hardware suspends the thread inside try_wait): for
// latency-critical roles (MMA issuer, producers) where a nanosleep backoff
// would delay the wake-up
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
// Kernel attributes (cudaFuncSetAttribute) are per device context: a launch
// path sets them once per device it runs on, tracked in a per-call-site mask.
inline bool attr_needed(uint64_t done_mask, int* dev_out = nullptr) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev_out) *dev_out = dev;
  return !((done_mask >> (dev & 63)) & 1ull);
}
// Keep freed stream-ordered blocks in the device's default pool across
// synchronizations (the default release threshold returns them to the OS at
// every sync, and the next cudaMallocAsync would map memory again: ~1 ms).
inline void pool_keep() {
  static int pool_dev = -1;
  int cur = 0;
  cudaGetDevice(&cur);
  if (pool_dev == cur) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, cur) == cudaSuccess) {
    uint64_t thr = 1ull << 30;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  pool_dev = cur;
}
// generic-proxy shared-memory accesses of this thread ordered against the async proxy (TMA / bulk copies / tcgen05)
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// global -> shared bulk copy completing on `bar` (16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
}  // namespace tnc
