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
