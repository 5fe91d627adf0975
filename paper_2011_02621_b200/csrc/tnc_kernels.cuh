// SIMT kernels of libtnc: projection gather, generic tiled contraction,
// bandwidth ("skinny") contraction, slice sum.
#pragma once
#include "tnc_common.cuh"

namespace tnc {

// ---------------------------------------------------------------------------
// Projection / slicing gather (network.py:321-335 with product-state bras,
// network.py:446-453 cut restriction): out[z][i] = site(z)[off(i)].
// ---------------------------------------------------------------------------
template <typename R>
__global__ void __launch_bounds__(256)
k_project(const __grid_constant__ tnc_project_desc d, int64_t elems) {
  using C = typename cplx<R>::T;
  const C* src = reinterpret_cast<const C*>(d.site.ptr);
  C* out = reinterpret_cast<C*>(d.out);
  const int64_t total = d.Z * elems;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = g / elems;
    int64_t i = g - z * elems;
    int64_t off = site_offset(d.site, z, d.slices_per_b, d.s0);
    for (int j = d.nd - 1; j >= 0; --j) {
      const int64_t q = i / d.dim[j];
      off += (i - q * d.dim[j]) * d.src_stride[j];
      i = q;
    }
    C v = src[off];
    if (d.conj) v = cconj(v);
    out[z * d.out_zstride + (g - z * elems)] = v;
  }
}

// mixed-radix row decomposition -> (acc offset, out offset)
// Mixed-radix row decomposition.  Leg extents are products of bond
// dimensions, almost always powers of two: those legs take a mask and a shift
// (the branch is warp-uniform, extents come from the descriptor) instead of a
// 64-bit division, which dominated the SIMT steps' instruction count.
__device__ __forceinline__ void row_offsets(const tnc_step_desc& d, int64_t f, int64_t& oa, int64_t& oc) {
  oa = 0; oc = 0;
  for (int j = d.nf - 1; j >= 0; --j) {
    const int64_t dm = d.f_dim[j];
    int64_t r;
    if ((dm & (dm - 1)) == 0) {
      r = f & (dm - 1);
      f >>= (__ffsll(dm) - 1);
    } else {
      const int64_t q = f / dm;
      r = f - q * dm;
      f = q;
    }
    oa += r * d.f_astride[j];
    oc += r * d.f_cstride[j];
  }
}

// ---------------------------------------------------------------------------
// Generic tiled contraction: any leg layout, any K and N.  Register-blocked
// SIMT complex GEMM whose operand/result addresses come from the step's
// stride tables (correctness reference kernel and catch-all).
// ---------------------------------------------------------------------------
template <typename R, int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
k_step_generic(const __grid_constant__ tnc_step_desc d, int64_t tiles_m, int64_t tiles_n) {
  using C = typename cplx<R>::T;
  constexpr int TX = BN / TN, TY = BM / TM, NT = TX * TY;
  __shared__ C As[BK][BM + 1];
  __shared__ C Bs[BK][BN + 1];
  __shared__ int64_t rowA[BM], rowC[BM];

  int64_t t = blockIdx.x;
  const int64_t tiles = tiles_m * tiles_n;
  const int64_t z = t / tiles;
  t -= z * tiles;
  const int64_t m0 = (t / tiles_n) * BM, n0 = (t % tiles_n) * BN;
  const C* A = reinterpret_cast<const C*>(d.acc) + z * d.acc_zstride;
  const C* B = reinterpret_cast<const C*>(d.site.ptr) + site_offset(d.site, z, d.slices_per_b, d.s0);
  C* Co = reinterpret_cast<C*>(d.out) + z * d.out_zstride;

  for (int i = threadIdx.x; i < BM; i += NT) {
    int64_t oa = 0, oc = 0;
    if (m0 + i < d.M) row_offsets(d, m0 + i, oa, oc);
    rowA[i] = oa;
    rowC[i] = oc;
  }
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  C acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = czero<R>();
  __syncthreads();

  for (int64_t k0 = 0; k0 < d.K; k0 += BK) {
    for (int e = threadIdx.x; e < BM * BK; e += NT) {
      const int i = e / BK, kk = e % BK;
      const int64_t k = k0 + kk;
      C v = czero<R>();
      if (m0 + i < d.M && k < d.K) v = A[rowA[i] + d.a_koff[k]];
      As[kk][i] = v;
    }
    for (int e = threadIdx.x; e < BK * BN; e += NT) {
      const int kk = e / BN, j = e % BN;
      const int64_t k = k0 + kk, n = n0 + j;
      C v = czero<R>();
      if (k < d.K && n < d.N) {
        v = B[d.b_koff[k] + d.b_noff[n]];
        if (d.conj_b) v = cconj(v);
      }
      Bs[kk][j] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < BK; ++kk) {
      C a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx + j * TX];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) cfma(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int r = ty * TM + i;
    if (m0 + r >= d.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t n = n0 + tx + j * TX;
      if (n < d.N) Co[rowC[r] + d.c_noff[n]] = acc[i][j];
    }
  }
}

// ---------------------------------------------------------------------------
// Skinny contraction, accumulator-resident (N <= NMAX <= 32): one thread per
// row of the row-contiguous accumulator; the row is streamed through
// registers in chunks, the dense [K][N] site block is read as warp-uniform
// broadcasts, the N results stay in registers.  HBM-bound for K*N <~ 256.
// ---------------------------------------------------------------------------
template <typename R, int NMAX>
__global__ void __launch_bounds__(128)
k_step_skinny_acc(const __grid_constant__ tnc_step_desc d) {
  using C = typename cplx<R>::T;
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= d.Z * d.M) return;
  const int64_t z = g / d.M, f = g - z * d.M;
  const int K = (int)d.K, N = (int)d.N;
  const C* __restrict__ a = reinterpret_cast<const C*>(d.acc) + z * d.acc_zstride + f * d.K;
  const C* __restrict__ S = reinterpret_cast<const C*>(d.site.ptr) + site_offset(d.site, z, d.slices_per_b, d.s0);
  C acc[NMAX];
#pragma unroll
  for (int n = 0; n < NMAX; ++n) acc[n] = czero<R>();
  constexpr int KC = 8;
  int k0 = 0;
  for (; k0 + KC <= K; k0 += KC) {
    C av[KC];
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) av[kk] = __ldg(a + k0 + kk);
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      const C* srow = S + (int64_t)(k0 + kk) * N;
#pragma unroll
      for (int n = 0; n < NMAX; ++n)
        if (n < N) cfma(acc[n], av[kk], __ldg(srow + n));
    }
  }
  for (; k0 < K; ++k0) {
    const C av = __ldg(a + k0);
    const C* srow = S + (int64_t)k0 * N;
#pragma unroll
    for (int n = 0; n < NMAX; ++n)
      if (n < N) cfma(acc[n], av, __ldg(srow + n));
  }
  C* o = reinterpret_cast<C*>(d.out) + z * d.out_zstride;
  if (d.c_rows_contig) {
    o += f * d.N;
#pragma unroll
    for (int n = 0; n < NMAX; ++n)
      if (n < N) o[n] = acc[n];
  } else {
    int64_t oa, oc;
    row_offsets(d, f, oa, oc);
#pragma unroll
    for (int n = 0; n < NMAX; ++n)
      if (n < N) o[oc + d.c_noff[n]] = acc[n];
  }
}

// ---------------------------------------------------------------------------
// Skinny contraction, row-resident (K <= KMAX <= 32, any N): the thread keeps
// its whole accumulator row in registers and emits the N outputs in chunks.
// ---------------------------------------------------------------------------
template <typename R, int KMAX>
__global__ void __launch_bounds__(128)
k_step_skinny_row(const __grid_constant__ tnc_step_desc d) {
  using C = typename cplx<R>::T;
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= d.Z * d.M) return;
  const int64_t z = g / d.M, f = g - z * d.M;
  const int K = (int)d.K, N = (int)d.N;
  const C* __restrict__ a = reinterpret_cast<const C*>(d.acc) + z * d.acc_zstride + f * d.K;
  const C* __restrict__ S = reinterpret_cast<const C*>(d.site.ptr) + site_offset(d.site, z, d.slices_per_b, d.s0);
  C av[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) av[k] = (k < K) ? __ldg(a + k) : czero<R>();
  C* o = reinterpret_cast<C*>(d.out) + z * d.out_zstride;
  int64_t oc = f * d.N;
  if (!d.c_rows_contig) {
    int64_t oa;
    row_offsets(d, f, oa, oc);
  }
  constexpr int NC = 8;
  for (int n0 = 0; n0 < N; n0 += NC) {
    C acc[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[j] = czero<R>();
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      if (k < K) {
        const C* srow = S + (int64_t)k * N + n0;
#pragma unroll
        for (int j = 0; j < NC; ++j)
          if (n0 + j < N) cfma(acc[j], av[k], __ldg(srow + j));
      }
    }
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int n = n0 + j;
      if (n < N) o[d.c_rows_contig ? oc + n : oc + d.c_noff[n]] = acc[j];
    }
  }
}

// ---------------------------------------------------------------------------
// Slice sum (network.py:546-551): one warp per bitstring, fixed summation
// order (lane-strided partial sums + xor-shuffle tree) -> deterministic.
// ---------------------------------------------------------------------------
template <typename R>
__global__ void __launch_bounds__(256)
k_slice_sum(const __grid_constant__ tnc_slice_sum_desc d) {
  using C = typename cplx<R>::T;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= d.B) return;
  const C* x = reinterpret_cast<const C*>(d.x);
  C s = czero<R>();
  for (int64_t j = lane; j < d.slices_per_b; j += 32) s = cadd(s, x[(warp * d.slices_per_b + j) * d.x_zstride]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
    s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
  }
  if (lane == 0) {
    C* amp = reinterpret_cast<C*>(d.amp);
    amp[warp] = d.accumulate ? cadd(amp[warp], s) : s;
  }
}

// ---------------------------------------------------------------------------
// Few-row steps (Z*M small, e.g. the first and last steps of a path, where M
// is tiny and N or K large): one thread per result element, so the launch
// still spans the GPU.  The row of acc is a warp-wide broadcast, the site
// column is read coalesced across consecutive n.
// ---------------------------------------------------------------------------
template <typename R>
__global__ void __launch_bounds__(256)
k_step_cols(const __grid_constant__ tnc_step_desc d) {
  using C = typename cplx<R>::T;
  const int64_t total = d.Z * d.M * d.N;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t zf = g / d.N, n = g - zf * d.N;
    const int64_t z = zf / d.M, f = zf - z * d.M;
    const C* a = reinterpret_cast<const C*>(d.acc) + z * d.acc_zstride + f * d.K;
    const C* S = reinterpret_cast<const C*>(d.site.ptr) + site_offset(d.site, z, d.slices_per_b, d.s0) + n;
    C acc = czero<R>();
    for (int64_t k = 0; k < d.K; ++k) {
      C b = __ldg(S + k * d.N);
      if (d.conj_b) b = cconj(b);
      cfma(acc, __ldg(a + k), b);
    }
    C* o = reinterpret_cast<C*>(d.out) + z * d.out_zstride;
    if (d.c_rows_contig) {
      o[f * d.N + n] = acc;
    } else {
      int64_t oa, oc;
      row_offsets(d, f, oa, oc);
      o[oc + d.c_noff[n]] = acc;
    }
  }
}

// Few rows and long K (the last steps of a path: M = 1..256, K = 2^13): one
// warp per result element, lanes striding over K (coalesced acc row reads),
// shuffle reduction.
template <typename R>
__global__ void __launch_bounds__(256)
k_step_dot(const __grid_constant__ tnc_step_desc d) {
  using C = typename cplx<R>::T;
  const int lane = threadIdx.x & 31;
  const int64_t total = d.Z * d.M * d.N;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); g < total; g += wstride) {
    const int64_t zf = g / d.N, n = g - zf * d.N;
    const int64_t z = zf / d.M, f = zf - z * d.M;
    const C* a = reinterpret_cast<const C*>(d.acc) + z * d.acc_zstride + f * d.K;
    const C* S = reinterpret_cast<const C*>(d.site.ptr) + site_offset(d.site, z, d.slices_per_b, d.s0) + n;
    C acc = czero<R>();
    for (int64_t k = lane; k < d.K; k += 32) {
      C b = __ldg(S + k * d.N);
      if (d.conj_b) b = cconj(b);
      cfma(acc, __ldg(a + k), b);
    }
    for (int o = 16; o; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) {
      C* o = reinterpret_cast<C*>(d.out) + z * d.out_zstride;
      if (d.c_rows_contig) {
        o[f * d.N + n] = acc;
      } else {
        int64_t oa, oc;
        row_offsets(d, f, oa, oc);
        o[oc + d.c_noff[n]] = acc;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Split-K step for few rows and a long contracted extent (path ends: e.g.
// M = 1024, K = 32768, N = 64): every CTA computes a BM x BN register-blocked
// partial product over one K range of rows-contiguous A and a dense site
// block into a workspace W[split][row][n]; k_splitk_reduce sums the splits
// in a fixed order (bit-reproducible) and scatters through the row map.
// ---------------------------------------------------------------------------
template <typename R, int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
k_step_splitk(const __grid_constant__ tnc_step_desc d, int64_t tiles_n, int64_t ks,
              typename cplx<R>::T* __restrict__ W) {
  using C = typename cplx<R>::T;
  constexpr int TX = BN / TN, TY = BM / TM, NT = TX * TY;
  __shared__ C As[BK][BM + 1];
  __shared__ C Bs[BK][BN + 1];
  const int64_t rows = d.Z * d.M;
  const int64_t r0 = (blockIdx.x / tiles_n) * BM, n0 = (blockIdx.x % tiles_n) * BN;
  const int64_t k_begin = blockIdx.y * ks, k_end = min(k_begin + ks, d.K);
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  C acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = czero<R>();
  for (int64_t k0 = k_begin; k0 < k_end; k0 += BK) {
    for (int e = threadIdx.x; e < BM * BK; e += NT) {
      const int i = e / BK, kk = e % BK;              // consecutive threads: consecutive k of one row
      const int64_t row = r0 + i, k = k0 + kk;
      C v = czero<R>();
      if (row < rows && k < k_end) {
        const int64_t z = row / d.M, f = row - z * d.M;
        v = reinterpret_cast<const C*>(d.acc)[z * d.acc_zstride + f * d.K + k];
      }
      As[kk][i] = v;
    }
    for (int e = threadIdx.x; e < BK * BN; e += NT) {
      const int kk = e / BN, j = e % BN;
      const int64_t k = k0 + kk, n = n0 + j;
      C v = czero<R>();
      if (k < k_end && n < d.N) {
        // one site block per z: the tile's rows may span z (same site unless
        // variants / slices differ, handled by the caller: Z * M rows share it)
        v = reinterpret_cast<const C*>(d.site.ptr)[site_offset(d.site, r0 / d.M, d.slices_per_b, d.s0) + k * d.N + n];
        if (d.conj_b) v = cconj(v);
      }
      Bs[kk][j] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < BK; ++kk) {
      C a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx + j * TX];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) cfma(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
  C* Wp = W + (int64_t)blockIdx.y * rows * d.N;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t row = r0 + ty * TM + i;
    if (row >= rows) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t n = n0 + tx + j * TX;
      if (n < d.N) Wp[row * d.N + n] = acc[i][j];
    }
  }
}

template <typename R>
__global__ void __launch_bounds__(256)
k_splitk_reduce(const __grid_constant__ tnc_step_desc d, int64_t splits, const typename cplx<R>::T* __restrict__ W) {
  using C = typename cplx<R>::T;
  const int64_t rows = d.Z * d.M, total = rows * d.N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    C v = czero<R>();
    for (int64_t s = 0; s < splits; ++s) {
      const C w = W[s * total + e];
      v.x += w.x;
      v.y += w.y;
    }
    const int64_t row = e / d.N, n = e - row * d.N;
    const int64_t z = row / d.M, f = row - z * d.M;
    C* o = reinterpret_cast<C*>(d.out) + z * d.out_zstride;
    if (d.c_rows_contig) {
      o[f * d.N + n] = v;
    } else {
      int64_t oa, oc;
      row_offsets(d, f, oa, oc);
      o[oc + d.c_noff[n]] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// Warp-cooperative skinny step (complex64, K = 2L in {2..64}, N <= NN <= 4):
// L lanes share one acc row, each loading 16 contiguous bytes (two complex),
// so every warp load is a coalesced 512-byte stream of 32/L whole rows; the
// N partial sums are reduced across the L lanes with xor shuffles.  UNR row
// groups per iteration keep several loads in flight per warp.
// ---------------------------------------------------------------------------
// 32-bit mixed-radix row decomposition (all extents and offsets < 2^31)
__device__ __forceinline__ uint32_t row_cout32(const tnc_step_desc& d, uint32_t f) {
  uint32_t oc = 0;
  for (int j = d.nf - 1; j >= 0; --j) {
    const uint32_t dm = (uint32_t)d.f_dim[j];
    if ((dm & (dm - 1)) == 0) {                  // power-of-two leg: mask + shift
      oc += (f & (dm - 1)) * (uint32_t)d.f_cstride[j];
      f >>= (__ffs(dm) - 1);
    } else {
      const uint32_t q = f / dm;
      oc += (f - q * dm) * (uint32_t)d.f_cstride[j];
      f = q;
    }
  }
  return oc;
}

template <int L, int NN>
__global__ void __launch_bounds__(256)
k_step_warp(const __grid_constant__ tnc_step_desc d) {
  constexpr int RP = 32 / L;                 // rows per warp pass
  constexpr int UNR = NN >= 8 ? 2 : 4;       // passes in flight per warp
  constexpr int OWN = NN >= L ? NN / L : 1;  // results owned by a lane after the reduction
  const int lane = threadIdx.x & 31;
  const int j = lane % L;                    // complex pair index within the row
  const int rg = lane / L;                   // row within the pass
  const int N = (int)d.N;
  const uint32_t M = (uint32_t)d.M;
  const uint32_t wpb = blockDim.x >> 5;
  const uint32_t wstride = gridDim.x * wpb * RP * UNR;
  const uint32_t wbase = (blockIdx.x * wpb + (threadIdx.x >> 5)) * RP * UNR;
  // results n0 .. n0 + OWN - 1 of each row end up in this lane
  const int n0 = NN >= L ? j * OWN : j;
  float vmax = 0.f;
  for (int64_t z = blockIdx.y; z < d.Z; z += gridDim.y) {
    const float4* Az = reinterpret_cast<const float4*>(reinterpret_cast<const float2*>(d.acc) + z * d.acc_zstride);
    float2* Oz = reinterpret_cast<float2*>(d.out) + z * d.out_zstride;
    const float2* S = reinterpret_cast<const float2*>(d.site.ptr) + site_offset(d.site, z, d.slices_per_b, d.s0) +
                      (int64_t)(2 * j) * N;
    float2 s0[NN], s1[NN];                   // this lane's two site rows, for the whole z
#pragma unroll
    for (int n = 0; n < NN; ++n) {
      s0[n] = n < N ? __ldg(S + n) : make_float2(0.f, 0.f);
      s1[n] = n < N ? __ldg(S + N + n) : make_float2(0.f, 0.f);
    }
    for (uint32_t base = wbase; base < M; base += wstride) {
      float4 av[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const uint32_t f = base + u * RP + rg;
        av[u] = f < M ? __ldg(Az + (size_t)f * L + j) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        float2 v[NN];
#pragma unroll
        for (int n = 0; n < NN; ++n) {
          v[n] = make_float2(0.f, 0.f);
          cfma(v[n], make_float2(av[u].x, av[u].y), s0[n]);
          cfma(v[n], make_float2(av[u].z, av[u].w), s1[n]);
        }
        if constexpr (NN >= L) {
          // reduce-scatter: each halving step keeps the half selected by one
          // bit of j (most significant first), so lane j ends with n in
          // [j*OWN, (j+1)*OWN)
          int cnt = NN;
#pragma unroll
          for (int off = L / 2; off > 0; off >>= 1) {
            const bool up = (j & off) != 0;
            cnt >>= 1;
#pragma unroll
            for (int i = 0; i < NN / 2; ++i) {
              if (i < cnt) {
                const float2 lo = v[i], hi = v[i + cnt];
                const float2 send = up ? lo : hi;
                float2 recv;
                recv.x = __shfl_xor_sync(0xffffffffu, send.x, off);
                recv.y = __shfl_xor_sync(0xffffffffu, send.y, off);
                const float2 keep = up ? hi : lo;
                v[i] = make_float2(keep.x + recv.x, keep.y + recv.y);
              }
            }
          }
        } else {
#pragma unroll
          for (int off = L / 2; off > 0; off >>= 1) {
#pragma unroll
            for (int n = 0; n < NN; ++n) {
              v[n].x += __shfl_xor_sync(0xffffffffu, v[n].x, off);
              v[n].y += __shfl_xor_sync(0xffffffffu, v[n].y, off);
            }
          }
          // lane j keeps result j
#pragma unroll
          for (int n = 1; n < NN; ++n)
            if (j == n) v[0] = v[n];
        }
        const uint32_t f = base + u * RP + rg;
        if (f < M && n0 < N) {
          if (d.amax_out) {
#pragma unroll
            for (int i = 0; i < OWN; ++i)
              if (n0 + i < N) vmax = fmaxf(vmax, fmaxf(fabsf(v[i].x), fabsf(v[i].y)));
          }
          if (d.c_rows_contig || d.c_n_contig) {
            // the lane's OWN results are consecutive in the row: 16-byte stores
            float2* o = Oz + (d.c_rows_contig ? (size_t)f * N : (size_t)row_cout32(d, f)) + n0;
            if constexpr (OWN >= 2) {
              if ((OWN & 1) == 0 && n0 + OWN <= N) {
#pragma unroll
                for (int i = 0; i < OWN; i += 2)
                  *reinterpret_cast<float4*>(o + i) = make_float4(v[i].x, v[i].y, v[i + 1].x, v[i + 1].y);
                continue;
              }
            }
#pragma unroll
            for (int i = 0; i < OWN; ++i)
              if (n0 + i < N) o[i] = v[i];
          } else {
            const uint32_t oc = row_cout32(d, f);
#pragma unroll
            for (int i = 0; i < OWN; ++i)
              if (n0 + i < N) Oz[oc + (uint32_t)d.c_noff[n0 + i]] = v[i];
          }
        }
      }
    }
    if (d.amax_out) {                              // max |re|, |im| of out[z] for the next fp16-split GEMM step
      for (int o = 16; o; o >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
      if (lane == 0 && vmax > 0.f) atomicMax(reinterpret_cast<unsigned int*>(d.amax_out) + z, __float_as_uint(vmax));
      vmax = 0.f;
    }
  }
}

// amax[z] = max |re|, |im| over x[z * zstride + i], i < count (atomicMax on
// the float bits: non-negative floats order like their bit patterns)
__global__ void k_amax(const float2* __restrict__ x, int64_t Z, int64_t zstride, int64_t count, float* amax) {
  for (int64_t z = blockIdx.y; z < Z; z += gridDim.y) {
    const float2* xz = x + z * zstride;
    float m = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
      const float2 v = __ldg(xz + i);
      m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
    }
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(reinterpret_cast<unsigned int*>(amax) + z, __float_as_uint(m));
  }
}

}  // namespace tnc

