// Fused permute + contract kernel for pairwise steps whose contracted legs sit
// anywhere in the accumulator (tensor.py:103 contract_pair semantics; the
// BASELINE configs[1] sweep, where the leg order is a random permutation).
#pragma once
#include "tnc_common.cuh"

namespace tnc {

// Tile = every value of the shared legs x the innermost legs of a: Kout
// contiguous segments of Lseg elements (one per value of the shared legs that
// lie outside the segment).  A tile holds R rows (combinations of the free
// legs inside the segment); tiles are indexed by the free legs outside it.
struct PairTile {
  int64_t U;                   // tiles per batch element
  int64_t a_zstride, b_zstride, out_zstride;
  int32_t nfo;                 // outer free legs
  int32_t conj_b;
  int64_t fo_dim[TNC_MAX_LEGS], fo_stride[TNC_MAX_LEGS];
  int64_t Kout, Lseg, R, K, N;
  const int64_t* segoff;       // [Kout] offset of segment j relative to the tile base
  const int32_t* rowoff;       // [R]    offset of row r inside a segment
  const int32_t* koff;         // [K]    seg(k) * Lseg + offset of k inside its segment
  const int64_t* b_koff;       // [K]
  const int64_t* b_noff;       // [N]
  int32_t vec16;               // segment base offsets and Lseg allow 16-byte copies
  int32_t _pad;
};

template <typename C>
__device__ __forceinline__ void stage_tile(const PairTile& p, const C* __restrict__ A, int64_t base, C* tile) {
  if (sizeof(C) == 8 && p.vec16) {
    const int64_t halves = p.Lseg >> 1;
    const int64_t total = p.Kout * halves;
    for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
      const int64_t s = e / halves, i = e - s * halves;
      const float4 v = __ldg(reinterpret_cast<const float4*>(A + base + p.segoff[s]) + i);
      reinterpret_cast<float4*>(tile + s * p.Lseg)[i] = v;
    }
  } else {
    const int64_t total = p.Kout * p.Lseg;
    for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
      const int64_t s = e / p.Lseg, i = e - s * p.Lseg;
      tile[e] = __ldg(A + base + p.segoff[s] + i);
    }
  }
}

template <typename C>
__device__ __forceinline__ void stage_site(const PairTile& p, const C* __restrict__ Bz, C* S, int32_t* koff_s,
                                           const int64_t z) {
  for (int64_t e = threadIdx.x; e < p.K * p.N; e += blockDim.x) {
    const int64_t k = e / p.N, n = e - k * p.N;
    C v = __ldg(Bz + p.b_koff[k] + p.b_noff[n]);
    if (p.conj_b) v = cconj(v);
    S[e] = v;
  }
  for (int64_t k = threadIdx.x; k < p.K; k += blockDim.x) koff_s[k] = p.koff[k];
}

__device__ __forceinline__ int64_t tile_base(const PairTile& p, int64_t z, int64_t u) {
  int64_t base = z * p.a_zstride;
  for (int j = p.nfo - 1; j >= 0; --j) {
    const int64_t q = u / p.fo_dim[j];
    base += (u - q * p.fo_dim[j]) * p.fo_stride[j];
    u = q;
  }
  return base;
}

// N <= NMAX: accumulators of one row in registers.
template <typename R, int NMAX>
__global__ void __launch_bounds__(256)
k_pair_tiled_acc(const __grid_constant__ PairTile p, const void* __restrict__ A_, const void* __restrict__ B_,
                 void* __restrict__ O_) {
  using C = typename cplx<R>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* tile = reinterpret_cast<C*>(smem_raw);
  C* S = tile + p.Kout * p.Lseg;
  int32_t* koff_s = reinterpret_cast<int32_t*>(S + p.K * p.N);
  const int64_t z = blockIdx.x / p.U, u = blockIdx.x - z * (int64_t)p.U;
  stage_tile<C>(p, reinterpret_cast<const C*>(A_), tile_base(p, z, u), tile);
  stage_site<C>(p, reinterpret_cast<const C*>(B_) + z * p.b_zstride, S, koff_s, z);
  __syncthreads();
  const int K = (int)p.K, N = (int)p.N;
  C* O = reinterpret_cast<C*>(O_) + z * p.out_zstride + u * p.R * p.N;
  for (int64_t r = threadIdx.x; r < p.R; r += blockDim.x) {
    const C* trow = tile + p.rowoff[r];
    C acc[NMAX];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) acc[n] = czero<R>();
    for (int k = 0; k < K; ++k) {
      const C a = trow[koff_s[k]];
      const C* srow = S + k * N;
#pragma unroll
      for (int n = 0; n < NMAX; ++n)
        if (n < N) cfma(acc[n], a, srow[n]);
    }
    C* orow = O + r * N;
    if (sizeof(C) == 8 && (N & 1) == 0) {
#pragma unroll
      for (int n = 0; n < NMAX; n += 2)
        if (n < N) {
          float4 v;
          v.x = acc[n].x; v.y = acc[n].y;
          v.z = acc[n + 1 < NMAX ? n + 1 : n].x; v.w = acc[n + 1 < NMAX ? n + 1 : n].y;
          *reinterpret_cast<float4*>(orow + n) = v;
        }
    } else {
#pragma unroll
      for (int n = 0; n < NMAX; ++n)
        if (n < N) orow[n] = acc[n];
    }
  }
}

// K <= KMAX: one row's shared values in registers, outputs in chunks of 8.
template <typename R, int KMAX>
__global__ void __launch_bounds__(256)
k_pair_tiled_row(const __grid_constant__ PairTile p, const void* __restrict__ A_, const void* __restrict__ B_,
                 void* __restrict__ O_) {
  using C = typename cplx<R>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* tile = reinterpret_cast<C*>(smem_raw);
  C* S = tile + p.Kout * p.Lseg;
  int32_t* koff_s = reinterpret_cast<int32_t*>(S + p.K * p.N);
  const int64_t z = blockIdx.x / p.U, u = blockIdx.x - z * (int64_t)p.U;
  stage_tile<C>(p, reinterpret_cast<const C*>(A_), tile_base(p, z, u), tile);
  stage_site<C>(p, reinterpret_cast<const C*>(B_) + z * p.b_zstride, S, koff_s, z);
  __syncthreads();
  const int K = (int)p.K, N = (int)p.N;
  C* O = reinterpret_cast<C*>(O_) + z * p.out_zstride + u * p.R * p.N;
  for (int64_t r = threadIdx.x; r < p.R; r += blockDim.x) {
    const C* trow = tile + p.rowoff[r];
    C av[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) av[k] = (k < K) ? trow[koff_s[k]] : czero<R>();
    C* orow = O + r * N;
    for (int n0 = 0; n0 < N; n0 += 8) {
      C acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = czero<R>();
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        if (k < K) {
          const C* srow = S + k * N + n0;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (n0 + j < N) cfma(acc[j], av[k], srow[j]);
        }
      }
      if (sizeof(C) == 8 && n0 + 8 <= N && (N & 1) == 0) {
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          float4 v;
          v.x = acc[j].x; v.y = acc[j].y; v.z = acc[j + 1].x; v.w = acc[j + 1].y;
          *reinterpret_cast<float4*>(orow + n0 + j) = v;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (n0 + j < N) orow[n0 + j] = acc[j];
      }
    }
  }
}

}  // namespace tnc
