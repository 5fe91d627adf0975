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
  int32_t pipe;                // use the pipelined persistent kernel when alignment allows
  const int64_t* fo_lo;        // optional two-level tile base tables:
  const int64_t* fo_hi;        //   base(u) = fo_hi[u / f_plo] + fo_lo[u % f_plo]
  int64_t f_plo;
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
  if (p.fo_lo) {
    const int64_t q = u / p.f_plo;
    return base + __ldg(p.fo_hi + q) + __ldg(p.fo_lo + (u - q * p.f_plo));
  }
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
  extern __shared__ __align__(1024) unsigned char smem_raw[];
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
  extern __shared__ __align__(1024) unsigned char smem_raw[];
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

namespace tnc {

// ---------------------------------------------------------------------------
// Pipelined persistent version: each CTA walks a contiguous range of tiles;
// thread 0 streams the next tiles' K_out segments into a 2-stage ring with
// cp.async.bulk (TMA 1-D, mbarrier completion) while all threads contract the
// current tile.  Shared-k reads are lane-rotated ((k + lane) % K) and the site
// block is stored with an odd row pitch, so both smem streams are
// conflict-free for the power-of-two extents of lattice networks.
// ---------------------------------------------------------------------------
constexpr int PIPE_STAGES = 2;
// k_pair_pipe<..., PROD = true>: 8 compute warps + 1 producer warp.  Stage
// release is a per-stage "empty" mbarrier (one arrival per compute warp), so
// compute warps never wait for each other at a CTA barrier between tiles (that
// barrier was a third of the stall samples at K = 16: 10-16% faster there; at
// K <= 4 the tiles are short and the CTA-barrier version measured faster).
constexpr int PIPE_CWARPS = 8;
constexpr int PIPE_THREADS = (PIPE_CWARPS + 1) * 32;

// called by all 32 lanes of warp 0: lane 0 arms the barrier, then lane j
// issues segments j, j+32, ... (many small segments are not serialised
// behind one thread's issue loop and its segment-offset loads)
template <typename C>
__device__ __forceinline__ void issue_tile(const PairTile& p, const C* A, int64_t t, C* dst, uint64_t* bar) {
  const int lane = threadIdx.x & 31;
  const int64_t z = t / p.U, u = t - (t / p.U) * p.U;
  const int64_t base = tile_base(p, z, u);
  const uint32_t seg_bytes = (uint32_t)(p.Lseg * sizeof(C));
  if (lane == 0) mbar_expect_tx(bar, (uint32_t)(p.Kout * seg_bytes));
  __syncwarp();
  for (int64_t j = lane; j < p.Kout; j += 32) bulk_g2s(dst + j * p.Lseg, A + base + p.segoff[j], seg_bytes, bar);
}

template <typename R, int NMAX, int KMAX, bool PROD = false>
__global__ void __launch_bounds__(PROD ? PIPE_THREADS : 256, 2)
k_pair_pipe(const __grid_constant__ PairTile p, const void* __restrict__ A_, const void* __restrict__ B_,
            void* __restrict__ O_, int64_t tiles_total, int64_t tiles_per_cta) {
  using C = typename cplx<R>::T;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  C* ring = reinterpret_cast<C*>(smem_raw + 128);
  const int64_t tile_elems = p.Kout * p.Lseg;
  const int SP = (int)p.N + 1;
  C* S = ring + PIPE_STAGES * tile_elems;
  int32_t* koff_s = reinterpret_cast<int32_t*>(S + p.K * SP);
  int32_t* rowoff_s = koff_s + p.K;            // tile row offsets (a global load per row stalled on long scoreboard)
  const C* A = reinterpret_cast<const C*>(A_);
  const C* B = reinterpret_cast<const C*>(B_);
  C* O = reinterpret_cast<C*>(O_);
  const int64_t t0 = blockIdx.x * tiles_per_cta;
  const int64_t t1 = min(t0 + tiles_per_cta, tiles_total);
  if (t0 >= t1) return;
  const int K = (int)p.K, N = (int)p.N;
  const int lane = threadIdx.x & 31;
  uint64_t* empty = bars + PIPE_STAGES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < PIPE_STAGES; ++s) {
      mbar_init(&bars[s], 1);
      mbar_init(&empty[s], PIPE_CWARPS);
    }
    mbar_fence_init();
  }
  for (int k = threadIdx.x; k < K; k += blockDim.x) koff_s[k] = p.koff[k];
  for (int64_t r = threadIdx.x; r < p.R; r += blockDim.x) rowoff_s[r] = p.rowoff[r];
  __syncthreads();
  if (!PROD && threadIdx.x < 32)
    for (int s = 0; s < PIPE_STAGES && t0 + s < t1; ++s) issue_tile<C>(p, A, t0 + s, ring + s * tile_elems, &bars[s]);
  if (PROD && (threadIdx.x >> 5) == PIPE_CWARPS) {
    // producer warp: refill a stage once all compute warps released it
    for (int64_t i = 0; t0 + i < t1; ++i) {
      const int stage = (int)(i % PIPE_STAGES);
      if (i >= PIPE_STAGES) mbar_wait_spin(&empty[stage], (uint32_t)((i / PIPE_STAGES - 1) & 1));
      issue_tile<C>(p, A, t0 + i, ring + stage * tile_elems, &bars[stage]);
    }
    return;
  }
  constexpr int CT = PIPE_CWARPS * 32;   // compute threads (named barrier 1)
  int64_t cur_z = -1;
  const int rot = (K >= 8) ? lane % K : 0;   // lane-rotated start in the shared index
  for (int64_t i = 0; t0 + i < t1; ++i) {
    const int64_t t = t0 + i;
    const int stage = (int)(i % PIPE_STAGES);
    const uint32_t phase = (uint32_t)((i / PIPE_STAGES) & 1);
    const int64_t z = t / p.U, u = t - (t / p.U) * p.U;
    if (z != cur_z) {
      asm volatile("bar.sync 1, %0;" ::"n"(CT) : "memory");
      const C* Bz = B + z * p.b_zstride;
      for (int64_t e = threadIdx.x; e < p.K * p.N; e += CT) {
        const int64_t k = e / p.N, n = e - k * p.N;
        C v = __ldg(Bz + p.b_koff[k] + p.b_noff[n]);
        if (p.conj_b) v = cconj(v);
        S[k * SP + n] = v;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(CT) : "memory");
      cur_z = z;
    }
    mbar_wait_spin(&bars[stage], phase);
    const C* tile = ring + stage * tile_elems;
    C* Ot = O + z * p.out_zstride + u * p.R * p.N;
    for (int64_t r = threadIdx.x; r < p.R; r += CT) {
      const C* trow = tile + rowoff_s[r];
      C* orow = Ot + r * N;
      if constexpr (KMAX == 0) {
        // accumulator-resident: N <= NMAX outputs in registers
        C acc[NMAX];
#pragma unroll
        for (int n = 0; n < NMAX; ++n) acc[n] = czero<R>();
        int k = rot;
        for (int kk = 0; kk < K; ++kk) {
          const C a = trow[koff_s[k]];
          const C* srow = S + k * SP;
#pragma unroll
          for (int n = 0; n < NMAX; ++n)
            if (n < N) cfma(acc[n], a, srow[n]);
          k = (k + 1 == K) ? 0 : k + 1;
        }
        if constexpr (sizeof(R) == 4 && NMAX % 2 == 0) {
          if (N == NMAX && (reinterpret_cast<uintptr_t>(orow) & 15) == 0) {
#pragma unroll
            for (int n = 0; n < NMAX; n += 2)
              *reinterpret_cast<float4*>(orow + n) = make_float4(acc[n].x, acc[n].y, acc[n + 1].x, acc[n + 1].y);
            continue;
          }
        }
#pragma unroll
        for (int n = 0; n < NMAX; ++n)
          if (n < N) orow[n] = acc[n];
      } else {
        // row-resident: the row's K <= KMAX values in registers (rotated)
        C av[KMAX];
        int kidx[KMAX];
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
          int k = rot + j;
          k = (k >= K) ? k - K : k;
          kidx[j] = k;
          av[j] = (j < K) ? trow[koff_s[j < K ? k : 0]] : czero<R>();
        }
        for (int n0 = 0; n0 < N; n0 += 8) {
          C acc[8];
#pragma unroll
          for (int jn = 0; jn < 8; ++jn) acc[jn] = czero<R>();
#pragma unroll
          for (int j = 0; j < KMAX; ++j) {
            if (j < K) {
              const C* srow = S + kidx[j] * SP + n0;
#pragma unroll
              for (int jn = 0; jn < 8; ++jn)
                if (n0 + jn < N) cfma(acc[jn], av[j], srow[jn]);
            }
          }
#pragma unroll
          for (int jn = 0; jn < 8; ++jn)
            if (n0 + jn < N) orow[n0 + jn] = acc[jn];
        }
      }
    }
    fence_proxy_async();   // order this stage's generic reads before the async-proxy refill
    if constexpr (PROD) {
      mbar_arrive_warp(&empty[stage]);
    } else {
      __syncthreads();     // everyone is done with this stage
      if (threadIdx.x < 32 && t + PIPE_STAGES < t1)
        issue_tile<C>(p, A, t + PIPE_STAGES, ring + stage * tile_elems, &bars[stage]);
    }
  }
}

}  // namespace tnc

namespace tnc {

// ---------------------------------------------------------------------------
// Element-mapped pipelined variant for N >= 8 (N | 256): consecutive threads
// own consecutive *outputs* of the tile's contiguous [R][N] result block, so
// stores are fully coalesced; a thread's output column n is fixed, its site
// column S[:, n] lives in registers, and the accumulator values a[row][k] are
// warp broadcasts (N >= 32) or few-way reads from the staged tile.
// ---------------------------------------------------------------------------
template <typename R, int KMAX, int NV = 1>
__global__ void __launch_bounds__(256, 1)
k_pair_pipe_cols(const __grid_constant__ PairTile p, const void* __restrict__ A_, const void* __restrict__ B_,
                 void* __restrict__ O_, int64_t tiles_total, int64_t tiles_per_cta) {
  using C = typename cplx<R>::T;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  C* ring = reinterpret_cast<C*>(smem_raw + 128);
  const int64_t tile_elems = p.Kout * p.Lseg;
  int32_t* koff_s = reinterpret_cast<int32_t*>(ring + PIPE_STAGES * tile_elems);
  int32_t* rowoff_s = koff_s + KMAX;
  const C* A = reinterpret_cast<const C*>(A_);
  const C* B = reinterpret_cast<const C*>(B_);
  C* O = reinterpret_cast<C*>(O_);
  const int64_t t0 = blockIdx.x * tiles_per_cta;
  const int64_t t1 = min(t0 + tiles_per_cta, tiles_total);
  if (t0 >= t1) return;
  const int K = (int)p.K, N = (int)p.N;
  const int Rr = (int)p.R;
  if (threadIdx.x == 0) {
    for (int s = 0; s < PIPE_STAGES; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
  }
  for (int k = threadIdx.x; k < K; k += blockDim.x) koff_s[k] = p.koff[k];
  for (int r = threadIdx.x; r < Rr; r += blockDim.x) rowoff_s[r] = p.rowoff[r];
  __syncthreads();
  if (threadIdx.x < 32)
    for (int s = 0; s < PIPE_STAGES && t0 + s < t1; ++s) issue_tile<C>(p, A, t0 + s, ring + s * tile_elems, &bars[s]);
  // NV consecutive output columns per thread (NV = 2: one 16-byte store per
  // row and half the shared-memory reads per output)
  const int NN = N / NV;
  const int n = (threadIdx.x % NN) * NV;  // first output column of this thread
  const int row_step = blockDim.x / NN;
  const int row0 = threadIdx.x / NN;
  C scol[NV][KMAX];
  int kof[KMAX];                          // shared-index offsets in registers (no per-row table reads)
#pragma unroll
  for (int k = 0; k < KMAX; ++k) kof[k] = (k < K) ? koff_s[k] : 0;
  int64_t cur_z = -1;
  for (int64_t i = 0; t0 + i < t1; ++i) {
    const int64_t t = t0 + i;
    const int stage = (int)(i % PIPE_STAGES);
    const uint32_t phase = (uint32_t)((i / PIPE_STAGES) & 1);
    const int64_t z = t / p.U, u = t - (t / p.U) * p.U;
    if (z != cur_z) {
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const C* Bz = B + z * p.b_zstride + p.b_noff[n + j];
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
          C v = (k < K) ? __ldg(Bz + p.b_koff[k < K ? k : 0]) : czero<R>();
          if (p.conj_b) v = cconj(v);
          scol[j][k] = v;
        }
      }
      cur_z = z;
    }
    mbar_wait_spin(&bars[stage], phase);
    const C* tile = ring + stage * tile_elems;
    C* Ot = O + z * p.out_zstride + u * p.R * p.N;
    auto store = [&](int row, const C (&acc)[NV]) {
      if constexpr (NV % 2 == 0 && sizeof(R) == 4) {
#pragma unroll
        for (int j = 0; j < NV; j += 2)
          *reinterpret_cast<float4*>(Ot + (int64_t)row * N + n + j) =
              make_float4(acc[j].x, acc[j].y, acc[j + 1].x, acc[j + 1].y);
      } else {
#pragma unroll
        for (int j = 0; j < NV; ++j) Ot[(int64_t)row * N + n + j] = acc[j];
      }
    };
    // two rows per iteration: twice the independent FMA chains and shared
    // loads in flight (short-scoreboard and fixed-latency stalls dominated)
    int row = row0;
    for (; row + row_step < Rr; row += 2 * row_step) {
      const C* tr0 = tile + rowoff_s[row];
      const C* tr1 = tile + rowoff_s[row + row_step];
      C acc0[NV], acc1[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) acc0[j] = acc1[j] = czero<R>();
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K) {
          const C a0 = tr0[kof[k]], a1 = tr1[kof[k]];
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            cfma(acc0[j], a0, scol[j][k]);
            cfma(acc1[j], a1, scol[j][k]);
          }
        }
      store(row, acc0);
      store(row + row_step, acc1);
    }
    if (row < Rr) {
      const C* trow = tile + rowoff_s[row];
      C acc[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) acc[j] = czero<R>();
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K) {
          const C a = trow[kof[k]];
#pragma unroll
          for (int j = 0; j < NV; ++j) cfma(acc[j], a, scol[j][k]);
        }
      store(row, acc);
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x < 32 && t + PIPE_STAGES < t1)
      issue_tile<C>(p, A, t + PIPE_STAGES, ring + stage * tile_elems, &bars[stage]);
  }
}

}  // namespace tnc
