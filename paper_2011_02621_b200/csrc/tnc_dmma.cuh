// complex128 contraction step on the FP64 tensor cores (DMMA,
// mma.sync.m8n8k4.f64): the complex rows are real rows of length 2K
// (interleaved re/im), the site block is embedded as the real 2K x 2N matrix
// B' = [[Re, Im], [-Im, Re]] per (k, n), so C' = A' B' is the interleaved
// complex result.  Used for engine steps with row-contiguous accumulators and
// K*N >= 256 (FP64-compute-bound at these extents).
#pragma once
#include "tnc_common.cuh"

namespace tnc {

constexpr int DM_BM = 64;        // rows per CTA tile
constexpr int DM_BN = 64;        // real output columns per CTA tile (32 complex)
constexpr int DM_BK = 32;        // real K per smem stage (16 complex)
constexpr int DM_THREADS = 128;  // 4 warps, 16 rows each

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

// grid: (tiles_m * tiles_n) per z, z-major
__global__ void __launch_bounds__(DM_THREADS)
k_dmma_c128(const __grid_constant__ tnc_step_desc d, int64_t tiles_m, int64_t tiles_n) {
  // two smem stages; the next stage's global loads are issued into registers
  // before the current stage's DMMAs and stored after them (the synchronous
  // load -> sync -> DMMA loop left the DMMA sub-pipe 57% active, ncu)
  extern __shared__ __align__(16) unsigned char dm_smem[];
  double (*As)[DM_BM][DM_BK + 4] = reinterpret_cast<double (*)[DM_BM][DM_BK + 4]>(dm_smem);   // [stage][row][k'] (padded)
  double (*Bs)[DM_BK][DM_BN + 4] =
      reinterpret_cast<double (*)[DM_BK][DM_BN + 4]>(dm_smem + 2 * sizeof(double) * DM_BM * (DM_BK + 4));  // [stage][k'][n']
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t t = blockIdx.x;
  const int64_t tiles = tiles_m * tiles_n;
  const int64_t z = t / tiles;
  t -= z * tiles;
  const int64_t m0 = (t / tiles_n) * DM_BM;
  const int64_t n0r = (t % tiles_n) * DM_BN;               // real column offset
  const double2* A = reinterpret_cast<const double2*>(d.acc) + z * d.acc_zstride;
  const double2* S = reinterpret_cast<const double2*>(d.site.ptr) + site_offset(d.site, z, d.slices_per_b, d.s0);
  double2* O = reinterpret_cast<double2*>(d.out) + z * d.out_zstride;
  const int Kr = (int)(2 * d.K);
  double acc[2][8][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  constexpr int NA = DM_BM * (DM_BK / 2) / DM_THREADS;          // 8 A elements per thread and stage
  constexpr int NB = (DM_BK / 2) * (DM_BN / 2) / DM_THREADS;    // 4 site elements
  double2 ra[NA], rb[NB];
  // this thread's site columns do not change over the K loop
  int64_t bno[NB];
  bool bnv[NB];
#pragma unroll
  for (int u = 0; u < NB; ++u) {
    const int e = threadIdx.x + u * DM_THREADS;
    const int64_t n = n0r / 2 + e % (DM_BN / 2);
    bnv[u] = n < d.N;
    bno[u] = bnv[u] ? d.b_noff[n] : 0;
  }
  auto fetch = [&](int k0) {
#pragma unroll
    for (int u = 0; u < NA; ++u) {
      const int e = threadIdx.x + u * DM_THREADS;
      const int r = e / (DM_BK / 2), kc = e % (DM_BK / 2);
      const int64_t row = m0 + r, k = k0 / 2 + kc;
      ra[u] = (row < d.M && k < d.K) ? A[row * d.K + k] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const int e = threadIdx.x + u * DM_THREADS;
      const int64_t k = k0 / 2 + e / (DM_BN / 2);
      double2 sv = make_double2(0.0, 0.0);
      if (k < d.K && bnv[u]) {
        sv = S[d.b_koff[k] + bno[u]];
        if (d.conj_b) sv.y = -sv.y;
      }
      rb[u] = sv;
    }
  };
  auto stash = [&](int st) {
#pragma unroll
    for (int u = 0; u < NA; ++u) {
      const int e = threadIdx.x + u * DM_THREADS;
      const int r = e / (DM_BK / 2), kc = e % (DM_BK / 2);
      As[st][r][2 * kc] = ra[u].x;
      As[st][r][2 * kc + 1] = ra[u].y;
    }
    // B' stage: rows k' = 2k + c, cols n' = 2n + c'
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const int e = threadIdx.x + u * DM_THREADS;
      const int kc = e / (DM_BN / 2), nc = e % (DM_BN / 2);
      Bs[st][2 * kc][2 * nc] = rb[u].x;      Bs[st][2 * kc][2 * nc + 1] = rb[u].y;
      Bs[st][2 * kc + 1][2 * nc] = -rb[u].y; Bs[st][2 * kc + 1][2 * nc + 1] = rb[u].x;
    }
  };
  fetch(0);
  stash(0);
  __syncthreads();
  int st = 0;
  for (int k0 = 0; k0 < Kr; k0 += DM_BK, st ^= 1) {
    const bool more = k0 + DM_BK < Kr;
    if (more) fetch(k0 + DM_BK);                   // in flight during this stage's DMMAs
#pragma unroll
    for (int ks = 0; ks < DM_BK; ks += 4) {
      double af[2], bf[8];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = As[st][warp * 16 + i * 8 + (lane >> 2)][ks + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 8; ++j) bf[j] = Bs[st][ks + (lane & 3)][j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma_8x8x4(acc[i][j], af[i], bf[j]);
    }
    if (more) stash(st ^ 1);                       // the other stage: last read before the previous barrier
    __syncthreads();
  }
  // C fragment: row = lane/4, real cols 2*(lane%4), +1  -> one complex per fragment
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int64_t row = m0 + warp * 16 + i * 8 + (lane >> 2);
    if (row >= d.M) continue;
    int64_t oc = row * d.N;
    if (!d.c_rows_contig) {
      int64_t oa;
      row_offsets(d, row, oa, oc);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t n = (n0r + j * 8 + 2 * (lane & 3)) / 2;
      if (n < d.N) O[d.c_rows_contig ? oc + n : oc + d.c_noff[n]] = make_double2(acc[i][j][0], acc[i][j][1]);
    }
  }
}

template <typename R>
int try_dmma(const tnc_step_desc& d, cudaStream_t s) {
  if constexpr (sizeof(R) != 8) {
    return 0;
  } else {
    if (!d.a_rows_contig || d.K * d.N < 256) return 0;
    const int64_t tm = (d.M + DM_BM - 1) / DM_BM, tn = (2 * d.N + DM_BN - 1) / DM_BN;
    const int64_t blocks = d.Z * tm * tn;
    if (blocks <= 0 || blocks > 0x7fffffffLL) return 0;
    constexpr size_t smem = 2 * sizeof(double) * (DM_BM * (DM_BK + 4) + DM_BK * (DM_BN + 4));   // 70 KB: two stages
    static uint64_t attr = 0;
    int adev = 0;
    if (attr_needed(attr, &adev)) {
      cudaFuncSetAttribute(k_dmma_c128, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr |= 1ull << (adev & 63);
    }
    k_dmma_c128<<<(unsigned)blocks, DM_THREADS, smem, s>>>(d, tm, tn);
    return cudaGetLastError() == cudaSuccess ? 1 : -1;
  }
}

}  // namespace tnc
