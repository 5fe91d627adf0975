// Tensor-core contraction step for complex64: tcgen05.mma kind::tf32 with a
// 3xTF32 split (hi*hi + hi*lo + lo*hi, fp32 accumulation in TMEM) so the
// result keeps ~fp32 accuracy (north-star tolerance 1e-4 for complex64).
//
// Complex -> real embedding: an accumulator row [a_0 .. a_{K-1}] (interleaved
// re/im) is the real row A' = [Re a_0, Im a_0, ...] of length 2K; the site block
// S[K][N] becomes B' (2K x 2N) with B'[(k,re),(n,re)] = Re s, B'[(k,im),(n,re)] =
// -Im s, B'[(k,re),(n,im)] = Im s, B'[(k,im),(n,im)] = Re s, so D = A' B' is the
// interleaved complex result row.  A persistent CTA (one wave, <= #SMs) owns
// a contiguous range of 128-row tiles over (batch element z, row block); the
// MMA warp rebuilds B' in place when its tiles cross into a new z.
//
// Warp roles (416 threads): warps 0-7 convert accumulator chunks (global ->
// tf32 hi/lo -> canonical K-major smem), warps 8-11 drain TMEM (epilogue),
// warp 12 issues the MMAs.  Pipelines: A-chunk ring (2 stages, mbarriers),
// TMEM accumulators (2 stages).
#pragma once
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <cuda.h>
#include <cuda_fp16.h>
#include "tnc_common.cuh"

namespace tnc {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*tg_encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline tg_encode_fn tg_encoder() {
  static tg_encode_fn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<tg_encode_fn>(f);
  }
  return fn;
}

struct TcDesc {
  int64_t M, K, N;                 // rows per batch element (multiple of 128)
  int64_t tiles_per_z, per_cta, Z;
  const float2* a;
  int64_t a_zstride;
  int32_t nho;                     // outer free legs above the 128-row block
  int32_t conj_b;
  int64_t ho_dim[TNC_MAX_LEGS], ho_stride[TNC_MAX_LEGS];
  const int64_t* lo_off;           // [128] accumulator offset of row r inside a block
  const int64_t* akoff;            // [K]
  tnc_site site;
  int64_t slices_per_b, s0;
  const int64_t* b_koff;           // [K]
  const int64_t* b_noff;           // [N]
  float2* out;
  int64_t out_zstride;             // out rows are contiguous: out + z*zs + g*N + n
  int32_t rows_contig;             // lo_off[r] = r*K and akoff[k] = k (tables unused)
  int32_t nstages;                 // A-chunk ring depth (host: as many as fit)
  int32_t f16;                     // 1: fp16-split operands, per-row A scales, per-z site scales (bscale)
  const float* bscale;             // [Z] max |re|,|im| of the site block of z (f16)
  // raw-ring mode: each tile's 128 x K accumulator block is staged by cp.async.bulk
  // as Kout contiguous segments of Lseg elements; element (r, k) sits at
  // lo_off[r] + kraw[k] inside the staged tile
  int32_t raw_stages;              // 0: converters gather from global directly
  int32_t raw_ok;                  // host: layout admits the raw ring
  int64_t Kout, Lseg;
  const int64_t* segoff;           // [Kout] segment offsets from the tile base
  const int32_t* kraw;             // [K]
  // bank-conflict avoidance for the converters' staged-tile reads: row r of a
  // half-warp reads chunk slot q from k = q ^ x(r), x(r) = XOR of kx_row[i] over
  // the set bits i < 4 of r (host: 0 unless kraw is XOR-linear within a chunk)
  int32_t kx_row[4];
  const int64_t* ho_lo;            // optional two-level row-block base tables:
  const int64_t* ho_hi;            //   base(m) = ho_hi[m / p_lo] + ho_lo[m % p_lo]
  int64_t p_lo;
  // 1: the epilogue stages each warp's 32 result rows (one full accumulator
  // chunk: 2N == padded width <= 32, so the rows are one contiguous block)
  // and writes them with one cp.async.bulk store, double-buffered per warp;
  // 2: N >= 32 (2N == padded width, several 32-column chunks): each chunk's
  // 32 rows x 128 B go out as one TMA tensor-store box (tmO: [Z][M][2N] fp32)
  int32_t bulk_out;
};

constexpr int TC_CONV_WARPS = 8;
constexpr int TC_EPI_WARP0 = 8;
constexpr int TC_EPI_WARPS = 8;          // two epilogue groups alternate tiles
constexpr int TC_MMA_WARP = 16;
constexpr int TC_PROD_WARP = 17;         // raw-ring producer (cp.async.bulk)
constexpr int TC_THREADS = 18 * 32;
constexpr int TC_MAX_STAGES = 8;
constexpr int TC_MAX_TILES = 2048;      // tiles per CTA (one wave; smem base table)

__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
// hi = x rounded to the nearest tf32 (add half an ulp, clear the 13 low
// mantissa bits), lo = x - hi (exact in fp32; the tensor core reads its top 19
// bits).  Rounding hi to nearest keeps lo sign-random, so the dropped lo*lo
// term and the truncation of lo do not correlate with the sign of a*b and
// cancel in long sums (a truncated hi biases every product by ~2^-23).
// Three instructions per value (cvt.rna.tf32 expands to ~8).
__device__ __forceinline__ void split3(float x, float& hi, float& lo) {
  hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
  lo = x - hi;
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;          // descriptor version (sm_100)
  return d;                        // base_offset 0, lbo_mode 0, SWIZZLE_NONE
}

__device__ __forceinline__ uint32_t tf32_idesc(int n_real) {
  return (1u << 4)                 // D f32
       | (2u << 7) | (2u << 10)    // A, B tf32
       | ((uint32_t)(n_real >> 3) << 17)
       | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// smem sizes (bytes) for a (K, N) problem
__host__ __device__ inline int64_t tc_b_bytes(int64_t K, int64_t N) { return 2 * (2 * N) * (2 * K) * 4; }
__host__ __device__ inline int64_t tc_kc(int64_t K) { return K >= 16 ? 16 : K; }
__host__ __device__ inline int64_t tc_npad(int64_t N) { return N <= 8 ? 8 : ((N + 7) / 8) * 8; }
constexpr int TC_EPI_PITCH = 144;        // bytes per staged row (128 + 16 pad: conflict-free)
__host__ __device__ inline int64_t tc_raw_bytes(int64_t K) { return 128 * K * 8; }
constexpr int TC_EPI_BULK_BYTES = 2 * 4096;  // bulk_out: two 32-row x 128 B buffers per warp
__host__ __device__ inline int64_t tc_epi_warp_bytes(int bulk) { return bulk ? TC_EPI_BULK_BYTES : 32 * TC_EPI_PITCH; }
__host__ __device__ inline int64_t tc_smem_bytes(int64_t K, int64_t N, int64_t per, int64_t rs, int bulk = 0) {
  return 1024 + tc_b_bytes(K, tc_npad(N)) + K * 8 + K * 4 + 128 * 8 + 6 * TC_MAX_STAGES * 8 + 128 + per * 8
         + TC_EPI_WARPS * tc_epi_warp_bytes(bulk) + 128 + rs * tc_raw_bytes(K);
}
// TMEM plan: TS accumulators of Nr columns, AS A-chunk stages of 4*KC columns (hi + lo)
// f16: A stages of 2*kc columns (two fp16 per column) and TC_SCALE_COLS
// columns at the top of TMEM: a ring of per-row inverse scales indexed by tile
constexpr int TC_SCALE_COLS = 32;
__host__ __device__ inline void tc_tmem_plan(int64_t K, int64_t N, int& TS, int& AS, bool f16 = false) {
  const int Nr = (int)(2 * N), kc = (int)tc_kc(K);
  TS = 256 / Nr;
  if (TS > TC_MAX_STAGES) TS = TC_MAX_STAGES;
  TS &= ~1;                                     // even: each epilogue group owns its stages
  if (TS < 2) TS = 2;
  AS = f16 ? (512 - TS * Nr - TC_SCALE_COLS) / (2 * kc) : (512 - TS * Nr) / (4 * kc);
  if (AS > TC_MAX_STAGES) AS = TC_MAX_STAGES;
}

// power-of-two scale s with max * s in [2^14, 2^15) (1 for zero / non-finite)
__host__ __device__ inline float tc_f16_scale(float amax) {
  if (!(amax > 0.f) || !(amax < 3.0e38f)) return 1.f;
  int e;
#ifdef __CUDA_ARCH__
  e = (int)((__float_as_uint(amax) >> 23) & 0xff) - 127;
#else
  uint32_t u;
  memcpy(&u, &amax, 4);
  e = (int)((u >> 23) & 0xff) - 127;
#endif
  int pw = 14 - e;
  pw = pw < -126 ? -126 : (pw > 127 ? 127 : pw);
#ifdef __CUDA_ARCH__
  return __uint_as_float((uint32_t)(pw + 127) << 23);
#else
  const uint32_t b = (uint32_t)(pw + 127) << 23;
  float f;
  memcpy(&f, &b, 4);
  return f;
#endif
}
// y0, y1 -> packed fp16 hi and lo (low half = y0); see tnc_tcgemm.cuh split_f16x2
__device__ __forceinline__ void tc_split_f16x2(float y0, float y1, uint32_t& h, uint32_t& l) {
  const float h0 = __uint_as_float((__float_as_uint(y0) + 0x1000u) & 0xFFFFE000u);
  const float h1 = __uint_as_float((__float_as_uint(y1) + 0x1000u) & 0xFFFFE000u);
  const float l0 = y0 - h0, l1 = y1 - h1;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(h1), "f"(h0));
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(l1), "f"(l0));
}
__device__ __forceinline__ void tc_split_f16(float y, uint16_t& h, uint16_t& l) {
  const __half hh = __float2half_rn(y);
  const __half ll = __float2half_rn(y - __half2float(hh));
  h = __half_as_ushort(hh);
  l = __half_as_ushort(ll);
}
// per batch element z: max |re|, |im| over its site block (f16 scale of B')
__global__ void k_tc_bmax(const __grid_constant__ TcDesc p, float* out) {
  for (int64_t z = blockIdx.x; z < p.Z; z += gridDim.x) {
    const float2* S = reinterpret_cast<const float2*>(p.site.ptr) + site_offset(p.site, z, p.slices_per_b, p.s0);
    float m = 0.f;
    for (int64_t e = threadIdx.x; e < p.K * p.N; e += blockDim.x) {
      const int64_t k = e / p.N, n = e - k * p.N;
      const float2 v = __ldg(S + p.b_koff[k] + p.b_noff[n]);
      m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
    }
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ float red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
      out[z] = m;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_f16_tc(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
template <int NW, int LEN>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const uint32_t (&v)[LEN]) {
  static_assert(NW <= LEN, "tmem_st width");
  if constexpr (NW == 32) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                 ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                   "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
                   "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
                   "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
  } else if constexpr (NW == 16) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                   "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
  } else if constexpr (NW == 8) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
  } else {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};"
                 ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]));
  }
}
// one lane of a converged warp (warp-uniform operands stay in uniform registers)
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(e));
  return e != 0;
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// B' (hi, lo) for batch element z, written by threads [tid0, tid0 + nthr)
template <bool F16>
__device__ __forceinline__ void build_b(const TcDesc& p, int64_t z, float* Bhi, float* Blo, int tid, int nthr) {
  const int K = (int)p.K, N = (int)p.N;
  const uint32_t SBO_B = ((2 * K) / 4) * 128;
  const float2* S = reinterpret_cast<const float2*>(p.site.ptr) + site_offset(p.site, z, p.slices_per_b, p.s0);
  const float t = F16 ? tc_f16_scale(__ldg(p.bscale + z)) : 1.f;
  for (int e = tid; e < K * N; e += nthr) {
    const int k = e / N, n = e - (e / N) * N;
    float2 sv = __ldg(S + p.b_koff[k] + p.b_noff[n]);
    if (p.conj_b) sv.y = -sv.y;
    // rows n' = 2n (re out), 2n+1 (im out); cols k' = 2k (re in), 2k+1 (im in)
    const float vals[4] = {sv.x, -sv.y, sv.y, sv.x};
    if constexpr (F16) {
      // 16-bit K-major canonical: 8 rows x 16 B core matrices, LBO 128 B along K, SBO (2K/8)*128 B along N
      const uint32_t SBO16 = ((2 * K) / 8) * 128;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int nr = 2 * n + (q >> 1), kr = 2 * k + (q & 1);
        const uint32_t off = (nr & 7) * 16 + (nr >> 3) * SBO16 + (kr >> 3) * 128 + (kr & 7) * 2;
        uint16_t h, l;
        tc_split_f16(vals[q] * t, h, l);
        *reinterpret_cast<uint16_t*>(reinterpret_cast<unsigned char*>(Bhi) + off) = h;
        *reinterpret_cast<uint16_t*>(reinterpret_cast<unsigned char*>(Blo) + off) = l;
      }
      continue;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int nr = 2 * n + (q >> 1), kr = 2 * k + (q & 1);
      const uint32_t off = (nr & 7) * 16 + (nr >> 3) * SBO_B + (kr >> 2) * 128 + (kr & 3) * 4;
      float h, l;
      split3(vals[q], h, l);
      *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(Bhi) + off) = h;
      *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(Blo) + off) = l;
    }
  }
}

// KH = complex values per converter thread per chunk (KC / 2)
// TMO: N >= 32 results written as TMA tensor-store boxes (bulk_out == 2); a
// separate instantiation, so the other kernels' code is unchanged (with the
// store path compiled in, the N = 16 kernel measured 3-5% slower)
template <int KH, bool F16, bool TMO = false>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_tc_c64(const __grid_constant__ TcDesc p, const __grid_constant__ CUtensorMap tmO) {
  static_assert(!F16 || KH == 8, "F16 needs 16-complex chunks");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  constexpr int KC = 2 * KH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = (int)p.K, N = (int)p.N;          // N: real outputs per row
  const int Np = (int)tc_npad(p.N);              // MMA width (multiple of 8, >= 8)
  const int Kr = 2 * K, Nr = 2 * Np;
  const int nchunk = K / KC;
  const uint32_t SBO_B = (Kr / 4) * 128;
  int TS, AS;
  tc_tmem_plan(p.K, Np, TS, AS, F16);
  const uint32_t A0 = (uint32_t)(TS * Nr);      // first A column
  // per A stage: tf32 hi (2KC) + lo (2KC) columns; f16 hi (KC) + lo (KC), one complex per column
  constexpr uint32_t ACOLS = F16 ? 2 * KC : 4 * KC;
  // f16: column SCOL + t % TC_SCALE_COLS holds tile t's per-row inverse scales.  A
  // converter is at most AS + TS tiles ahead of the epilogue's scale read
  // (A stages, then accumulator stages), and AS + TS <= 16 < TC_SCALE_COLS,
  // so a column is never rewritten before it has been read -- no extra wait
  const uint32_t SCOL = 512u - (uint32_t)TC_SCALE_COLS;
  // ---- shared memory carve-up ----
  float* Bhi = reinterpret_cast<float*>(smem_raw);
  float* Blo = Bhi + (size_t)Nr * Kr;
  unsigned char* rawring = reinterpret_cast<unsigned char*>(Blo + (size_t)Nr * Kr);   // [RS][128*K complex]
  const int RS = p.raw_stages;
  int64_t* akoff_s = reinterpret_cast<int64_t*>(rawring + (size_t)RS * tc_raw_bytes(p.K));
  int64_t* looff_s = akoff_s + K;
  int32_t* kraw_s = reinterpret_cast<int32_t*>(looff_s + 128);
  uint64_t* bar = reinterpret_cast<uint64_t*>(kraw_s + ((K + 1) & ~1));
  uint64_t* full = bar;                        // [AS] converters -> MMA
  uint64_t* empty = bar + TC_MAX_STAGES;       // [AS] MMA commit -> converters
  uint64_t* tfull = bar + 2 * TC_MAX_STAGES;   // [TS] MMA commit -> epilogue
  uint64_t* tempty = tfull + TC_MAX_STAGES;    // [TS] epilogue -> MMA
  uint64_t* rfull = tempty + TC_MAX_STAGES;    // [RS] bulk copy landed -> converters
  uint64_t* rempty = rfull + TC_MAX_STAGES;    // [RS] converters done -> producer
  uint64_t* bdone = rempty + TC_MAX_STAGES;    // MMA-warp-local: B' retire
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bdone + 1);
  int64_t* tbase = reinterpret_cast<int64_t*>(bdone + 2);   // [per_cta] accumulator base of each tile
  unsigned char* epi_stage = reinterpret_cast<unsigned char*>(
      TMO ? (reinterpret_cast<uintptr_t>(tbase + p.per_cta) + 127) & ~(uintptr_t)127    // TMA store boxes
          : (reinterpret_cast<uintptr_t>(tbase + p.per_cta) + 15) & ~(uintptr_t)15);

  // global tile index g = z * tiles_per_z + m; this CTA owns [g0, g1)
  const int64_t g0 = blockIdx.x * p.per_cta;
  const int64_t g1 = min(g0 + p.per_cta, p.Z * p.tiles_per_z);
  const int ntiles = (int)(g1 - g0);
  const int64_t z0 = g0 / p.tiles_per_z;

  // ---- setup ----
  if (threadIdx.x == 0) {
    for (int s = 0; s < AS; ++s) {
      mbar_init(&full[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < TS; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
    }
    for (int s = 0; s < RS; ++s) {
      mbar_init(&rfull[s], 1);
      mbar_init(&rempty[s], 4);
    }
    mbar_init(bdone, 1);
    mbar_fence_init();
  }
  if (warp == TC_EPI_WARP0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int k = threadIdx.x; k < K; k += blockDim.x) akoff_s[k] = p.rows_contig ? k : p.akoff[k];
  for (int r = threadIdx.x; r < 128; r += blockDim.x) looff_s[r] = p.rows_contig ? (int64_t)r * K : p.lo_off[r];
  for (int k = threadIdx.x; k < K && RS > 0; k += blockDim.x) kraw_s[k] = p.rows_contig ? k : p.kraw[k];
  if (Np != N) {
    uint4* bz = reinterpret_cast<uint4*>(Bhi);
    for (int i = threadIdx.x; i < 2 * Nr * Kr / 4; i += blockDim.x) bz[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
  }
  if (ntiles > 0) build_b<F16>(p, z0, Bhi, Blo, threadIdx.x, blockDim.x);
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
    const int64_t g = g0 + t;
    const int64_t zt = g / p.tiles_per_z;
    int64_t mb = g - zt * p.tiles_per_z, hb = zt * p.a_zstride;
    if (p.ho_lo) {
      const int64_t q = mb / p.p_lo;
      hb += __ldg(p.ho_hi + q) + __ldg(p.ho_lo + (mb - q * p.p_lo));
    } else {
      for (int j = p.nho - 1; j >= 0; --j) {
        const int64_t q = mb / p.ho_dim[j];
        hb += (mb - q * p.ho_dim[j]) * p.ho_stride[j];
        mb = q;
      }
    }
    tbase[t] = hb;
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < TC_CONV_WARPS) {
    // ---------------- converters: 2 groups of 4 warps alternate tiles; thread =
    // one tile row (TMEM lane) and all KC values of a chunk ----------------
    // Each group owns its own slice of the A ring (stages [grp*ASg, (grp+1)*ASg))
    // and, with RS even, its own raw stages, so no waiter can alias a barrier
    // phase two uses ahead.
    const int NG = (AS >= 4 && (RS == 0 || RS % 2 == 0)) ? 2 : 1;
    const int grp = warp >> 2;
    const int ASg = AS / NG;
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const float2* A = p.a + looff_s[r];
    // staged-tile reads: slot q of this row comes from k = q ^ xk (see TcDesc::kx_row)
    int xk = 0, xm = 0;
    if (RS > 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        xm |= p.kx_row[i];
        if ((r >> i) & 1) xk ^= p.kx_row[i];
      }
    }
    const int32_t kx = RS > 0 ? kraw_s[xk] : 0;
    int j = 0;                                   // this group's chunk counter
    for (int t = grp; t < ntiles && grp < NG; t += NG) {
      const float2* raw = nullptr;
      if (RS > 0) {
        const int rs = t % RS;
        mbar_wait_spin(&rfull[rs], (uint32_t)((t / RS) & 1));
        raw = reinterpret_cast<const float2*>(rawring + (size_t)rs * tc_raw_bytes(p.K)) + looff_s[r];
      }
      const float2* Ar = A + tbase[t];
      float sA = 1.f;
      bool scale_pending = false;
      if constexpr (F16) {
        if (nchunk > 1) {
          // per-row scale from the whole row (the raw stage holds the full 128 x K tile)
          float m = 0.f;
          for (int k = 0; k < K; ++k) {
            const float2 x = raw[kraw_s[k] ^ kx];
            m = fmaxf(m, fmaxf(fabsf(x.x), fabsf(x.y)));
          }
          sA = tc_f16_scale(m);
        } else {
          scale_pending = true;                  // one chunk: the row max comes from its registers below
        }
      }
      for (int c = 0; c < nchunk; ++c, ++j) {
        const int stage = grp * ASg + j % ASg;
        const uint32_t ph = (j / ASg) & 1;
        float2 v[KC];
        if (RS > 0) {
          const int32_t* kr = kraw_s + c * KC;
#pragma unroll
          for (int q = 0; q < KC; ++q) v[q] = raw[kr[q] ^ kx];
          if (xm) {                              // undo the per-row slot permutation
#pragma unroll
            for (int b = 0; (1 << b) < KC; ++b) {
              if ((xm >> b) & 1) {
                const bool sw = (xk >> b) & 1;
#pragma unroll
                for (int q = 0; q < KC; ++q) {
                  if (q & (1 << b)) continue;
                  const float2 u0 = v[q], u1 = v[q | (1 << b)];
                  v[q] = sw ? u1 : u0;
                  v[q | (1 << b)] = sw ? u0 : u1;
                }
              }
            }
          }
        } else {
          const int64_t* ko = akoff_s + c * KC;
#pragma unroll
          for (int q = 0; q < KC; ++q) v[q] = __ldg(Ar + ko[q]);
        }
        if constexpr (F16) {
          if (scale_pending) {
            float m = 0.f;
#pragma unroll
            for (int q = 0; q < KC; ++q) m = fmaxf(m, fmaxf(fabsf(v[q].x), fabsf(v[q].y)));
            sA = tc_f16_scale(m);
            scale_pending = false;
          }
        }
        mbar_wait_spin(&empty[stage], ph ^ 1);
        tc_fence_after();
        const uint32_t col = A0 + (uint32_t)stage * ACOLS;
        if constexpr (F16) {
          if (c == 0) {                          // tile's inverse row scales (site factor 1/t(z) in the epilogue)
            const uint32_t iv = __float_as_uint(1.f / sA);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};"
                         ::"r"(tmem + lane_base + SCOL + (uint32_t)(t % TC_SCALE_COLS)), "r"(iv));
          }
          uint32_t hi[KC], lo[KC];
#pragma unroll
          for (int q = 0; q < KC; ++q) tc_split_f16x2(v[q].x * sA, v[q].y * sA, hi[q], lo[q]);
          tmem_st<KC>(tmem + lane_base + col, hi);
          tmem_st<KC>(tmem + lane_base + col + KC, lo);
        }
#pragma unroll
        for (int half = 0; half < (F16 ? 0 : 2); ++half) {
          uint32_t hi[KC], lo[KC];
#pragma unroll
          for (int q = 0; q < KC / 2; ++q) {
            float a, b;
            split3(v[half * KC / 2 + q].x, a, b);
            hi[2 * q] = __float_as_uint(a);
            lo[2 * q] = __float_as_uint(b);
            split3(v[half * KC / 2 + q].y, a, b);
            hi[2 * q + 1] = __float_as_uint(a);
            lo[2 * q + 1] = __float_as_uint(b);
          }
          tmem_st<KC>(tmem + lane_base + col + half * KC, hi);
          tmem_st<KC>(tmem + lane_base + col + 2 * KC + half * KC, lo);
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive_warp(&full[stage]);
        if (RS > 0 && c == nchunk - 1) {
          // the tile's raw values have been consumed (converted and stored);
          // order these generic reads before the async-proxy refill
          fence_proxy_async();
          mbar_arrive_warp(&rempty[t % RS]);
        }
      }
    }
  } else if (warp < TC_MMA_WARP) {
    // ---------------- epilogue: TMEM -> registers -> padded smem -> coalesced global ----------------
    const int eg = (warp - TC_EPI_WARP0) >> 2;   // epilogue group (alternate tiles; TS even)
    const int q = warp & 3;                      // lane quarter
    const int r = q * 32 + lane;                 // tile row
    unsigned char* stg = epi_stage + (eg * 4 + q) * tc_epi_warp_bytes(p.bulk_out);
    const bool bulk = p.bulk_out != 0;
    int oblk = 0;                                // bulk_out: staging buffer parity
    // tile -> (z, row block) tracked incrementally (this group steps by 2 tiles)
    int64_t zt = (g0 + eg) / p.tiles_per_z, mb = (g0 + eg) - zt * p.tiles_per_z;
    int64_t inv2_z = -1;
    float inv2 = 1.f;
    for (int t = eg; t < ntiles; t += 2) {
      const int acc = t % TS;
      const uint32_t ph = (t / TS) & 1;
      if (t != eg) {
        mb += 2;
        while (mb >= p.tiles_per_z) { mb -= p.tiles_per_z; ++zt; }
      }
      mbar_wait_spin(&tfull[acc], ph);
      tc_fence_after();
      const int64_t grow = mb * 128 + r;
      float2* otile = p.out + zt * p.out_zstride + (grow - lane) * N;   // this warp's 32 rows
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * Nr);
      float inv = 1.f;
      uint32_t iv = 0;
      if constexpr (F16) {
        if (zt != inv2_z) { inv2_z = zt; inv2 = 1.f / tc_f16_scale(__ldg(p.bscale + zt)); }
        // the row's inverse scale rides along with the first accumulator read (one wait)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                     : "=r"(iv) : "r"(tmem + ((uint32_t)(q * 32) << 16) + SCOL + (uint32_t)(t % TC_SCALE_COLS)));
      }
      for (int c0 = 0; c0 < Nr; c0 += 32) {
        const int cols = (c0 + 32 <= Nr) ? 32 : 16;
        uint32_t v[32];
        if (cols == 32) {
          tmem_ld32(taddr + c0, v);
        } else {
          uint32_t w16[16];
          tmem_ld16(taddr + c0, w16);
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = w16[j];
        }
        tmem_wait_ld();
        if constexpr (F16) inv = __uint_as_float(iv);
        if (c0 + 32 >= Nr) {              // accumulator drained: hand it back before the stores
          tc_fence_before();
          mbar_arrive_warp(&tempty[acc]);
        }
        if constexpr (F16) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * inv * inv2);
        }
        if (bulk) {
          // rows of cols*4 bytes, packed: the warp's 32 rows are the contiguous
          // output block otile[0 .. 32N).  Lane writes 16-byte piece m of its row
          // in slot order j = m ^ x (x = the lane's position inside a 128-byte
          // wavefront), so a quarter-warp's stores hit distinct banks; the
          // register blocks are permuted with uniform conditional swaps
          const int P = cols / 4;                        // 16-byte pieces per row (4 or 8)
          const int x = P == 8 ? (lane & 7) : ((lane >> 1) & 3);
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            if ((1 << b) >= P) continue;
            const bool sw = (x >> b) & 1;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (j >= P || (j & (1 << b))) continue;
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const uint32_t u0 = v[4 * j + e], u1 = v[4 * (j | (1 << b)) + e];
                v[4 * j + e] = sw ? u1 : u0;
                v[4 * (j | (1 << b)) + e] = sw ? u0 : u1;
              }
            }
          }
          unsigned char* sb = stg + (oblk & 1) * 4096;
          ++oblk;
          // the bulk store that last read this buffer (two tiles ago) is done reading
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < P)
              *reinterpret_cast<uint4*>(sb + lane * (P * 16) + (j ^ x) * 16) =
                  make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            if constexpr (TMO) {
              asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];"
                           ::"l"(reinterpret_cast<uint64_t>(&tmO)), "r"(c0), "r"((int)(grow - lane)), "r"((int)zt),
                             "r"(smem_u32(sb)) : "memory");
            } else {
              asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                           ::"l"(otile), "r"(smem_u32(sb)), "r"((uint32_t)(32 * P * 16)) : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          continue;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (4 * j < cols)
            *reinterpret_cast<uint4*>(stg + lane * TC_EPI_PITCH + j * 16) =
                make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        __syncwarp();
        const int real = min(cols, 2 * N - c0);        // real (unpadded) columns in this chunk
        const int per_row = real / 4;
        // per_row is 2, 4 or 8 for the padded widths: shifts instead of divisions
        const int prs = (per_row & (per_row - 1)) == 0 ? __ffs(per_row) - 1 : -1;
        if (per_row > 0) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int idx = i * 32 + lane;
            const int row = prs >= 0 ? idx >> prs : idx / per_row;
            const int piece = idx - row * per_row;
            if (row < 32) {
              const uint4 val = *reinterpret_cast<const uint4*>(stg + row * TC_EPI_PITCH + piece * 16);
              *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(otile + (int64_t)row * N + c0 / 2) + piece * 16) = val;
            }
          }
        }
        __syncwarp();
      }
    }
    if (bulk && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (warp == TC_MMA_WARP) {
    // ---------------- MMA issuer (A from TMEM, B from smem) ----------------
    // The CTA owns all 512 columns, so its TMEM base is 0: a compile-time base
    // keeps every MMA operand warp-uniform (no per-MMA register broadcasts)
    if (tmem != 0u) __trap();
    const uint32_t tmem = 0u;
    const uint32_t idesc = tf32_idesc(Nr);
    const uint32_t idesc16 = (1u << 4) | ((uint32_t)(Nr >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t bhi = smem_u32(Bhi), blo = smem_u32(Blo);
    int it = 0;
    int64_t cur_z = z0;
    uint32_t bdone_phase = 0;
    // ring positions as counters (no div/mod on the issue path)
    const int NGm = (AS >= 4 && (RS == 0 || RS % 2 == 0)) ? 2 : 1;
    const int ASg = AS / NGm;
    int gpos[2] = {0, 0};
    uint32_t gph[2] = {0, 0};
    int acc = 0;
    uint32_t aph = 0;
    int64_t zt = z0, zleft = p.tiles_per_z - (g0 - z0 * p.tiles_per_z);
    for (int t = 0; t < ntiles; ++t) {
      if (zleft == 0) { ++zt; zleft = p.tiles_per_z; }
      --zleft;
      if (zt != cur_z) {
        if (lane == 0) umma_commit(bdone);
        __syncwarp();
        mbar_wait(bdone, bdone_phase);
        bdone_phase ^= 1;
        tc_fence_after();
        build_b<F16>(p, zt, Bhi, Blo, lane, 32);
        fence_proxy_async();
        __syncwarp();
        tc_fence_before();
        cur_z = zt;
      }
      mbar_wait_spin(&tempty[acc], aph ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + (uint32_t)(acc * Nr);
      const int g = NGm == 2 ? (t & 1) : 0;
      for (int c = 0; c < nchunk; ++c, ++it) {
        const int stage = g * ASg + gpos[g];
        const uint32_t ph = gph[g];
        if (++gpos[g] == ASg) { gpos[g] = 0; gph[g] ^= 1; }
        mbar_wait_spin(&full[stage], ph);
        tc_fence_after();
        if (F16 && elect_one()) {
          // chunk c = reals [2KC c, 2KC (c+1)) of K'; per 16-real k-step: one column group of 8
          const uint32_t SBO16 = (Kr / 8) * 128;
          const uint32_t ahi = tmem + A0 + (uint32_t)stage * ACOLS, alo = ahi + KC;
#pragma unroll
          for (int s = 0; s < KC / 8; ++s) {
            const uint32_t kb = (uint32_t)((2 * KC * c + 16 * s) / 8) * 128;   // byte offset along K'
            const uint64_t dbh = umma_desc(bhi + kb, 128, SBO16), dbl = umma_desc(blo + kb, 128, SBO16);
            const uint32_t first = (c == 0 && s == 0) ? 0u : 1u;
            mma_f16_tc(d, alo + 8 * s, dbh, idesc16, first);
            mma_f16_tc(d, ahi + 8 * s, dbl, idesc16, 1u);
            mma_f16_tc(d, ahi + 8 * s, dbh, idesc16, 1u);
          }
          umma_commit(&empty[stage]);
          if (c == nchunk - 1) umma_commit(&tfull[acc]);
        } else if (!F16 && elect_one()) {
          const uint32_t ahi = tmem + A0 + (uint32_t)stage * ACOLS, alo = ahi + 2 * KC;
          const uint64_t dbh0 = umma_desc(bhi + (uint32_t)(c * KC / 2) * 128, 128, SBO_B);
          const uint64_t dbl0 = umma_desc(blo + (uint32_t)(c * KC / 2) * 128, 128, SBO_B);
#pragma unroll
          for (int s = 0; s < KC / 4; ++s) {
            const uint64_t step = (uint64_t)(s * 256) >> 4;     // two 16-byte units of B' per k-step
            const uint32_t first = (c == 0 && s == 0) ? 0u : 1u;
            mma_tf32_ts(d, alo + 8 * s, dbh0 + step, idesc, first);   // small terms first
            mma_tf32_ts(d, ahi + 8 * s, dbl0 + step, idesc, 1u);
            mma_tf32_ts(d, ahi + 8 * s, dbh0 + step, idesc, 1u);
          }
          umma_commit(&empty[stage]);
          if (c == nchunk - 1) umma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
      if (++acc == TS) { acc = 0; aph ^= 1; }
    }
  } else if (warp == TC_PROD_WARP && RS > 0) {
    // ---------------- raw-ring producer: cp.async.bulk of each tile's segments ----------------
    // the whole warp issues: lane j copies segments j, j+32, ... (segment offsets
    // held in registers), so a tile of many small segments is not serialised
    // behind one thread's issue loop
    const uint32_t seg_bytes = (uint32_t)(p.Lseg * 8);
    const int nseg = (int)p.Kout;
    int64_t so[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = lane + 32 * u;
      so[u] = (p.segoff && j < nseg) ? p.segoff[j] : 0;
    }
    int rs = -1;
    uint32_t rph = 1;
    for (int t = 0; t < ntiles; ++t) {
      if (++rs == RS) rs = 0;
      if (rs == 0) rph ^= 1;
      mbar_wait_spin(&rempty[rs], rph ^ 1);
      unsigned char* dst = rawring + (size_t)rs * tc_raw_bytes(p.K);
      const float2* src = p.a + tbase[t];
      if (lane == 0) mbar_expect_tx(&rfull[rs], (uint32_t)(p.Kout * seg_bytes));
      __syncwarp();
      if (nseg <= 64) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int j = lane + 32 * u;
          if (j < nseg) bulk_g2s(dst + (size_t)j * seg_bytes, src + so[u], seg_bytes, &rfull[rs]);
        }
      } else {
        for (int j = lane; j < nseg; j += 32)
          bulk_g2s(dst + (size_t)j * seg_bytes, src + (p.segoff ? p.segoff[j] : 0), seg_bytes, &rfull[rs]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == TC_EPI_WARP0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// envelope of the tensor-core kernel
__host__ inline bool tc_shape_ok(int64_t K, int64_t N, int64_t M) {
  if (!(K == 4 || K == 8 || (K % 16) == 0) || K > 64) return false;
  if (N < 2 || N > 64 || (N % 2) != 0 || (N > 8 && (N % 8) != 0) || (M % 128) != 0 || M <= 0) return false;
  int TS, AS;
  tc_tmem_plan(K, tc_npad(N), TS, AS);
  return AS >= 2 && tc_smem_bytes(K, N, 64, 0) <= 227 * 1024;
}

// returns 0 if launched, -1 on launch error
__host__ inline int launch_tc(TcDesc p, int64_t Z, cudaStream_t s) {
  static uint64_t attr_done = 0;
  int adev = 0;
  if (attr_needed(attr_done, &adev)) {
    if (cudaFuncSetAttribute(k_tc_c64<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess ||
        cudaFuncSetAttribute(k_tc_c64<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess ||
        cudaFuncSetAttribute(k_tc_c64<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess ||
        cudaFuncSetAttribute(k_tc_c64<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess ||
        cudaFuncSetAttribute(k_tc_c64<8, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
      return -1;
    attr_done |= 1ull << (adev & 63);
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  p.tiles_per_z = p.M / 128;
  p.Z = Z;
  const int64_t total = Z * p.tiles_per_z;
  int64_t per = (total + sms - 1) / sms;
  if (per < 1) per = 1;
  while (per > 256 && tc_smem_bytes(p.K, p.N, per, 2) > 227 * 1024) per = (per + 1) / 2;
  p.per_cta = per;
  // raw ring (TMA bulk staging) when alignment allows and >= 2 stages fit
  p.raw_stages = 0;
  const bool aligned = (((uintptr_t)p.a) % 16 == 0) && ((p.a_zstride * 8) % 16 == 0);
  const bool use_raw = p.raw_ok && aligned;
  // bulk result stores: one full accumulator chunk per tile (2N = padded
  // width <= 32) and 16-byte aligned warp blocks; TNC_TC_BULKOUT=0 turns it off
  const char* ebo = getenv("TNC_TC_BULKOUT");
  const bool want_bulk = tc_npad(p.N) == p.N && !(ebo && ebo[0] == '0') &&
                         ((uintptr_t)p.out) % 16 == 0 && (p.out_zstride * 8) % 16 == 0 &&
                         (p.N <= 16 || (p.N % 16 == 0 && p.Z <= 0x7fffffff && p.M <= 0x7fffffff));
  // N >= 32: tensor map over the result, [Z][M][2N] fp32, box 32 floats x 32 rows
  CUtensorMap tmO;
  memset(&tmO, 0, sizeof tmO);
  bool tm_ok = false;
  if (want_bulk && p.N > 16 && p.K == 16) {
    tg_encode_fn enc = tg_encoder();
    if (enc) {
      const cuuint64_t gdim[3] = {(cuuint64_t)(2 * p.N), (cuuint64_t)p.M, (cuuint64_t)Z};
      const cuuint64_t gstr[2] = {(cuuint64_t)(p.N * 8), (cuuint64_t)((Z == 1 ? p.M * p.N : p.out_zstride) * 8)};
      const cuuint32_t box[3] = {32, 32, 1};
      const cuuint32_t es[3] = {1, 1, 1};
      tm_ok = Z == 1 || p.out_zstride >= p.M * p.N;
      tm_ok = tm_ok && enc(&tmO, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, p.out, gdim, gstr, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
  }
  p.bulk_out = 0;
  for (int bo = (want_bulk && (p.N <= 16 || tm_ok)) ? 1 : 0; bo >= 0; --bo) {
    p.raw_stages = 0;
    if (use_raw) {
      for (int rs = 4; rs >= 2; rs -= 2)
        if (tc_smem_bytes(p.K, p.N, per, rs, bo) <= 227 * 1024) { p.raw_stages = rs; break; }
      if (bo && p.raw_stages == 0) continue;     // the raw ring matters more than the store path
    }
    if (tc_smem_bytes(p.K, p.N, per, p.raw_stages, bo) <= 227 * 1024) { p.bulk_out = bo ? (p.N > 16 ? 2 : 1) : 0; break; }
  }
  if (tc_smem_bytes(p.K, p.N, per, p.raw_stages, p.bulk_out != 0) > 227 * 1024) return -1;
  p.nstages = 0;
  const size_t smem = (size_t)tc_smem_bytes(p.K, p.N, per, p.raw_stages, p.bulk_out != 0);
  const int64_t grid = (total + per - 1) / per;     // one wave when per fits in smem
  if (grid <= 0) return 0;
  const int kc = (int)tc_kc(p.K);
  // fp16-split operands (per-row A scales, per-z site scales) when the raw
  // ring holds whole tiles and the chunks are 16 complex (kind::f16 K = 16)
  int TS16, AS16;
  tc_tmem_plan(p.K, tc_npad(p.N), TS16, AS16, true);
  // (K = 16 only: one chunk per tile, so the row max comes from the values
  // being converted.  Opt-in, TNC_TC_F16=1: once the MMA issue was made
  // warp-uniform, 3xTF32 measured equal or faster on every K = 16 sweep case,
  // without the per-z scale pre-pass and with the smaller error.)
  const char* e16 = getenv("TNC_TC_F16");
  p.f16 = (kc == 16 && p.K == 16 && p.raw_stages > 0 && AS16 >= 2 && e16 && e16[0] == '1') ? 1 : 0;
  if (p.f16 && p.bulk_out == 2) p.bulk_out = 0;     // the tensor-store epilogue is a tf32-kernel instantiation
  float* bsc = nullptr;
  if (p.f16) {
    pool_keep();
    if (cudaMallocAsync(reinterpret_cast<void**>(&bsc), (size_t)Z * sizeof(float), s) != cudaSuccess) return -1;
    p.bscale = bsc;
    k_tc_bmax<<<(unsigned)std::min<int64_t>(Z, 4096), 128, 0, s>>>(p, bsc);
    k_tc_c64<8, true><<<(unsigned)grid, TC_THREADS, smem, s>>>(p, tmO);
    cudaFreeAsync(bsc, s);
  } else if (kc == 4) k_tc_c64<2, false><<<(unsigned)grid, TC_THREADS, smem, s>>>(p, tmO);
  else if (kc == 8) k_tc_c64<4, false><<<(unsigned)grid, TC_THREADS, smem, s>>>(p, tmO);
  else if (p.bulk_out == 2) k_tc_c64<8, false, true><<<(unsigned)grid, TC_THREADS, smem, s>>>(p, tmO);
  else k_tc_c64<8, false><<<(unsigned)grid, TC_THREADS, smem, s>>>(p, tmO);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// tnc_step entry: accumulator rows contiguous, result rows contiguous, complex64
template <typename R>
int try_tc(const tnc_step_desc& d, cudaStream_t s) {
  if constexpr (sizeof(R) != 4) {
    return 0;
  } else {
    if (!d.a_rows_contig || !d.c_rows_contig) return 0;
    if (!tc_shape_ok(d.K, d.N, d.M)) return 0;
    if (d.kernel == TNC_K_AUTO && d.K * d.N < 256) return 0;   // SIMT is HBM-bound there
    TcDesc p;
    memset(&p, 0, sizeof p);
    p.M = d.M; p.K = d.K; p.N = d.N;
    p.a = reinterpret_cast<const float2*>(d.acc);
    p.a_zstride = d.acc_zstride;
    p.nho = 1;
    p.ho_dim[0] = d.M / 128;
    p.ho_stride[0] = 128 * d.K;
    p.rows_contig = 1;
    p.raw_ok = 1;
    p.Kout = 1;
    p.Lseg = 128 * d.K;
    p.segoff = nullptr;
    p.site = d.site;
    p.slices_per_b = d.slices_per_b;
    p.s0 = d.s0;
    p.b_koff = d.b_koff;
    p.b_noff = d.b_noff;
    p.conj_b = d.conj_b;
    p.out = reinterpret_cast<float2*>(d.out);
    p.out_zstride = d.out_zstride;
    return launch_tc(p, d.Z, s) == 0 ? 1 : -1;
  }
}

}  // namespace tnc
