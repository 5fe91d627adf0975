// Tensor-core GEMM path for large engine steps (complex64): C[z] = A[z] S(z)
// with A row-contiguous [M][K] (the engine's due-ordered accumulator), K a
// multiple of 8, any N (tiled by NT <= 64 complex) and a general result map
// out = rowC(f) + c_noff[n] (the due-ordered result layout).
//
// The complex product runs on de-interleaved operands as two real products of
// width N = 2*NT into one accumulator D = [D_re | D_im]:
//   D += Ar [Br | Bi],   D += Ai [-Bi | Br],
// both windows of the three smem blocks [-Bi | Br | Bi] (3/4 of the bytes of
// the 2x2 real embedding, and MMAs of N = 128 -- the full-rate width; N = 64
// MMAs issue ~30% slower).  Each real product is 3xTF32 (lo*hi + hi*lo +
// hi*hi, fp32 accumulation in TMEM).
//
// F16 mode (amax_in given): the same three products on fp16 operands, which
// issue at twice the tf32 rate (kind::f16, K = 16 per MMA).  Every operand is
// scaled by a power of two before the split -- A by 2^(15 - e(max|A[z]|))
// from the producer's per-z amax, the site block by its own max -- so
// |x| < 2^15, hi = fp16(x), lo = fp16(x - hi) carry 22 significant bits like
// 3xTF32 (values below 2^-18 of the tensor max lose low bits of lo, which is
// below the fp32 rounding of the tensor's L2 norm).  The epilogue undoes the
// two scales exactly and, when asked, records max|out| per z for the next step.
//
// Data movement:
//  * A tiles (128 rows x KC complex) arrive by TMA (cp.async.bulk.tensor.3d,
//    128B/64B swizzle) in a raw smem ring; converter warps read them
//    conflict-free, split to tf32 hi/lo, de-interleave re/im and write the A
//    operand into TMEM (tcgen05.st).  Rows past M are zero-filled by TMA.
//  * Br/Bi hi/lo chunks (canonical K-major, prepared per call per distinct
//    site block by k_bprime) stream in by cp.async.bulk.
//  * Epilogue: tcgen05.ld of D_re / D_im -> complex; when the innermost
//    result leg is a new leg the tile is staged in padded smem and written
//    n-major with 16-byte stores, otherwise (innermost leg is a free leg)
//    per-row stores, which are then coalesced across lanes.
//
// Warps: 0-7 converters (each chunk: 4 lane quadrants x 2 K halves), 8-11 epilogue,
// 12 MMA issuer, 13 A producer (TMA), 14 B producer (bulk copies).
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include "tnc_tc.cuh"

namespace tnc {

struct GemmDesc {
  int64_t Z, M, K, N;
  int64_t tiles_m, per_cta, items;
  int32_t ilv, _pad5;            // 1: row tiles dealt round-robin over CTAs (neighbouring CTAs on neighbouring tiles)
  int32_t NT, tiles_n;           // complex columns per N tile (multiple of 16)
  int32_t KC, nchunk;            // complex K per chunk
  int32_t RS, BS;                // raw A stages, B stages
  const unsigned char* bp;       // [combo][tile_n][chunk][hi: -Bi|Br|Bi][lo: -Bi|Br|Bi][NT x KC] canonical
  int64_t bp_combo_stride;       // bytes per combo
  int32_t f16, cn_smem;          // 1: fp16 split operands (needs amax_in); c_noff staged in smem (int32)
  int32_t blk_contig, g3;        // blk_contig: every warp's 32 rows x 16 columns block is one contiguous 4 KB run;
                                 // g3: 3M (Gauss) complex products, F16 wide tiles (k_tc_gemm<16, true, true>)
  int64_t row_stride;            // != 0: rows r..r+31 of a warp block sit at oc(r) + i * row_stride
  const float* amax_in;          // [Z] max |re|,|im| of acc[z] (F16 scale)
  float* amax_out;               // [Z] max |re|,|im| of out[z] (zeroed by the host), or null
  const float* bscale;           // [combo] max |re|,|im| of the site block (F16)
  tnc_site site;                 // site blocks: combo -> offset
  const int64_t* b_koff;         // [K] site offsets
  const int64_t* b_noff;         // [N]
  int32_t conj_b, n_contig;      // n_contig: c_noff[n] == n
  int64_t slices_per_b, s0;
  float2* out;
  int64_t out_zstride;
  int32_t nf, c_rows_contig;
  int64_t f_dim[TNC_MAX_LEGS], f_cstride[TNC_MAX_LEGS];
  const int64_t* c_noff;         // [N]
  unsigned int* progress;        // pair kernel: items whose A loads have been issued, summed over CTAs (zeroed by the host)
  float comp;                    // 1 + TG_RZ_LOSS * (MMA accumulations per accumulator element), applied by the epilogue
  int32_t kseg;                  // pair kernel: chunks per K segment (TG2_KSEG)
};

// warps: converters [0, CONVW), epilogue [CONVW, MMA), MMA issuer, A and B producers;
// fp16-split tiles: 8 converter + 8 epilogue warps (19), 3xTF32: 8 + 4 (15 warps in all)
constexpr int TG_THREADS = 15 * 32;
constexpr int TG_THREADS_G3 = 19 * 32;
constexpr int TG_EPI_WARP0 = 8;
__host__ __device__ constexpr int tg_mma_warp(bool f16) { return f16 ? 16 : 12; }
constexpr int TG_MAX_RS = 8, TG_MAX_BS = 8;
constexpr int TG_EPI_PITCH = 16 * 8 + 16;      // staged row: 16 complex + 16 B pad

__device__ __forceinline__ int64_t gemm_combo(const GemmDesc& p, int64_t z) {
  const int64_t b = z / p.slices_per_b;
  const int64_t sl = p.s0 + (z - b * p.slices_per_b);
  int64_t c = p.site.sel ? (int64_t)p.site.sel[b] : 0;
  for (int j = 0; j < p.site.ncut; ++j) c = c * p.site.cut_ext[j] + (sl / p.site.cut_div[j]) % p.site.cut_ext[j];
  return c;
}

// bytes of one operand block (NT rows x KC k) -- fp32 or fp16 elements
__host__ __device__ inline int64_t tg_block_bytes(int NT, int KC, int f16) { return (int64_t)NT * KC * (f16 ? 2 : 4); }

// power-of-two scale s with max * s in [2^14, 2^15) (1 for a zero / non-finite max)
__device__ __forceinline__ float f16_scale(float amax) {
  if (!(amax > 0.f) || !(amax < 3.0e38f)) return 1.f;
  const int e = (int)((__float_as_uint(amax) >> 23) & 0xff) - 127;   // amax in [2^e, 2^(e+1))
  int p = 14 - e;
  p = p < -126 ? -126 : (p > 127 ? 127 : p);
  return __uint_as_float((uint32_t)(p + 127) << 23);
}
// 3M operands add re and im before the split (|re + im| < 2 max), so their
// scales leave one more bit of headroom
__device__ __forceinline__ float op_scale(float amax, int g3) { return g3 ? 0.5f * f16_scale(amax) : f16_scale(amax); }
__device__ __forceinline__ void split_f16(float y, uint16_t& h, uint16_t& l) {
  const __half hh = __float2half_rn(y);
  const __half ll = __float2half_rn(y - __half2float(hh));
  h = __half_as_ushort(hh);
  l = __half_as_ushort(ll);
}

// Two values -> packed fp16 hi and lo (low half = y0).  hi is rounded to 11
// significant bits in fp32 (integer add + mask, as split3) so lo = y - hi is
// exact and each pair needs one packed conversion per part instead of a
// round trip through fp16 per value.
__device__ __forceinline__ void split_f16x2(float y0, float y1, uint32_t& h, uint32_t& l) {
  const float h0 = __uint_as_float((__float_as_uint(y0) + 0x1000u) & 0xFFFFE000u);
  const float h1 = __uint_as_float((__float_as_uint(y1) + 0x1000u) & 0xFFFFE000u);
  const float l0 = y0 - h0, l1 = y1 - h1;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(h1), "f"(h0));
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(l1), "f"(l0));
}

// Two values -> packed fp16 hi and lo (low half = y0): hi by one packed
// conversion, converted back (one HADD2.F32 each) for lo = y - hi, which is
// exact in fp32 (6 instructions per pair; split_f16x2's integer rounding takes 8)
__device__ __forceinline__ void split_f16x2_cvt(float y0, float y1, uint32_t& h, uint32_t& l) {
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(y1), "f"(y0));
  const __half2 hh = *reinterpret_cast<const __half2*>(&h);
  const float l0 = y0 - __low2float(hh), l1 = y1 - __high2float(hh);
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(l1), "f"(l0));
}

// wait of a mostly idle role (epilogue on tfull): the hardware may suspend the
// thread for up to ~4 us per try_wait, so the poll loop takes no issue slots
// from the converter warps of its SM sub-partition
__device__ __forceinline__ void mbar_wait_idle(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)), "r"(phase), "r"(4000u) : "memory");
}

// tcgen05.mma adds each instruction's dot product to the fp32 accumulator with
// truncation (round toward zero), so every accumulation loses on average
// 1.6e-8 of the accumulator's magnitude (measured, tools/rz_bias_probe.py: the
// result of a step shrinks by 3.03e-9 K with 3 accumulations per 16 k (3M
// fp16), 6.04e-9 K with 6 (4M fp16), 1.21e-8 K with 6 per 8 k (3xTF32), for
// every tile shape).  Over the ~25 GEMM steps of a path the shrink adds up to
// 1e-4 of the amplitude, the whole complex64 tolerance; the epilogue scales
// the result by 1 + TG_RZ_LOSS * accumulations, which removes the mean loss.
constexpr float TG_RZ_LOSS = 1.616e-8f;

// per combo (blockIdx.x): max |re|, |im| over the site block (F16 scale of
// B'); blockIdx.y strides over K rows, atomicMax into the zeroed bscale
__global__ void k_bscale(const __grid_constant__ GemmDesc p, float* bscale) {
  const int64_t combo = blockIdx.x;
  int64_t off = 0, cc = combo;
  for (int j = p.site.ncut - 1; j >= 0; --j) {
    off += (cc % p.site.cut_ext[j]) * p.site.cut_stride[j];
    cc /= p.site.cut_ext[j];
  }
  off += cc * p.site.vstride;
  const float2* S = reinterpret_cast<const float2*>(p.site.ptr) + off;
  float m = 0.f;
  for (int64_t k = blockIdx.y; k < p.K; k += gridDim.y) {
    const float2* Sk = S + p.b_koff[k];
    for (int64_t n = threadIdx.x; n < p.N; n += blockDim.x) {
      const float2 v = Sk[p.b_noff[n]];
      m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
    }
  }
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(reinterpret_cast<unsigned int*>(bscale) + combo, __float_as_uint(m));
}

// Site operand for every (combo, N tile, K chunk): hi then lo, each three
// blocks [-Bi | Br | Bi] of NT rows (n) x KC cols (k), K-major canonical (8 x
// 16 B core matrices, LBO = 128 B along K, SBO = (KC/4) * 128 B along N).
// Consecutive blocks continue the 8-row-group sequence, so [Br | Bi] (blocks
// 1-2) and [-Bi | Br] (blocks 0-1) are both one N = 2*NT descriptor.
template <bool F16>
__global__ void k_bprime(const __grid_constant__ GemmDesc p, int64_t combos) {
  const int NT = p.NT, KC = p.KC;
  const int64_t bbytes = tg_block_bytes(NT, KC, F16);
  const uint32_t SBO = F16 ? (KC / 8) * 128 : (KC / 4) * 128;
  const int64_t per_combo = (int64_t)p.tiles_n * p.nchunk * NT * KC;
  const int64_t total = combos * per_combo;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t combo = e / per_combo;
    int64_t rem = e - combo * per_combo;
    const int64_t tn = rem / ((int64_t)p.nchunk * NT * KC);
    rem -= tn * p.nchunk * NT * KC;
    const int64_t c = rem / (NT * KC);
    rem -= c * NT * KC;
    const int nl = (int)(rem / KC), kl = (int)(rem - (int64_t)nl * KC);
    const int64_t n = tn * NT + nl, k = c * KC + kl;
    int64_t off = 0, cc = combo;
    for (int j = p.site.ncut - 1; j >= 0; --j) {
      off += (cc % p.site.cut_ext[j]) * p.site.cut_stride[j];
      cc /= p.site.cut_ext[j];
    }
    off += cc * p.site.vstride;
    float2 sv = make_float2(0.f, 0.f);
    if (n < p.N && k < p.K) {
      sv = reinterpret_cast<const float2*>(p.site.ptr)[off + p.b_koff[k] + p.b_noff[n]];
      if (p.conj_b) sv.y = -sv.y;
    }
    unsigned char* base = const_cast<unsigned char*>(p.bp) + combo * p.bp_combo_stride + ((tn * p.nchunk + c) * 6) * bbytes;
    if constexpr (F16) {
      const uint32_t boff = (nl & 7) * 16 + (nl >> 3) * SBO + (kl >> 3) * 128 + (kl & 7) * 2;
      const float t = op_scale(p.bscale[combo], p.g3);
      uint16_t rh, rl, ih, il;
      split_f16(sv.x * t, rh, rl);
      split_f16(sv.y * t, ih, il);
      if (p.g3) {
        // 3M: [Br | Bi | Br + Bi] hi, then lo (each block used alone, N = NT)
        uint16_t sh, sl;
        split_f16((sv.x + sv.y) * t, sh, sl);
        const uint16_t v[6] = {rh, ih, sh, rl, il, sl};
#pragma unroll
        for (int b = 0; b < 6; ++b) *reinterpret_cast<uint16_t*>(base + b * bbytes + boff) = v[b];
        continue;
      }
      const uint16_t v[6] = {(uint16_t)(ih ^ 0x8000u), rh, ih, (uint16_t)(il ^ 0x8000u), rl, il};
#pragma unroll
      for (int b = 0; b < 6; ++b) *reinterpret_cast<uint16_t*>(base + b * bbytes + boff) = v[b];
    } else {
      const uint32_t boff = (nl & 7) * 16 + (nl >> 3) * SBO + (kl >> 2) * 128 + (kl & 3) * 4;
      float rh, rl, ih, il;
      split3(sv.x, rh, rl);
      split3(sv.y, ih, il);
      const float v[6] = {-ih, rh, ih, -il, rl, il};
#pragma unroll
      for (int b = 0; b < 6; ++b) *reinterpret_cast<float*>(base + b * bbytes + boff) = v[b];
    }
  }
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}


__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// kind::f16 instruction descriptor: fp16 A/B (K-major), fp32 D, M = 128
__device__ __forceinline__ uint32_t f16_idesc(int n_real) {
  return (1u << 4) | ((uint32_t)(n_real >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// G3 (3M, Gauss): three real products per complex product instead of four --
// T1 = Ar Br, T2 = Ai Bi, T3 = (Ar + Ai)(Br + Bi) in three accumulators of NT
// columns, re = T1 - T2, im = T3 - T1 - T2 in the epilogue: 9 instead of 12
// N = NT MMA units per chunk (wide tiles, NT = 128, one accumulator stage)
template <int KC, bool F16, bool G3 = false>
__global__ void __launch_bounds__(F16 ? TG_THREADS_G3 : TG_THREADS, 1)
k_tc_gemm(const __grid_constant__ GemmDesc p, const __grid_constant__ CUtensorMap tmA) {
  static_assert(!F16 || KC == 16, "F16 mode needs 16-complex chunks (K = 16 per MMA)");
  static_assert(!G3 || F16, "3M products run on the fp16-split operands");
  extern __shared__ __align__(128) unsigned char smem_dyn[];
  constexpr int RB = KC * 8;                       // raw row bytes (KC complex)
  constexpr uint32_t SWM = RB == 128 ? 7u : 3u;    // swizzle row-group mask (128B / 64B)
  constexpr uint32_t RAW_BYTES = 128 * RB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NT = p.NT;
  const int nchunk = p.nchunk;
  const int RS = p.RS, BS = p.BS;
  const uint32_t bbytes = (uint32_t)tg_block_bytes(NT, KC, F16);   // one block (NT x KC)
  const uint32_t SBO_B = F16 ? (KC / 8) * 128 : (KC / 4) * 128;
  // TMEM: TS accumulators of [D_re NT | D_im NT], A stages of 4*KC (tf32) or
  // 2*KC (fp16: two values per column) columns
  constexpr uint32_t ACOLS = G3 ? 3 * KC : (F16 ? 2 * KC : 4 * KC);
  constexpr int NACC = G3 ? 3 : 2;                 // accumulator blocks of NT columns per stage
  // warp roles: converters [0, 8), epilogue [8, MMA) in EPIG groups of four
  // (one per TMEM lane quadrant; groups split the columns), then the MMA
  // issuer and the two producers.
  constexpr int TG_MMA_WARP = tg_mma_warp(F16), TG_APROD_WARP = TG_MMA_WARP + 1, TG_BPROD_WARP = TG_MMA_WARP + 2;
  constexpr int CONVW = 8;
  constexpr int EPIW = TG_MMA_WARP - CONVW;
  constexpr int EPIG = EPIW / 4;
  // narrow tiles (NT <= 32, short epilogue per item, latency-bound): the
  // epilogue groups alternate items instead of splitting columns, over four
  // accumulator stages
  const bool alt = F16 && !G3 && NT <= 32;
  // NT = 128 (F16, one N tile for N = 128): a single accumulator stage
  const int TS = alt ? 4 : (NT > 64 || G3 ? 1 : 2);
  // A-resident (ares): the whole converted 128 x K tile fits TMEM next to the
  // accumulators, so it is converted once per row tile and reused by all
  // tiles_n column tiles (stage = chunk; released after the last column tile)
  const bool ares = F16 && !G3 && p.tiles_n > 1 && TS * 2 * NT + nchunk * (int)ACOLS <= 512 && nchunk <= TC_MAX_STAGES;
  const int AS = ares ? nchunk : min(TC_MAX_STAGES, (512 - TS * NACC * NT) / (int)ACOLS);
  const uint32_t A0 = (uint32_t)(TS * NACC * NT);
  // smem: raw A ring (1024-aligned stages: swizzle atoms), B ring, epilogue staging, barriers
  unsigned char* araw = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  unsigned char* bring = araw + (size_t)RS * RAW_BYTES;
  unsigned char* estage = bring + (size_t)BS * 6 * bbytes;   // 1024-aligned (stage sizes are KB multiples)
  uint64_t* bar = reinterpret_cast<uint64_t*>(estage + EPIW * 32 * TG_EPI_PITCH);
  uint64_t* rfull = bar;                           // [RS] TMA -> converters
  uint64_t* rempty = rfull + TG_MAX_RS;            // [RS] converters -> TMA
  uint64_t* afull = rempty + TG_MAX_RS;            // [AS] converters -> MMA
  uint64_t* aempty = afull + TC_MAX_STAGES;        // [AS] MMA -> converters
  uint64_t* bfull = aempty + TC_MAX_STAGES;        // [BS]
  uint64_t* bempty = bfull + TG_MAX_BS;            // [BS]
  uint64_t* tfull = bempty + TG_MAX_BS;            // [TS <= 4]
  uint64_t* tempty = tfull + 4;                    // [TS <= 4]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);
  // result column offsets (int32) staged once per CTA: the per-row epilogue
  // reads one per value, and global loads there sit on its critical path
  int32_t* cn_s = reinterpret_cast<int32_t*>(tmem_slot + 4);   // 16-byte aligned
  if (p.cn_smem)
    for (int n = threadIdx.x; n < p.N; n += blockDim.x) cn_s[n] = (int32_t)p.c_noff[n];

  // items of this CTA: a contiguous range (ilv = 0), or whole row tiles
  // (groups of tiles_n items) dealt round-robin, so that at any moment the
  // CTAs stream neighbouring rows of A and of the result (DRAM page locality)
  // ilv == 2: items dealt one by one round-robin (item it of CTA b is
  // it * grid + b): the tiles_n column tiles of a row tile run on neighbouring
  // CTAs at the same time, so the A row tile is read from DRAM about once and
  // from L2 by the others (not with ares, which keeps a row tile per CTA)
  const int64_t G = p.Z * p.tiles_m;
  const int64_t w0 = p.ilv ? 0 : blockIdx.x * p.per_cta;
  const int nitems = p.ilv == 2 ? (int)((p.items - blockIdx.x + gridDim.x - 1) / gridDim.x)
                   : p.ilv ? (int)(((G - blockIdx.x + gridDim.x - 1) / gridDim.x) * p.tiles_n)
                           : (int)(min(w0 + p.per_cta, p.items) - w0);
  auto itemw = [&](int it) -> int64_t {
    if (!p.ilv) return w0 + it;
    if (p.ilv == 2) return (int64_t)it * gridDim.x + blockIdx.x;
    const int g = it / p.tiles_n;
    return ((int64_t)g * gridDim.x + blockIdx.x) * p.tiles_n + (it - g * p.tiles_n);
  };
  const int64_t per_z = p.tiles_m * p.tiles_n;
  // ares groups: consecutive items of one row tile (column tile index = w % tiles_n)
  auto gstart = [&](int it) { return it == 0 || itemw(it) % p.tiles_n == 0; };
  auto gend = [&](int it) { return it == nitems - 1 || itemw(it) % p.tiles_n == p.tiles_n - 1; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < RS; ++s) { mbar_init(&rfull[s], 1); mbar_init(&rempty[s], CONVW); }
    for (int s = 0; s < AS; ++s) { mbar_init(&afull[s], CONVW); mbar_init(&aempty[s], 1); }
    for (int s = 0; s < BS; ++s) { mbar_init(&bfull[s], 1); mbar_init(&bempty[s], 1); }
    for (int s = 0; s < TS; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], alt ? 4 : EPIW); }
    mbar_fence_init();
  }
  if (warp == TG_EPI_WARP0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < CONVW) {
    // ---------------- converters: raw smem -> tf32/fp16 hi/lo -> TMEM ----------------
    // warp w converts rows 32*(w%4).. (its TMEM lane quadrant), complex
    // [h*KC/2, (h+1)*KC/2) with h = w/4.
    const int h = warp >> 2;
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    constexpr int KH = KC / 2;                     // complex per warp
    int j = 0;
    int rstage = 0, astage = 0;
    uint32_t rph = 0, aph = 0;
    float sA = 1.f;
    int64_t sz = -1;                             // z whose scale sA holds (z changes rarely)
    for (int it = 0; it < nitems; ++it) {
      if (ares && !gstart(it)) continue;
      if constexpr (F16) {
        const int64_t zz = itemw(it) / per_z;
        if (zz != sz) { sz = zz; sA = op_scale(__ldg(p.amax_in + zz), G3); }
      }
      for (int c = 0; c < nchunk; ++c, ++j) {
        mbar_wait_spin(&rfull[rstage], rph);
        const uint32_t src = smem_u32(araw + (size_t)rstage * RAW_BYTES);
        if constexpr (G3) {
          // warp (quadrant, half h): complex [8h, 8h + 8) of its 32 rows ->
          // Ar, Ai, As = Ar + Ai, hi/lo fp16, two per TMEM column (4 per plane)
          uint32_t rh[4], ih[4], sh[4], rl[4], il[4], sl[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t off = (uint32_t)(r * RB + 16 * (4 * h + q));
            const uint32_t phys = off ^ (((off >> 7) & SWM) << 4);
            float4 x;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "r"(src + phys));
            const float r0 = x.x * sA, i0 = x.y * sA, r1 = x.z * sA, i1 = x.w * sA;
            split_f16x2_cvt(r0, r1, rh[q], rl[q]);
            split_f16x2_cvt(i0, i1, ih[q], il[q]);
            split_f16x2_cvt(r0 + i0, r1 + i1, sh[q], sl[q]);
          }
          mbar_wait_spin(&aempty[astage], aph ^ 1);
          tc_fence_after();
          // stage layout: [Ar_hi | Ai_hi | As_hi | Ar_lo | Ai_lo | As_lo], 8 columns each
          const uint32_t col = A0 + (uint32_t)astage * ACOLS + 4 * h;
          tmem_st<4>(tmem + lane_base + col, rh);
          tmem_st<4>(tmem + lane_base + col + 8, ih);
          tmem_st<4>(tmem + lane_base + col + 16, sh);
          tmem_st<4>(tmem + lane_base + col + 24, rl);
          tmem_st<4>(tmem + lane_base + col + 32, il);
          tmem_st<4>(tmem + lane_base + col + 40, sl);
        } else if constexpr (F16) {
          // warp (quadrant, half h): complex [8h, 8h + 8) of its 32 rows -> Ar, Ai
          // hi/lo fp16, two per TMEM column (4 per plane)
          uint32_t rh[4], ih[4], rl[4], il[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t off = (uint32_t)(r * RB + 16 * (4 * h + q));
            const uint32_t phys = off ^ (((off >> 7) & SWM) << 4);
            float4 x;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "r"(src + phys));
            split_f16x2_cvt(x.x * sA, x.z * sA, rh[q], rl[q]);   // re of complex 2q, 2q+1
            split_f16x2_cvt(x.y * sA, x.w * sA, ih[q], il[q]);   // im
          }
          mbar_wait_spin(&aempty[astage], aph ^ 1);
          tc_fence_after();
          // stage layout: [Ar_hi 8 | Ai_hi 8 | Ar_lo 8 | Ai_lo 8] columns (16 k each)
          const uint32_t col = A0 + (uint32_t)astage * ACOLS + 4 * h;
          tmem_st<4>(tmem + lane_base + col, rh);
          tmem_st<4>(tmem + lane_base + col + 8, ih);
          tmem_st<4>(tmem + lane_base + col + 16, rl);
          tmem_st<4>(tmem + lane_base + col + 24, il);
        }
        if constexpr (F16) {
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive_warp(&afull[astage]);
          fence_proxy_async();
          mbar_arrive_warp(&rempty[rstage]);
          if (++rstage == RS) { rstage = 0; rph ^= 1; }
          if (++astage == AS) { astage = 0; aph ^= 1; }
          continue;
        }
        uint32_t rh[KH], ih[KH], rl[KH], il[KH];
#pragma unroll
        for (int q = 0; q < KH / 2; ++q) {         // 16-byte piece: complex 2q, 2q+1 of this half
          const uint32_t off = (uint32_t)(r * RB + 16 * (h * KH / 2 + q));
          const uint32_t phys = off ^ (((off >> 7) & SWM) << 4);
          float4 x;
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "r"(src + phys));
          float hh, ll;
          split3(x.x, hh, ll); rh[2 * q] = __float_as_uint(hh);     rl[2 * q] = __float_as_uint(ll);
          split3(x.y, hh, ll); ih[2 * q] = __float_as_uint(hh);     il[2 * q] = __float_as_uint(ll);
          split3(x.z, hh, ll); rh[2 * q + 1] = __float_as_uint(hh); rl[2 * q + 1] = __float_as_uint(ll);
          split3(x.w, hh, ll); ih[2 * q + 1] = __float_as_uint(hh); il[2 * q + 1] = __float_as_uint(ll);
        }
        mbar_wait_spin(&aempty[astage], aph ^ 1);
        tc_fence_after();
        // stage layout per 8-k step s: [Ar_hi 8 | Ai_hi 8 | Ar_lo 8 | Ai_lo 8]
        const uint32_t k0 = (uint32_t)(h * KH);
        const uint32_t col = A0 + (uint32_t)astage * ACOLS + (k0 / 8) * 32 + (k0 % 8);
        tmem_st<KH>(tmem + lane_base + col, rh);
        tmem_st<KH>(tmem + lane_base + col + 8, ih);
        tmem_st<KH>(tmem + lane_base + col + 16, rl);
        tmem_st<KH>(tmem + lane_base + col + 24, il);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive_warp(&afull[astage]);
        // release the raw stage only once its values have certainly been
        // consumed (the shared loads can still be in flight when an earlier
        // arrive retires, and the next TMA write would race them); the proxy
        // fence orders these generic-proxy reads before the async-proxy refill
        fence_proxy_async();
        mbar_arrive_warp(&rempty[rstage]);
        if (++rstage == RS) { rstage = 0; rph ^= 1; }
        if (++astage == AS) { astage = 0; aph ^= 1; }
      }
    }
  } else if (warp < TG_MMA_WARP) {
    // ---------------- epilogue: TMEM -> complex -> result ----------------
    const int q = warp & 3;                      // TMEM lane quadrant (CONVW is a multiple of 4)
    const int eg = (warp - CONVW) >> 2;          // column group
    const int r = q * 32 + lane;
    unsigned char* stg = estage + (size_t)(warp - CONVW) * 32 * TG_EPI_PITCH;
    // staged n-major stores when the innermost result leg is a new leg (runs
    // of consecutive n are contiguous); per-row stores otherwise (then the
    // innermost result leg is a free leg: consecutive rows are contiguous)
    const bool staged = (p.c_rows_contig || p.n_contig || (p.N > 1 && p.c_noff[1] == p.c_noff[0] + 1));
    const int cfirst = alt ? 0 : eg * 16, cstep = alt ? 16 : 16 * EPIG;
    float inv = p.comp, inv2 = 1.f;
    int64_t inv_z = -1;
    const uint32_t stg_s = smem_u32(stg);
    for (int it = alt ? eg : 0; it < nitems; it += alt ? EPIG : 1) {
      const int acc = it % TS;
      const uint32_t ph = (it / TS) & 1;
      int64_t z, mt, nt;
      {
        const int64_t w = itemw(it);
        if (p.items < 0x7fffffffLL) {
          const uint32_t w32 = (uint32_t)w, pz = (uint32_t)per_z, tn = (uint32_t)p.tiles_n;
          const uint32_t z32 = w32 / pz, rem = w32 - z32 * pz, m32 = rem / tn;
          z = z32; mt = m32; nt = rem - m32 * tn;
        } else {
          z = w / per_z;
          const int64_t rem = w - z * per_z;
          mt = rem / p.tiles_n; nt = rem - mt * p.tiles_n;
        }
      }
      const int64_t row = mt * 128 + r;
      int64_t oc = row * p.N;
      if (!p.c_rows_contig && row < p.M) {
        uint32_t f = (uint32_t)row;              // M < 2^31 (try_tc_gemm): 32-bit divisions
        oc = 0;
        for (int jj = p.nf - 1; jj >= 0; --jj) {
          const uint32_t dd = (uint32_t)p.f_dim[jj];
          const uint32_t qq = f / dd;
          oc += (int64_t)(f - qq * dd) * p.f_cstride[jj];
          f = qq;
        }
      }
      float2* O = p.out + z * p.out_zstride;
      const int64_t n0 = nt * NT;
      float vmax = 0.f;
      if constexpr (F16) {
        if (z != inv_z) {                        // the per-z scales change rarely: reload only then
          inv_z = z;
          // two exact power-of-two factors: their product can leave the fp32 range
          // when both tensors are tiny although every result is representable
          inv = p.comp / op_scale(__ldg(p.amax_in + z), G3);
          inv2 = 1.f / op_scale(__ldg(p.bscale + gemm_combo(p, z)), G3);
        }
      }
      if constexpr (G3) mbar_wait_idle(&tfull[acc], ph);
      else mbar_wait(&tfull[acc], ph);
      tc_fence_after();
      const uint32_t tre = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * NACC * NT);
      if (cfirst >= NT) {                         // no columns for this group
        tc_fence_before();
        mbar_arrive_warp(&tempty[acc]);
      }
      float2* Orow = O + oc;
      for (int c0 = cfirst; c0 < NT; c0 += cstep) {
        uint32_t vr[16], vi[16];
        tmem_ld16(tre + c0, vr);
        tmem_ld16(tre + NT + c0, vi);
        if constexpr (G3) {
          uint32_t v3[16];
          tmem_ld16(tre + 2 * NT + c0, v3);
          tmem_wait_ld();
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {        // re = T1 - T2, im = T3 - T1 - T2
            const float t1 = __uint_as_float(vr[jj]), t2 = __uint_as_float(vi[jj]);
            vr[jj] = __float_as_uint(t1 - t2);
            vi[jj] = __float_as_uint(__uint_as_float(v3[jj]) - t1 - t2);
          }
        } else {
          tmem_wait_ld();
        }
        if (c0 + cstep >= NT) {
          tc_fence_before();
          mbar_arrive_warp(&tempty[acc]);
        }
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const float a = __uint_as_float(vr[jj]) * inv * inv2, b = __uint_as_float(vi[jj]) * inv * inv2;
          vmax = fmaxf(vmax, fmaxf(fabsf(a), fabsf(b)));
          vr[jj] = __float_as_uint(a);
          vi[jj] = __float_as_uint(b);
        }
        const int64_t nleft = p.N - (n0 + c0);
        const int ncols = nleft < 16 ? (int)nleft : 16;
        if (staged) {
          // stage the warp's 32 rows x 16 complex, then 8 lanes per row write
          // 16-byte pieces: runs of consecutive n are contiguous in the result
#pragma unroll
          for (int jj = 0; jj < 16; jj += 2) {
            const float4 v = make_float4(__uint_as_float(vr[jj]), __uint_as_float(vi[jj]),
                                         __uint_as_float(vr[jj + 1]), __uint_as_float(vi[jj + 1]));
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(stg_s + lane * TG_EPI_PITCH + jj * 8),
                         "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
          }
          __syncwarp();
          if (p.blk_contig && ncols == 16 && mt * 128 + q * 32 + 32 <= p.M) {
            // the warp's 32 rows x 16 columns are one contiguous 4 KB run:
            // eight fully coalesced 512-byte stores, no per-row addressing
            const int64_t oc0 = __shfl_sync(0xffffffffu, oc, 0);
            float4* dst = reinterpret_cast<float4*>(O + oc0 + (p.c_rows_contig ? n0 + c0 : (int64_t)cn_s[n0 + c0]));
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int c = i * 32 + lane;
              float4 v;
              asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                           : "r"(stg_s + (c >> 3) * TG_EPI_PITCH + (c & 7) * 16) : "memory");
              dst[c] = v;
            }
            __syncwarp();
            continue;
          }
          const int sub = lane & 7;                // 16-byte piece (2 complex) of a row
          const int64_t n = n0 + c0 + 2 * sub;
          int64_t a0 = 0, a1 = 0;
          if (2 * sub < ncols) a0 = p.c_rows_contig ? n : (p.cn_smem ? cn_s[n] : p.c_noff[n]);
          if (2 * sub + 1 < ncols) a1 = p.c_rows_contig ? n + 1 : (p.cn_smem ? cn_s[n + 1] : p.c_noff[n + 1]);
          // rows of a warp at one stride (innermost free leg >= 32 rows): no shuffles
          const int64_t oc0 = p.row_stride ? __shfl_sync(0xffffffffu, oc, 0) : 0;
#pragma unroll
          for (int rr = 0; rr < 32; rr += 4) {
            const int lr = rr + (lane >> 3);
            const int64_t grow = mt * 128 + q * 32 + lr;
            const int64_t ocr = p.row_stride ? oc0 + (int64_t)lr * p.row_stride : __shfl_sync(0xffffffffu, oc, lr);
            if (grow < p.M && 2 * sub < ncols) {
              float4 v;
              asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                           : "r"(stg_s + lr * TG_EPI_PITCH + sub * 16) : "memory");
              float2* dst = O + ocr + a0;
              if (2 * sub + 1 < ncols && a1 == a0 + 1 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                *reinterpret_cast<float4*>(dst) = v;
              } else {
                dst[0] = make_float2(v.x, v.y);
                if (2 * sub + 1 < ncols) O[ocr + a1] = make_float2(v.z, v.w);
              }
            }
          }
          __syncwarp();
        } else if (row < p.M) {
          if (p.cn_smem && ncols == 16) {
            // 16 result offsets by four broadcast 16-byte shared loads; 32-bit indices
            const int4* cq = reinterpret_cast<const int4*>(cn_s + n0 + c0);
            int cidx[16];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int4 t4 = cq[u];
              cidx[4 * u] = t4.x; cidx[4 * u + 1] = t4.y; cidx[4 * u + 2] = t4.z; cidx[4 * u + 3] = t4.w;
            }
#pragma unroll
            for (int jj = 0; jj < 16; ++jj)
              Orow[cidx[jj]] = make_float2(__uint_as_float(vr[jj]), __uint_as_float(vi[jj]));
          } else {
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              if (jj < ncols) {
                const int64_t n = n0 + c0 + jj;
                O[oc + (p.cn_smem ? (int64_t)cn_s[n] : p.c_noff[n])] = make_float2(__uint_as_float(vr[jj]), __uint_as_float(vi[jj]));
              }
            }
          }
        }
      }
      if (p.amax_out) {                          // rows past M / padded columns hold zeros
        for (int o = 16; o; o >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        if (lane == 0 && vmax > 0.f) atomicMax(reinterpret_cast<unsigned int*>(p.amax_out) + z, __float_as_uint(vmax));
      }
    }
  } else if (warp == TG_MMA_WARP) {
    // ---------------- MMA issuer ----------------
    // all 512 columns are this CTA's, so the TMEM base is 0: a compile-time base
    // keeps the MMA operands warp-uniform (see k_tc_c64)
    if (tmem != 0u) __trap();
    const uint32_t tmem = 0u;
    const uint32_t idesc = F16 ? f16_idesc(G3 ? NT : 2 * NT) : tf32_idesc(2 * NT);
    // ring positions kept as counters (no div/mod on the issue path: at F16
    // rates the issuer's own instruction latency is what starves the pipe)
    int bs = 0, stage = 0, acc = 0, stage0 = 0;
    uint32_t bph = 0, aph = 0, tph = 0, aph0 = 0;
    const uint64_t dB = umma_desc(smem_u32(bring), 128, SBO_B);   // + (byte offset >> 4) per block
    const uint32_t bstage16 = (6 * bbytes) >> 4, bblk16 = bbytes >> 4;
    for (int it = 0; it < nitems; ++it) {
      mbar_wait_spin(&tempty[acc], tph ^ 1);
      tc_fence_after();
      const uint32_t dre = tmem + (uint32_t)(acc * NACC * NT);
      const bool gs = !ares || gstart(it), ge = !ares || gend(it);
      if (gs) { stage0 = stage; aph0 = aph; }
      else { stage = stage0; aph = aph0; }         // ares: the group's stages again, same phase
      for (int c = 0; c < nchunk; ++c) {
        if (gs) mbar_wait_spin(&afull[stage], aph);
        mbar_wait_spin(&bfull[bs], bph);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t bb = dB + (uint64_t)(bs * bstage16);
          const uint64_t b2h = bb, b1h = bb + bblk16, b2l = bb + 3 * bblk16, b1l = bb + 4 * bblk16;
          if constexpr (G3) {
            // blocks [Br | Bi | Bs] hi then lo; small terms first, then hi*hi
            const uint32_t arh = tmem + A0 + (uint32_t)stage * ACOLS;
            const uint32_t aih = arh + 8, ash = arh + 16, arl = arh + 24, ail = arh + 32, asl = arh + 40;
            const uint64_t brh = bb, bih = bb + bblk16, bsh = bb + 2 * bblk16;
            const uint64_t brl = bb + 3 * bblk16, bil = bb + 4 * bblk16, bsl = bb + 5 * bblk16;
            const uint32_t first = c == 0 ? 0u : 1u;
            const uint32_t d1 = dre, d2 = dre + (uint32_t)NT, d3 = dre + 2u * (uint32_t)NT;
            mma_f16_ts(d1, arl, brh, idesc, first);
            mma_f16_ts(d2, ail, bih, idesc, first);
            mma_f16_ts(d3, asl, bsh, idesc, first);
            mma_f16_ts(d1, arh, brl, idesc, 1u);
            mma_f16_ts(d2, aih, bil, idesc, 1u);
            mma_f16_ts(d3, ash, bsl, idesc, 1u);
            mma_f16_ts(d1, arh, brh, idesc, 1u);
            mma_f16_ts(d2, aih, bih, idesc, 1u);
            mma_f16_ts(d3, ash, bsh, idesc, 1u);
          } else if constexpr (F16) {
            const uint32_t arh = tmem + A0 + (uint32_t)stage * ACOLS;
            const uint32_t aih = arh + 8, arl = arh + 16, ail = arh + 24;
            const uint32_t first = c == 0 ? 0u : 1u;
            mma_f16_ts(dre, arl, b1h, idesc, first);
            mma_f16_ts(dre, ail, b2h, idesc, 1u);
            mma_f16_ts(dre, arh, b1l, idesc, 1u);
            mma_f16_ts(dre, aih, b2l, idesc, 1u);
            mma_f16_ts(dre, arh, b1h, idesc, 1u);
            mma_f16_ts(dre, aih, b2h, idesc, 1u);
          }
#pragma unroll
          for (int s = 0; s < (F16 ? 0 : KC / 8); ++s) {
            const uint64_t st = (uint64_t)(s * 256) >> 4;   // 8 k = 2 core matrices = 256 B
            const uint32_t arh = tmem + A0 + (uint32_t)stage * ACOLS + 32 * s;
            const uint32_t aih = arh + 8, arl = arh + 16, ail = arh + 24;
            const uint32_t first = (c == 0 && s == 0) ? 0u : 1u;
            // small terms first (lo*hi, hi*lo), then hi*hi
            mma_tf32_ts(dre, arl, b1h + st, idesc, first);
            mma_tf32_ts(dre, ail, b2h + st, idesc, 1u);
            mma_tf32_ts(dre, arh, b1l + st, idesc, 1u);
            mma_tf32_ts(dre, aih, b2l + st, idesc, 1u);
            mma_tf32_ts(dre, arh, b1h + st, idesc, 1u);
            mma_tf32_ts(dre, aih, b2h + st, idesc, 1u);
          }
          if (ge) umma_commit(&aempty[stage]);
          umma_commit(&bempty[bs]);
          if (c == nchunk - 1) umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++bs == BS) { bs = 0; bph ^= 1; }
        if (++stage == AS) { stage = 0; aph ^= 1; }
      }
      if (++acc == TS) { acc = 0; tph ^= 1; }
    }
  } else if (warp == TG_APROD_WARP && lane == 0) {
    // ---------------- A producer: TMA tiles into the group's raw slice ----------------
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    int j = 0, rs = 0;
    uint32_t rph = 0;
    for (int it = 0; it < nitems; ++it) {
      if (ares && !gstart(it)) continue;
      const int64_t w = itemw(it);
      const int64_t z = w / per_z;
      const int64_t mt = (w - z * per_z) / p.tiles_n;
      for (int c = 0; c < nchunk; ++c, ++j) {
        mbar_wait_spin(&rempty[rs], rph ^ 1);
        mbar_expect_tx(&rfull[rs], RAW_BYTES);
        tma_load_3d(araw + (size_t)rs * RAW_BYTES, &tmA, c * 2 * KC, (int)(mt * 128), (int)z, &rfull[rs]);
        if (++rs == RS) { rs = 0; rph ^= 1; }
      }
    }
  } else if (warp == TG_BPROD_WARP && lane == 0) {
    // ---------------- B producer: Br/Bi hi/lo chunks ----------------
    int bi = 0, bs = 0;
    uint32_t bph = 0;
    for (int it = 0; it < nitems; ++it) {
      const int64_t w = itemw(it);
      const int64_t z = w / per_z;
      const int64_t nt = (w - z * per_z) % p.tiles_n;
      const unsigned char* src = p.bp + gemm_combo(p, z) * p.bp_combo_stride + (int64_t)nt * nchunk * 6 * bbytes;
      for (int c = 0; c < nchunk; ++c, ++bi) {
        mbar_wait_spin(&bempty[bs], bph ^ 1);
        mbar_expect_tx(&bfull[bs], 6 * bbytes);
        bulk_g2s(bring + (size_t)bs * 6 * bbytes, src + (int64_t)c * 6 * bbytes, 6 * bbytes, &bfull[bs]);
        if (++bs == BS) { bs = 0; bph ^= 1; }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == TG_EPI_WARP0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

}  // namespace tnc
#include "tnc_tcgemm2.cuh"
namespace tnc {

__host__ inline size_t tg_smem_bytes(int NT, int KC, int RS, int BS, int f16, int64_t cn = 0) {
  return 1024 + (size_t)RS * 128 * KC * 8 + (size_t)BS * 6 * tg_block_bytes(NT, KC, f16) +
         (size_t)(f16 ? 8 : 4) * 32 * TG_EPI_PITCH +
         8 * (2 * TG_MAX_RS + 2 * TC_MAX_STAGES + 2 * TG_MAX_BS + 8) + 16 + 4 * cn;
}

// tg_encode_fn / tg_encoder(): tnc_tc.cuh

// complex64 GEMM steps with an input bound (amax_in) run on fp16-split operands
inline bool tc16_enabled() { return true; }

// engine step on the GEMM path; returns 1 launched, 0 not applicable, -1 error
// (when launched with amax_out set, the epilogue has recorded max |out| per z)
template <typename R>
int try_tc_gemm(const tnc_step_desc& d, cudaStream_t s) {
  if constexpr (sizeof(R) != 4) {
    return 0;
  } else {
    if (!d.a_rows_contig || d.K * d.N < 256) return 0;
    if (d.Z * ((d.M + 127) / 128) < 64) return 0;     // too few row tiles to fill the GPU
    int KC;
    if (d.K % 16 == 0) KC = 16;
    else if (d.K == 8) KC = 8;
    else return 0;
    int64_t combos = 1;
    if (d.site.sel) {
      if (d.site.nvariants <= 0) return 0;
      combos = d.site.nvariants;
    }
    for (int j = 0; j < d.site.ncut; ++j) combos *= d.site.cut_ext[j];
    if (d.site.zstride != 0 || combos > 4096 || d.nf > TNC_MAX_LEGS) return 0;
    if ((((uintptr_t)d.acc) % 16) || (d.acc_zstride % 2)) return 0;
    if (d.M > 0x7fffffffLL || d.Z > 0x7fffffffLL || 2 * d.K > 0x7fffffffLL) return 0;
    tg_encode_fn enc = tg_encoder();
    if (!enc) return 0;
    GemmDesc p;
    memset(&p, 0, sizeof p);
    p.Z = d.Z; p.M = d.M; p.K = d.K; p.N = d.N;
    p.NT = d.N >= 64 ? 64 : (int)((d.N + 15) / 16 * 16);
    p.tiles_n = (int)((d.N + p.NT - 1) / p.NT);
    p.KC = KC;
    p.nchunk = (int)(d.K / KC);
    p.tiles_m = (d.M + 127) / 128;
    p.site = d.site;
    p.b_koff = d.b_koff; p.b_noff = d.b_noff;
    p.conj_b = d.conj_b;
    p.slices_per_b = d.slices_per_b; p.s0 = d.s0;
    p.out = reinterpret_cast<float2*>(d.out);
    p.out_zstride = d.out_zstride;
    p.nf = d.nf;
    p.c_rows_contig = d.c_rows_contig;
    for (int j = 0; j < d.nf; ++j) { p.f_dim[j] = d.f_dim[j]; p.f_cstride[j] = d.f_cstride[j]; }
    p.c_noff = d.c_noff;
    p.n_contig = (d.c_rows_contig || d.c_n_contig) ? 1 : 0;
    p.amax_out = d.amax_out;
    const int f16 = (d.amax_in != nullptr && KC == 16 && tc16_enabled()) ? 1 : 0;
    p.f16 = f16;
    p.amax_in = f16 ? d.amax_in : nullptr;
    // F16, N >= 128: 128-wide column tiles (N = 256 MMAs: the issuer's
    // per-chunk overhead stays below the MMA time), one accumulator stage; for
    // K <= 128 the converted A tile stays resident across column tiles
    if (f16 && d.N >= 128) {
      p.NT = 128;
      p.tiles_n = (int)((d.N + p.NT - 1) / p.NT);
    }
    // same decisions as the kernel: A-resident 4M tiles for K <= 128 with
    // several column tiles, 3M (Gauss) products on the other 128-wide F16 tiles
    bool ares = false;
    {
      const bool alt = f16 && p.NT <= 32;
      const int TS = alt ? 4 : (p.NT > 64 ? 1 : 2);
      const int acols = f16 ? 2 * KC : 4 * KC;
      ares = f16 && p.tiles_n > 1 && TS * 2 * p.NT + p.nchunk * acols <= 512 && p.nchunk <= TC_MAX_STAGES;
    }
    p.g3 = (f16 && p.NT == 128 && !ares) ? 1 : 0;
    // accumulations into each accumulator element over the K loop (see TG_RZ_LOSS)
    p.comp = 1.f + TG_RZ_LOSS * (float)(f16 ? (d.K / 16) * (p.g3 ? 3 : 6) : (d.K / 8) * 6);
    // stages: fill the shared-memory budget
    int RS = 4, BS = 3;
    const size_t budget = 226 * 1024;
    // the staged column offsets are int32: they fit when the result of one z does,
    // or when the new legs' own extents and strides say so (2^32+-element results)
    bool cn_fits = d.out_zstride < 0x7fffffffLL;
    if (!cn_fits && d.nn > 0) {
      int64_t mx = 0;
      for (int j = 0; j < d.nn; ++j) mx += (d.n_dim[j] - 1) * d.n_cstride[j];
      cn_fits = mx < 0x7fffffffLL;
    }
    p.cn_smem = (!d.c_rows_contig && d.N <= 1024 && cn_fits) ? 1 : 0;
    // contiguous 32 x 16 blocks: innermost free leg (>= 32 rows) at stride 16 and
    // 16 consecutive columns contiguous (innermost new leg of extent % 16 == 0 at stride 1)
    p.blk_contig = 0;
    p.row_stride = (d.c_rows_contig && d.M % 32 == 0) ? d.N
                   : ((d.nf >= 1 && d.f_dim[d.nf - 1] % 32 == 0) ? d.f_cstride[d.nf - 1] : 0);
    if (d.nf >= 1 && d.f_dim[d.nf - 1] % 32 == 0 && d.f_cstride[d.nf - 1] == 16 && d.M % 128 == 0) {
      if (d.c_rows_contig && d.N == 16) p.blk_contig = 1;
      else if (!d.c_rows_contig && p.cn_smem && d.nn > 0 && d.n_dim[d.nn - 1] % 16 == 0 && d.n_cstride[d.nn - 1] == 1)
        p.blk_contig = 1;
    }
    const int64_t cn = p.cn_smem ? d.N : 0;
    while (RS + 1 <= TG_MAX_RS && tg_smem_bytes(p.NT, KC, RS + 1, BS, f16, cn) <= budget) ++RS;
    while (BS + 1 <= TG_MAX_BS && tg_smem_bytes(p.NT, KC, RS, BS + 1, f16, cn) <= budget) ++BS;
    if (tg_smem_bytes(p.NT, KC, RS, BS, f16, cn) > budget) return 0;
    p.RS = RS; p.BS = BS;
    // A: [Z][M][2K floats] with row pitch K complex, batch pitch acc_zstride complex
    CUtensorMap tm;
    const cuuint64_t gdim[3] = {(cuuint64_t)(2 * d.K), (cuuint64_t)d.M, (cuuint64_t)d.Z};
    const cuuint64_t gstr[2] = {(cuuint64_t)(d.K * 8), (cuuint64_t)(d.acc_zstride * 8)};
    const cuuint32_t box[3] = {(cuuint32_t)(2 * KC), 128u, 1u};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(d.acc), gdim, gstr, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, KC == 16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 0;
    p.bp_combo_stride = (int64_t)p.tiles_n * p.nchunk * 6 * tg_block_bytes(p.NT, KC, f16);
    const bool pair = tg2_applicable(p);
    if (pair) {
      // pair kernel: 96 KB result stage, 12 KB B' half stages
      p.cn_smem = (!d.c_rows_contig && d.N <= 2048 && cn_fits) ? 1 : 0;
      const int64_t cn2 = p.cn_smem ? d.N : 0;
      RS = 3; BS = 3;
      while (RS + 1 <= TG2_MAX_RS && RS < 5 && tg2_smem_bytes(RS + 1, BS, cn2) <= budget) ++RS;
      while (BS + 1 <= TG2_MAX_BS && tg2_smem_bytes(RS, BS + 1, cn2) <= budget) ++BS;
      while (RS + 1 <= TG2_MAX_RS && tg2_smem_bytes(RS + 1, BS, cn2) <= budget) ++RS;
      if (tg2_smem_bytes(RS, BS, cn2) > budget) return 0;
      p.RS = RS; p.BS = BS;
      p.kseg = TG2_KSEG;
    }
    unsigned char* bp = nullptr;
    pool_keep();
    // one allocation: B' blocks, then (F16) the per-combo site maxima
    const size_t bp_bytes = ((size_t)combos * p.bp_combo_stride + 255) & ~(size_t)255;
    if (cudaMallocAsync(reinterpret_cast<void**>(&bp), bp_bytes + (f16 ? combos * 4 + 16 : 0), s) != cudaSuccess) return -1;
    p.bp = bp;
    {
      const int64_t work = combos * p.tiles_n * p.nchunk * p.NT * KC;
      int blocks = (int)std::min<int64_t>((work + 255) / 256, 148 * 16);
      if (f16) {
        float* bsc = reinterpret_cast<float*>(bp + bp_bytes);
        if (cudaMemsetAsync(bsc, 0, combos * 4 + 16, s) != cudaSuccess) return -1;
        p.progress = reinterpret_cast<unsigned int*>(bsc + combos);
        const unsigned ky = (unsigned)std::min<int64_t>(d.K, std::max<int64_t>(1, 296 / combos));
        k_bscale<<<dim3((unsigned)combos, ky), d.N >= 256 ? 256 : 128, 0, s>>>(p, bsc);
        p.bscale = bsc;
        if (pair) k_bprime_pair<<<blocks < 1 ? 1 : blocks, 256, 0, s>>>(p, combos);
        else k_bprime<true><<<blocks < 1 ? 1 : blocks, 256, 0, s>>>(p, combos);
      } else {
        k_bprime<false><<<blocks < 1 ? 1 : blocks, 256, 0, s>>>(p, combos);
      }
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    p.items = p.Z * p.tiles_m * p.tiles_n;
    p.per_cta = (p.items + sms - 1) / sms;
    // A-resident tiles keep each row tile on one CTA (contiguous items);
    // otherwise items go round-robin so a row tile's column tiles run on
    // neighbouring CTAs together and share the A tile through L2
    p.ilv = (ares || p.tiles_n == 1) ? 0 : 2;
    const int64_t grid = p.ilv == 2 ? std::min<int64_t>(sms, p.items) : (p.items + p.per_cta - 1) / p.per_cta;
    const size_t smem = tg_smem_bytes(p.NT, KC, RS, BS, f16, cn);
    static uint64_t attr = 0;
    int adev = 0;
    if (attr_needed(attr, &adev)) {
      cudaFuncSetAttribute(k_tc_gemm<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      cudaFuncSetAttribute(k_tc_gemm<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      cudaFuncSetAttribute(k_tc_gemm<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      cudaFuncSetAttribute(k_tc_gemm<16, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      attr |= 1ull << (adev & 63);
    }
    if (pair) {
      // B' as rows of 1 KB: one 12-row box per half chunk
      CUtensorMap tmb;
      const cuuint64_t bdim[2] = {256u, (cuuint64_t)((combos * p.bp_combo_stride) >> 10)};
      const cuuint64_t bstr[1] = {1024u};
      const cuuint32_t bbox[2] = {256u, 12u};
      const cuuint32_t bes[2] = {1u, 1u};
      if (enc(&tmb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, bp, bdim, bstr, bbox, bes, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        cudaFreeAsync(bp, s);
        return -1;
      }
      static uint64_t attr2 = 0;
      int adev2 = 0;
      if (attr_needed(attr2, &adev2)) {
        cudaFuncSetAttribute(k_tc_gemm2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(k_tc_gemm2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr2 |= 1ull << (adev2 & 63);
      }
      const int64_t W = p.Z * ((p.tiles_m + 1) / 2) * p.tiles_n;
      const size_t smem2 = tg2_smem_bytes(p.RS, p.BS, p.cn_smem ? d.N : 0);
      // every CTA of the grid must be resident (the drift bound spins on the
      // other CTAs' progress): at most the clusters the device can hold at once
      int max_pairs = sms / 2;
      {
        cudaLaunchConfig_t lc;
        memset(&lc, 0, sizeof lc);
        lc.gridDim = dim3((unsigned)sms & ~1u);
        lc.blockDim = dim3(TG2_THREADS);
        lc.dynamicSmemBytes = smem2;
        cudaLaunchAttribute la;
        la.id = cudaLaunchAttributeClusterDimension;
        la.val.clusterDim.x = 2; la.val.clusterDim.y = 1; la.val.clusterDim.z = 1;
        lc.attrs = &la;
        lc.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, k_tc_gemm2<true>, &lc) == cudaSuccess && nc > 0) max_pairs = std::min(max_pairs, nc);
        else cudaGetLastError();
      }
      const int64_t npairs = std::min<int64_t>(max_pairs, W);
      if (p.nchunk > p.kseg) k_tc_gemm2<true><<<(unsigned)(2 * npairs), TG2_THREADS, smem2, s>>>(p, tm, tmb);
      else k_tc_gemm2<false><<<(unsigned)(2 * npairs), TG2_THREADS, smem2, s>>>(p, tm, tmb);
    } else if (p.g3) k_tc_gemm<16, true, true><<<(unsigned)grid, TG_THREADS_G3, smem, s>>>(p, tm);
    else if (f16) k_tc_gemm<16, true><<<(unsigned)grid, TG_THREADS_G3, smem, s>>>(p, tm);
    else if (KC == 16) k_tc_gemm<16, false><<<(unsigned)grid, TG_THREADS, smem, s>>>(p, tm);
    else k_tc_gemm<8, false><<<(unsigned)grid, TG_THREADS, smem, s>>>(p, tm);
    const bool ok = cudaGetLastError() == cudaSuccess;
    cudaFreeAsync(bp, s);
    return ok ? 1 : -1;
  }
}

}  // namespace tnc
