// k_tc_gemm2: the wide complex64 GEMM step (N >= 128, fp16-split 3M products,
// see tnc_tcgemm.cuh) on CTA pairs -- tcgen05.mma.cta_group::2, M = 256 per
// instruction, each CTA of the pair owning 128 rows of A / of the result in its
// own TMEM and half (64 columns) of every site block in its own shared memory.
//
// Why pairs (measured on the 53-qubit depth-12 steps, tools/exp_dbg.sh): the
// single-CTA kernel moves 92 KB through shared memory per 128 x 16-complex
// chunk (24 KB B' in, 16 KB raw A in, 16 KB raw A out to the converters, 36 KB
// read by the nine MMAs) against 576 tensor-pipe clocks, i.e. 160 B/clk of a
// 128 B/clk port; removing any one of those streams gave the same ~13%.  A
// pair halves both B' streams (12 + 18 KB), 62 KB per chunk.  The shared memory
// this frees holds a 96 KB result stage: the epilogue drains the accumulators
// to it in ~2k clocks and releases them, and writes the tile to HBM while the
// next tile's MMAs run (the single accumulator stage -- 3 x 128 columns plus
// two A stages fill TMEM -- otherwise idles the tensor pipe for the whole
// store phase, ~12k clocks per tile).
//
// Warps per CTA: 0-7 converters (raw A -> fp16 hi/lo planes in TMEM), 8-15
// epilogue, 16 MMA issuer (leader CTA only), 17 A producer (TMA tensor tiles),
// 18 B producer (TMA, completion on the leader's barrier).
// Barriers: afull / tempty live in the leader (16 arrivals: 8 warps of each
// CTA, remote arrivals from the peer); aempty / bempty / tfull are multicast
// commits to both CTAs; bfull lives in the leader and counts both halves' bytes.
#pragma once
// included by tnc_tcgemm.cuh after its kernels (GemmDesc, split/scale helpers, tma_load_3d)

namespace tnc {

constexpr int TG2_THREADS = 19 * 32;
constexpr uint32_t TG2_RAW_BYTES = 128 * 128;          // 128 rows x 16 complex
constexpr uint32_t TG2_BBLK = 64 * 16 * 2;             // one half block: 64 n x 16 k fp16
constexpr uint32_t TG2_BSTAGE = 6 * TG2_BBLK;          // [Br | Bi | Bs] hi, lo halves: 12 KB
constexpr uint32_t TG2_EBUF = 32 * 128;                // one warp round: 32 rows x 16 complex
constexpr uint32_t TG2_ESTAGE = 8 * 3 * TG2_EBUF;      // 8 warps x 3 rounds: 96 KB
constexpr int TG2_MAX_RS = 8, TG2_MAX_BS = 8;
// chunks (16 complex of K each) per K segment: 2048 complex -- the truncation error of one segment's
// accumulation chain is 3.7e-6 of the result (1.2e-4 at K = 65536 unsegmented, tools/rz_bias_probe.py)
constexpr int TG2_KSEG = 128;

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `local` (a shared::cta address) in CTA `rank`
__device__ __forceinline__ uint32_t mapa_u32(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// wait on a barrier whose arrivals also come from the peer CTA (default .acquire.cta as CUTLASS's 2-SM
// pipelines: a cluster-scope acquire in the poll loop costs ~500 clk per try_wait)
__device__ __forceinline__ void mbar_wait_spin_cluster(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
__device__ __forceinline__ void mma_f16_ts_pair(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// B' half-chunk (12 rows of 1 KB) -> own shared memory, bytes counted on the
// leader's barrier (`mbar_cluster`: shared::cluster address)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int x, int y, uint32_t mbar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(mbar_cluster)
      : "memory");
}

// Pair layout of the site operand: per (combo, N tile, chunk) two halves (CTA
// rank), each [Br | Bi | Br + Bi] hi then lo, blocks of 64 n x 16 k, K-major
// canonical (8 x 16 B core matrices, LBO 128 B, SBO 256 B)
__global__ void k_bprime_pair(const __grid_constant__ GemmDesc p, int64_t combos) {
  constexpr int NT = 128, KC = 16;
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
    const int half = nl >> 6, nh = nl & 63;
    unsigned char* base = const_cast<unsigned char*>(p.bp) + combo * p.bp_combo_stride +
                          (((tn * p.nchunk + c) * 2 + half) * 6) * (int64_t)TG2_BBLK;
    const uint32_t boff = (nh & 7) * 16 + (nh >> 3) * 256 + (kl >> 3) * 128 + (kl & 7) * 2;
    const float t = op_scale(p.bscale[combo], 1);
    uint16_t rh, rl, ih, il, sh, sl;
    split_f16(sv.x * t, rh, rl);
    split_f16(sv.y * t, ih, il);
    split_f16((sv.x + sv.y) * t, sh, sl);
    const uint16_t v[6] = {rh, ih, sh, rl, il, sl};
#pragma unroll
    for (int b = 0; b < 6; ++b) *reinterpret_cast<uint16_t*>(base + b * TG2_BBLK + boff) = v[b];
  }
}

// staged round buffer: 32 rows x 128 B, 16-byte pieces XOR-swizzled by the row
__device__ __forceinline__ uint32_t tg2_piece(uint32_t buf_s, int row, int piece) {
  return buf_s + (uint32_t)row * 128u + (uint32_t)((piece ^ (row & 7)) << 4);
}

// result stores: streaming (evict-first) so that the result does not push the
// A rows that other column tiles are about to re-read out of L2
// `acc`: a later K segment of the tile -- the partial product is added to the
// stored one in fp32 round-to-nearest (the same thread stored it);
// `vmax`: max |re|, |im| of the final values (tracked on the last segment)
template <bool SEG>
__device__ __forceinline__ void tg2_st4(float4* dst, float4 v, bool acc, float& vmax) {
  if (SEG && acc) {
    const float4 o = *dst;
    v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
    vmax = fmaxf(vmax, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
  __stcs(dst, v);
}
template <bool SEG>
__device__ __forceinline__ void tg2_st2(float2* dst, float2 v, bool acc, float& vmax) {
  if (SEG && acc) {
    const float2 o = *dst;
    v.x += o.x; v.y += o.y;
    vmax = fmaxf(vmax, fmaxf(fabsf(v.x), fabsf(v.y)));
  }
  __stcs(dst, v);
}

// the warp's 32 rows x 16 columns [n0c0, n0c0 + ncols) of the result, from a
// staged round buffer to global memory (layouts as k_tc_gemm's epilogue)
template <bool SEG>
__device__ __forceinline__ void tg2_flush(const GemmDesc& p, uint32_t buf_s, int lane, int q, int64_t mt, int64_t row,
                                          int64_t oc, float2* O, int64_t n0c0, int ncols, const int32_t* cn_s,
                                          bool staged, bool acc, float& vmax) {
  if (staged) {
    if (p.blk_contig && ncols == 16 && mt * 128 + q * 32 + 32 <= p.M) {
      const int64_t oc0 = __shfl_sync(0xffffffffu, oc, 0);
      float4* dst = reinterpret_cast<float4*>(O + oc0 + (p.c_rows_contig ? n0c0 : (int64_t)cn_s[n0c0]));
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int c = i * 32 + lane;
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "r"(tg2_piece(buf_s, c >> 3, c & 7)) : "memory");
        tg2_st4<SEG>(dst + c, v, acc, vmax);
      }
      return;
    }
    const int sub = lane & 7;                // 16-byte piece (2 complex) of a row
    const int64_t n = n0c0 + 2 * sub;
    int64_t a0 = 0, a1 = 0;
    if (2 * sub < ncols) a0 = p.c_rows_contig ? n : (p.cn_smem ? cn_s[n] : p.c_noff[n]);
    if (2 * sub + 1 < ncols) a1 = p.c_rows_contig ? n + 1 : (p.cn_smem ? cn_s[n + 1] : p.c_noff[n + 1]);
    const int64_t oc0 = p.row_stride ? __shfl_sync(0xffffffffu, oc, 0) : 0;
#pragma unroll
    for (int rr = 0; rr < 32; rr += 4) {
      const int lr = rr + (lane >> 3);
      const int64_t grow = mt * 128 + q * 32 + lr;
      const int64_t ocr = p.row_stride ? oc0 + (int64_t)lr * p.row_stride : __shfl_sync(0xffffffffu, oc, lr);
      if (grow < p.M && 2 * sub < ncols) {
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "r"(tg2_piece(buf_s, lr, sub)) : "memory");
        float2* dst = O + ocr + a0;
        if (2 * sub + 1 < ncols && a1 == a0 + 1 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
          tg2_st4<SEG>(reinterpret_cast<float4*>(dst), v, acc, vmax);
        } else {
          tg2_st2<SEG>(dst, make_float2(v.x, v.y), acc, vmax);
          if (2 * sub + 1 < ncols) tg2_st2<SEG>(O + ocr + a1, make_float2(v.z, v.w), acc, vmax);
        }
      }
    }
    return;
  }
  // innermost result leg is a free leg: lane = row, consecutive rows contiguous
  if (row < p.M) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float4 v;
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                   : "r"(tg2_piece(buf_s, lane, u)) : "memory");
      if (2 * u < ncols) {
        const int64_t n = n0c0 + 2 * u;
        tg2_st2<SEG>(O + oc + (p.cn_smem ? (int64_t)cn_s[n] : p.c_noff[n]), make_float2(v.x, v.y), acc, vmax);
      }
      if (2 * u + 1 < ncols) {
        const int64_t n = n0c0 + 2 * u + 1;
        tg2_st2<SEG>(O + oc + (p.cn_smem ? (int64_t)cn_s[n] : p.c_noff[n]), make_float2(v.z, v.w), acc, vmax);
      }
    }
  }
}

// SEG: K longer than one segment (the accumulate paths of the epilogue are
// compiled only then: they cost registers in the drain, 3.7% on the K <= 2048 steps)
template <bool SEG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TG2_THREADS, 1)
k_tc_gemm2(const __grid_constant__ GemmDesc p, const __grid_constant__ CUtensorMap tmA,
           const __grid_constant__ CUtensorMap tmB) {
  extern __shared__ __align__(128) unsigned char smem_dyn[];
  constexpr int KC = 16, NT = 128, RB = 128;
  constexpr uint32_t ACOLS = 48, A0 = 384;             // accumulators T1 | T2 | T3, then two A stages
  constexpr int CONVW = 8, EPIW = 8, EPI_WARP0 = 8, MMA_WARP = 16, APROD_WARP = 17, BPROD_WARP = 18, AS = 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int nchunk = p.nchunk;
  const int RS = p.RS, BS = p.BS;
  unsigned char* araw = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  unsigned char* bring = araw + (size_t)RS * TG2_RAW_BYTES;
  unsigned char* estage = bring + (size_t)BS * TG2_BSTAGE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(estage + TG2_ESTAGE);
  uint64_t* rfull = bar;                           // [RS] TMA -> converters (own CTA)
  uint64_t* rempty = rfull + TG2_MAX_RS;           // [RS] converters -> A producer (own CTA)
  uint64_t* afull = rempty + TG2_MAX_RS;           // [AS] both CTAs' converters -> MMA (leader's copy)
  uint64_t* aempty = afull + AS;                   // [AS] MMA -> converters (multicast)
  uint64_t* bfull = aempty + AS;                   // [BS] both halves' bytes (leader's copy)
  uint64_t* bempty = bfull + TG2_MAX_BS;           // [BS] MMA -> B producers (multicast)
  uint64_t* tfull = bempty + TG2_MAX_BS;           // [1] MMA -> epilogues (multicast)
  uint64_t* tempty = tfull + 1;                    // [1] both CTAs' epilogues -> MMA (leader's copy)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  int32_t* cn_s = reinterpret_cast<int32_t*>(tmem_slot + 4);
  if (p.cn_smem)
    for (int n = threadIdx.x; n < p.N; n += blockDim.x) cn_s[n] = (int32_t)p.c_noff[n];

  // pair items: (z, row-tile pair, column tile), dealt round-robin over the
  // pairs so that the column tiles of a row-tile pair run on neighbouring
  // pairs at the same time and share the A rows through L2
  const int64_t pairs_m = (p.tiles_m + 1) / 2;
  const int64_t per_z = pairs_m * p.tiles_n;
  const int64_t W = p.Z * per_z;
  const int64_t npairs = gridDim.x >> 1, pair = blockIdx.x >> 1;
  const int nitems = (int)((W - pair + npairs - 1) / npairs);
  auto item = [&](int it, int64_t& z, int64_t& mt, int64_t& nt) {
    const int64_t w = (int64_t)it * npairs + pair;
    z = w / per_z;
    const int64_t rem = w - z * per_z;
    const int64_t mp = rem / p.tiles_n;
    nt = rem - mp * p.tiles_n;
    mt = 2 * mp + rank;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < RS; ++s) { mbar_init(&rfull[s], 1); mbar_init(&rempty[s], CONVW); }
    for (int s = 0; s < AS; ++s) { mbar_init(&afull[s], 2 * CONVW); mbar_init(&aempty[s], 1); }
    for (int s = 0; s < BS; ++s) { mbar_init(&bfull[s], 1); mbar_init(&bempty[s], 1); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * EPIW);
    mbar_fence_init();
  }
  if (warp == EPI_WARP0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();                              // the peer's barriers exist before anything targets them
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < CONVW) {
    // ---------------- converters: raw A -> Ar, Ai, Ar + Ai hi/lo fp16 planes in TMEM ----------------
    const int h = warp >> 2;                       // complex [8h, 8h + 8) of the chunk
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t afull_c = mapa_u32(smem_u32(afull), 0);
    int rstage = 0, astage = 0;
    uint32_t rph = 0, aph = 0;
    float sA = 1.f;
    int64_t sz = -1;
    for (int it = 0; it < nitems; ++it) {
      int64_t z, mt, nt;
      item(it, z, mt, nt);
      if (z != sz) { sz = z; sA = op_scale(__ldg(p.amax_in + z), 1); }
      for (int c = 0; c < nchunk; ++c) {
        mbar_wait_spin(&rfull[rstage], rph);
        const uint32_t src = smem_u32(araw + (size_t)rstage * TG2_RAW_BYTES);
        uint32_t rh[4], ih[4], sh[4], rl[4], il[4], sl[4];
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const uint32_t off = (uint32_t)(r * RB + 16 * (4 * h + qq));
          const uint32_t phys = off ^ (((off >> 7) & 7u) << 4);
          float4 x;
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "r"(src + phys));
          // scaled values and their sums; hi = packed fp16 conversion, lo = packed fp16 of (y - hi)
          const float r0 = x.x * sA, i0 = x.y * sA, r1 = x.z * sA, i1 = x.w * sA;
          split_f16x2_cvt(r0, r1, rh[qq], rl[qq]);
          split_f16x2_cvt(i0, i1, ih[qq], il[qq]);
          split_f16x2_cvt(r0 + i0, r1 + i1, sh[qq], sl[qq]);
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
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(afull_c + 8u * (uint32_t)astage);
        // the raw stage is released only after its shared loads have been
        // consumed; the proxy fence orders them before the TMA refill
        fence_proxy_async();
        mbar_arrive_warp(&rempty[rstage]);
        if (++rstage == RS) { rstage = 0; rph ^= 1; }
        if (++astage == AS) { astage = 0; aph ^= 1; }
      }
    }
  } else if (warp < MMA_WARP) {
    // ---------------- epilogue: TMEM -> staged tile (accumulators released) -> result ----------------
    const int q = warp & 3;                      // TMEM lane quadrant
    const int eg = (warp - EPI_WARP0) >> 2;      // column half
    const int r = q * 32 + lane;
    const uint32_t ebuf = smem_u32(estage) + (uint32_t)(warp - EPI_WARP0) * 3u * TG2_EBUF;
    const uint32_t tempty_c = mapa_u32(smem_u32(tempty), 0);
    const bool staged = (p.c_rows_contig || p.n_contig || (p.N > 1 && p.c_noff[1] == p.c_noff[0] + 1));
    float inv = 1.f, inv2 = 1.f;
    int64_t inv_z = -1;
    uint32_t tph = 0;
    const int kseg = SEG ? p.kseg : nchunk;      // chunks accumulated in TMEM before the sum leaves the tensor core
    for (int it = 0; it < nitems; ++it) {
      int64_t z, mt, nt;
      item(it, z, mt, nt);
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
      const int64_t n0 = nt * NT + eg * 64;        // first column of this warp
      if (z != inv_z) {
        inv_z = z;
        inv = 1.f / op_scale(__ldg(p.amax_in + z), 1);
        inv2 = 1.f / op_scale(__ldg(p.bscale + gemm_combo(p, z)), 1);
      }
      // K segments of at most kseg chunks: each is drained, scaled (with the
      // truncation compensation of its own accumulation count) and added to
      // the stored partial result in fp32 round-to-nearest, so the
      // round-toward-zero chain inside the tensor core stays short
      for (int c0 = 0; c0 < nchunk; c0 += kseg, tph ^= 1) {
      const int c1 = min(nchunk, c0 + kseg);
      const bool acc = SEG && c0 > 0, last = !SEG || c1 == nchunk;
      const float sc = inv * (1.f + TG_RZ_LOSS * (float)(3 * (c1 - c0)));
      float vmax = 0.f;
      mbar_wait_idle(tfull, tph);
      tc_fence_after();
      const uint32_t tre = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(eg * 64);
      uint32_t vr[16], vi[16];
#pragma unroll
      for (int rd = 0; rd < 4; ++rd) {
        uint32_t v3[16];
        tmem_ld16(tre + rd * 16, vr);
        tmem_ld16(tre + NT + rd * 16, vi);
        tmem_ld16(tre + 2 * NT + rd * 16, v3);
        tmem_wait_ld();
        if (rd == 3) {                             // everything read: release the accumulators
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty_c);
        }
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {          // re = T1 - T2, im = T3 - T1 - T2
          const float t1 = __uint_as_float(vr[jj]), t2 = __uint_as_float(vi[jj]);
          const float a = (t1 - t2) * sc * inv2, b = (__uint_as_float(v3[jj]) - t1 - t2) * sc * inv2;
          if (!SEG || !acc) vmax = fmaxf(vmax, fmaxf(fabsf(a), fabsf(b)));
          vr[jj] = __float_as_uint(a);
          vi[jj] = __float_as_uint(b);
        }
        if (rd < 3) {
#pragma unroll
          for (int jj = 0; jj < 16; jj += 2)
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(tg2_piece(ebuf + rd * TG2_EBUF, lane, jj >> 1)),
                         "f"(__uint_as_float(vr[jj])), "f"(__uint_as_float(vi[jj])),
                         "f"(__uint_as_float(vr[jj + 1])), "f"(__uint_as_float(vi[jj + 1])) : "memory");
        }
      }
      __syncwarp();
      auto ncols_of = [&](int rd) { const int64_t nl = p.N - (n0 + rd * 16); return nl < 16 ? (nl < 0 ? 0 : (int)nl) : 16; };
      tg2_flush<SEG>(p, ebuf, lane, q, mt, row, oc, O, n0, ncols_of(0), cn_s, staged, acc, vmax);
      __syncwarp();
      // round 3 (still in registers) takes round 0's buffer
#pragma unroll
      for (int jj = 0; jj < 16; jj += 2)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(tg2_piece(ebuf, lane, jj >> 1)),
                     "f"(__uint_as_float(vr[jj])), "f"(__uint_as_float(vi[jj])),
                     "f"(__uint_as_float(vr[jj + 1])), "f"(__uint_as_float(vi[jj + 1])) : "memory");
      __syncwarp();
      tg2_flush<SEG>(p, ebuf + TG2_EBUF, lane, q, mt, row, oc, O, n0 + 16, ncols_of(1), cn_s, staged, acc, vmax);
      tg2_flush<SEG>(p, ebuf + 2 * TG2_EBUF, lane, q, mt, row, oc, O, n0 + 32, ncols_of(2), cn_s, staged, acc, vmax);
      tg2_flush<SEG>(p, ebuf, lane, q, mt, row, oc, O, n0 + 48, ncols_of(3), cn_s, staged, acc, vmax);
      __syncwarp();
      if (p.amax_out && last) {                  // rows past M / padded columns hold zeros
        for (int o = 16; o; o >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        if (lane == 0 && vmax > 0.f) atomicMax(reinterpret_cast<unsigned int*>(p.amax_out) + z, __float_as_uint(vmax));
      }
      }
    }
  } else if (warp == MMA_WARP) {
    // ---------------- MMA issuer (leader CTA): M = 256 over both CTAs' TMEM ----------------
    if (rank == 0) {
      if (tmem != 0u) __trap();                    // all 512 columns: base 0 keeps the operands warp-uniform
      const uint32_t idesc = (1u << 4) | ((uint32_t)(NT >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
      int bs = 0, stage = 0;
      uint32_t bph = 0, aph = 0, tph = 0;
      const uint64_t dB = umma_desc(smem_u32(bring), 128, 256);
      constexpr uint32_t bstage16 = TG2_BSTAGE >> 4, bblk16 = TG2_BBLK >> 4;
      const int kseg = SEG ? p.kseg : nchunk;
      int cseg = 0;                                // chunks issued into the current K segment
      for (int it = 0; it < nitems; ++it) {
        for (int c = 0; c < nchunk; ++c) {
          if (cseg == 0) {                         // segment start: the epilogue has drained the accumulators
            mbar_wait_spin_cluster(tempty, tph ^ 1);
            tc_fence_after();
          }
          mbar_wait_spin_cluster(&afull[stage], aph);
          mbar_wait_spin_cluster(&bfull[bs], bph);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t bb = dB + (uint64_t)(bs * bstage16);
            const uint32_t arh = A0 + (uint32_t)stage * ACOLS;
            const uint32_t aih = arh + 8, ash = arh + 16, arl = arh + 24, ail = arh + 32, asl = arh + 40;
            const uint64_t brh = bb, bih = bb + bblk16, bsh = bb + 2 * bblk16;
            const uint64_t brl = bb + 3 * bblk16, bil = bb + 4 * bblk16, bsl = bb + 5 * bblk16;
            const uint32_t first = cseg == 0 ? 0u : 1u;
            const uint32_t d1 = 0u, d2 = (uint32_t)NT, d3 = 2u * (uint32_t)NT;
            // small terms first (lo*hi, hi*lo), then hi*hi
            mma_f16_ts_pair(d1, arl, brh, idesc, first);
            mma_f16_ts_pair(d2, ail, bih, idesc, first);
            mma_f16_ts_pair(d3, asl, bsh, idesc, first);
            mma_f16_ts_pair(d1, arh, brl, idesc, 1u);
            mma_f16_ts_pair(d2, aih, bil, idesc, 1u);
            mma_f16_ts_pair(d3, ash, bsl, idesc, 1u);
            mma_f16_ts_pair(d1, arh, brh, idesc, 1u);
            mma_f16_ts_pair(d2, aih, bih, idesc, 1u);
            mma_f16_ts_pair(d3, ash, bsh, idesc, 1u);
            umma_commit_pair(&aempty[stage]);
            umma_commit_pair(&bempty[bs]);
            if (cseg + 1 == kseg || c == nchunk - 1) umma_commit_pair(tfull);
          }
          __syncwarp();
          if (++cseg == kseg || c == nchunk - 1) { cseg = 0; tph ^= 1; }
          if (++bs == BS) { bs = 0; bph ^= 1; }
          if (++stage == AS) { stage = 0; aph ^= 1; }
        }
      }
    }
  } else if (warp == APROD_WARP && lane == 0) {
    // ---------------- A producer: this CTA's 128 rows of every chunk ----------------
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    int rs = 0;
    uint32_t rph = 0;
    for (int it = 0; it < nitems; ++it) {
      int64_t z, mt, nt;
      item(it, z, mt, nt);
      // bounded drift: the column tiles of a row-tile pair run on neighbouring
      // pairs and share its A rows through L2 only while those pairs stay
      // together (unbounded, the slower pairs fall items behind and re-read
      // their rows from HBM: 46 GB of DRAM reads for 8.6 GB of A at N = 2048).
      // A CTA starts item `it` once every CTA has issued the loads of item it - 1.
      if (it >= 1) {
        const unsigned int target = (unsigned int)it * gridDim.x;
        unsigned int seen;
        do {
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(p.progress) : "memory");
        } while (seen < target);
      }
      for (int c = 0; c < nchunk; ++c) {
        mbar_wait_spin(&rempty[rs], rph ^ 1);
        mbar_expect_tx(&rfull[rs], TG2_RAW_BYTES);
        tma_load_3d(araw + (size_t)rs * TG2_RAW_BYTES, &tmA, c * 2 * KC, (int)(mt * 128), (int)z, &rfull[rs]);
        if (++rs == RS) { rs = 0; rph ^= 1; }
      }
      atomicAdd(p.progress, 1u);
    }
  } else if (warp == BPROD_WARP && lane == 0) {
    // ---------------- B producer: this CTA's half of every site chunk ----------------
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    const uint32_t bfull_c = mapa_u32(smem_u32(bfull), 0);
    int bs = 0;
    uint32_t bph = 0;
    for (int it = 0; it < nitems; ++it) {
      int64_t z, mt, nt;
      item(it, z, mt, nt);
      // B' rows of 1 KB: 12 per half chunk
      const int64_t row0 = (gemm_combo(p, z) * p.bp_combo_stride >> 10) + (nt * nchunk * 2 + rank) * 12;
      for (int c = 0; c < nchunk; ++c) {
        mbar_wait_spin(&bempty[bs], bph ^ 1);
        if (rank == 0) mbar_expect_tx(&bfull[bs], 2 * TG2_BSTAGE);
        tma_load_2d_pair(bring + (size_t)bs * TG2_BSTAGE, &tmB, 0, (int)(row0 + (int64_t)c * 24), bfull_c + 8u * (uint32_t)bs);
        if (++bs == BS) { bs = 0; bph ^= 1; }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();                              // both CTAs done before either frees TMEM or exits
  if (warp == EPI_WARP0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

__host__ inline size_t tg2_smem_bytes(int RS, int BS, int64_t cn) {
  return 1024 + (size_t)RS * TG2_RAW_BYTES + (size_t)BS * TG2_BSTAGE + TG2_ESTAGE +
         8 * (2 * TG2_MAX_RS + 4 + 2 * TG2_MAX_BS + 2) + 16 + 4 * cn;
}

// The pair kernel takes the 3M steps with K >= 512 and at least half a wave of
// pair items; with fewer chunks per tile the single-CTA kernel is faster
// (measured on the K = 256, N = 512 steps: 3.5 vs 4.3 ms).
inline bool tg2_applicable(const GemmDesc& p) {
  return p.g3 && p.NT == 128 && p.KC == 16 && p.nchunk >= 32 && p.Z * ((p.tiles_m + 1) / 2) * p.tiles_n >= 37;
}

}  // namespace tnc
