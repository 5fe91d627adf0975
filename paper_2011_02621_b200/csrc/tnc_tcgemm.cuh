// Tensor-core GEMM path for large engine steps (complex64): C[z] = A[z] S(z)
// with A row-contiguous [M][K] (the engine's due-ordered accumulator), K a
// multiple of 16 (or 4 / 8), any N (tiled by NT <= 64 complex) and a general
// result map out = rowC(f) + c_noff[n] (the due-ordered result layout).
//
// Differences from k_tc_c64 (the skinny / sweep kernel): the site operand is
// not resident -- B' (complex->real embedding, tf32 hi/lo, canonical K-major
// chunks) is prepared once per distinct site block ("combo" = projected
// variant x slice digits of this node's cut legs) by k_bprime and streamed per
// K chunk by a cp.async.bulk producer; work items are (z, 128-row tile, N tile)
// with the N tiles of a row tile consecutive, so the A tile is re-read from L2.
//
// Warps: 0-7 converters (2 groups alternate work items; global -> tf32 hi/lo ->
// TMEM), 8-11 epilogue, 12 MMA issuer, 13 B' producer.
#pragma once
#include "tnc_tc.cuh"

namespace tnc {

struct GemmDesc {
  int64_t Z, M, K, N;
  int64_t tiles_m, per_cta, items;
  int32_t NT, tiles_n;           // complex columns per N tile
  int32_t KC, nchunk;            // complex K per chunk
  const float2* a;
  int64_t a_zstride;
  const float* bp;               // [combo][tile_n][chunk][hi|lo][2NT x 2KC] canonical
  int64_t bp_combo_stride;       // floats per combo
  tnc_site site;                 // site blocks: combo -> offset
  const int64_t* b_koff;         // [K] site offsets
  const int64_t* b_noff;         // [N]
  int32_t conj_b, _pad;
  int64_t slices_per_b, s0;
  float2* out;
  int64_t out_zstride;
  int32_t nf, c_rows_contig;
  int64_t f_dim[TNC_MAX_LEGS], f_cstride[TNC_MAX_LEGS];
  const int64_t* c_noff;         // [N]
};

constexpr int TG_THREADS = 14 * 32;
constexpr int TG_MMA_WARP = 12, TG_PROD_WARP = 13;
constexpr int TG_BSTAGES = 4;

__device__ __forceinline__ int64_t gemm_combo(const GemmDesc& p, int64_t z) {
  const int64_t b = z / p.slices_per_b;
  const int64_t sl = p.s0 + (z - b * p.slices_per_b);
  int64_t c = p.site.sel ? (int64_t)p.site.sel[b] : 0;
  for (int j = 0; j < p.site.ncut; ++j) c = c * p.site.cut_ext[j] + (sl / p.site.cut_div[j]) % p.site.cut_ext[j];
  return c;
}

__host__ __device__ inline int64_t tg_chunk_floats(int NT, int KC) { return (int64_t)(2 * NT) * (2 * KC); }

// B' for every (combo, N tile, K chunk): rows n' = 2n + c' of the tile, cols
// k' = 2k + c of the chunk, K-major canonical (8 x 16 B core matrices, LBO =
// 128 B along K, SBO = (2KC/4) * 128 B along N), hi chunk then lo chunk.
__global__ void k_bprime(const __grid_constant__ GemmDesc p, int64_t combos) {
  const int NT = p.NT, KC = p.KC, KCr = 2 * KC;
  const int64_t cf = tg_chunk_floats(NT, KC);
  const uint32_t SBO = (KCr / 4) * 128;
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
    float* base = const_cast<float*>(p.bp) + combo * p.bp_combo_stride + ((tn * p.nchunk + c) * 2) * cf;
    const float vals[4] = {sv.x, -sv.y, sv.y, sv.x};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int nr = 2 * nl + (q >> 1), kr = 2 * kl + (q & 1);
      const uint32_t boff = (nr & 7) * 16 + (nr >> 3) * SBO + (kr >> 2) * 128 + (kr & 3) * 4;
      float h, l;
      split3(vals[q], h, l);
      *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(base) + boff) = h;
      *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(base + cf) + boff) = l;
    }
  }
}

template <int KC>
__global__ void __launch_bounds__(TG_THREADS, 1)
k_tc_gemm(const __grid_constant__ GemmDesc p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NT = p.NT, Nr = 2 * NT;
  const int nchunk = p.nchunk;
  const int64_t cf = tg_chunk_floats(NT, KC);
  const uint32_t cbytes = (uint32_t)(cf * 4);
  const uint32_t SBO_B = ((2 * KC) / 4) * 128;
  // TMEM: 2 accumulators of Nr columns, A stages of 4*KC columns (hi + lo)
  const int TS = 2;
  constexpr uint32_t ACOLS = 4 * KC;
  const int AS = min(TC_MAX_STAGES, (512 - TS * Nr) / (int)ACOLS) & ~1;   // even: 2 converter groups
  const int ASg = AS / 2;
  const uint32_t A0 = (uint32_t)(TS * Nr);
  // smem: B ring [TG_BSTAGES][hi|lo chunk], c_noff tile, barriers
  unsigned char* bring = smem_raw;
  int64_t* cno = reinterpret_cast<int64_t*>(bring + (size_t)TG_BSTAGES * 2 * cbytes);   // [NT]
  uint64_t* bar = reinterpret_cast<uint64_t*>(cno + 64);
  uint64_t* afull = bar;                         // [AS]
  uint64_t* aempty = bar + TC_MAX_STAGES;        // [AS]
  uint64_t* bfull = bar + 2 * TC_MAX_STAGES;     // [TG_BSTAGES]
  uint64_t* bempty = bfull + TG_BSTAGES;         // [TG_BSTAGES]
  uint64_t* tfull = bempty + TG_BSTAGES;         // [TS]
  uint64_t* tempty = tfull + 2;                  // [TS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int64_t w0 = blockIdx.x * p.per_cta;
  const int64_t w1 = min(w0 + p.per_cta, p.items);
  const int nitems = (int)(w1 - w0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < AS; ++s) { mbar_init(&afull[s], 4); mbar_init(&aempty[s], 1); }
    for (int s = 0; s < TG_BSTAGES; ++s) { mbar_init(&bfull[s], 1); mbar_init(&bempty[s], 1); }
    for (int s = 0; s < TS; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 4); }
    mbar_fence_init();
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t per_z = p.tiles_m * p.tiles_n;

  if (warp < 8) {
    // ---------------- converters ----------------
    const int grp = warp >> 2;
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    int j = 0;
    for (int it = grp; it < nitems; it += 2) {
      const int64_t w = w0 + it;
      const int64_t z = w / per_z;
      const int64_t rem = w - z * per_z;
      const int64_t mt = rem / p.tiles_n;
      const int64_t row = mt * 128 + r;
      const bool valid = row < p.M;
      const float2* Ar = p.a + z * p.a_zstride + (valid ? row : 0) * p.K;
      float2 v[KC];
      auto ld = [&](int c) {
#pragma unroll
        for (int q = 0; q < KC; q += 2) {
          if (valid) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(Ar + c * KC + q));
            v[q] = make_float2(x.x, x.y);
            v[q + 1] = make_float2(x.z, x.w);
          } else {
            v[q] = v[q + 1] = make_float2(0.f, 0.f);
          }
        }
      };
      ld(0);
      for (int c = 0; c < nchunk; ++c, ++j) {
        const int stage = grp * ASg + j % ASg;
        const uint32_t ph = (j / ASg) & 1;
        uint32_t hi[2 * KC], lo[2 * KC];
#pragma unroll
        for (int q = 0; q < KC; ++q) {
          float a, b;
          split3(v[q].x, a, b);
          hi[2 * q] = __float_as_uint(a);
          lo[2 * q] = __float_as_uint(b);
          split3(v[q].y, a, b);
          hi[2 * q + 1] = __float_as_uint(a);
          lo[2 * q + 1] = __float_as_uint(b);
        }
        if (c + 1 < nchunk) ld(c + 1);             // next chunk's loads in flight during the handoff
        mbar_wait(&aempty[stage], ph ^ 1);
        tc_fence_after();
        const uint32_t col = A0 + (uint32_t)stage * ACOLS;
        tmem_st<2 * KC>(tmem + lane_base + col, hi);
        tmem_st<2 * KC>(tmem + lane_base + col + 2 * KC, lo);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive_warp(&afull[stage]);
      }
    }
  } else if (warp < 12) {
    // ---------------- epilogue: TMEM -> registers -> result map ----------------
    const int q = warp & 3;
    const int r = q * 32 + lane;
    for (int it = 0; it < nitems; ++it) {
      const int acc = it % TS;
      const uint32_t ph = (it / TS) & 1;
      const int64_t w = w0 + it;
      const int64_t z = w / per_z;
      const int64_t rem = w - z * per_z;
      const int64_t mt = rem / p.tiles_n, nt = rem - mt * p.tiles_n;
      const int64_t row = mt * 128 + r;
      // row map (mixed radix over the free legs) while the MMAs run
      int64_t oc = row * p.N;
      if (!p.c_rows_contig && row < p.M) {
        int64_t f = row;
        oc = 0;
        for (int jj = p.nf - 1; jj >= 0; --jj) {
          const int64_t qq = f / p.f_dim[jj];
          oc += (f - qq * p.f_dim[jj]) * p.f_cstride[jj];
          f = qq;
        }
      }
      float2* O = p.out + z * p.out_zstride;
      const int64_t n0 = nt * NT;
      mbar_wait(&tfull[acc], ph);
      tc_fence_after();
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * Nr);
      for (int c0 = 0; c0 < Nr; c0 += 32) {
        uint32_t vv[32];
        if (c0 + 32 <= Nr) {
          tmem_ld32(taddr + c0, vv);
        } else {
          uint32_t w16[16];
          tmem_ld16(taddr + c0, w16);
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) vv[jj] = w16[jj];
        }
        tmem_wait_ld();
        if (c0 + 32 >= Nr) {
          tc_fence_before();
          mbar_arrive_warp(&tempty[acc]);
        }
        if (row < p.M) {
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const int64_t n = n0 + c0 / 2 + jj;
            if (2 * jj < min(32, Nr - c0) && n < p.N) {
              const float2 val = make_float2(__uint_as_float(vv[2 * jj]), __uint_as_float(vv[2 * jj + 1]));
              O[p.c_rows_contig ? oc + n : oc + p.c_noff[n]] = val;
            }
          }
        }
      }
    }
  } else if (warp == TG_MMA_WARP) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = tf32_idesc(Nr);
    int bi = 0;
    for (int it = 0; it < nitems; ++it) {
      const int acc = it % TS;
      mbar_wait(&tempty[acc], ((it / TS) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + (uint32_t)(acc * Nr);
      const int g = it & 1;
      for (int c = 0; c < nchunk; ++c, ++bi) {
        const int jj = (it >> 1) * nchunk + c;
        const int stage = g * ASg + jj % ASg;
        mbar_wait(&afull[stage], (jj / ASg) & 1);
        const int bs = bi % TG_BSTAGES;
        mbar_wait(&bfull[bs], (bi / TG_BSTAGES) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t ahi = tmem + A0 + (uint32_t)stage * ACOLS, alo = ahi + 2 * KC;
          const uint32_t bh = smem_u32(bring + (size_t)bs * 2 * cbytes);
          const uint64_t dbh0 = umma_desc(bh, 128, SBO_B), dbl0 = umma_desc(bh + cbytes, 128, SBO_B);
#pragma unroll
          for (int s = 0; s < KC / 4; ++s) {
            const uint64_t step = (uint64_t)(s * 256) >> 4;
            const uint32_t first = (c == 0 && s == 0) ? 0u : 1u;
            mma_tf32_ts(d, alo + 8 * s, dbh0 + step, idesc, first);
            mma_tf32_ts(d, ahi + 8 * s, dbl0 + step, idesc, 1u);
            mma_tf32_ts(d, ahi + 8 * s, dbh0 + step, idesc, 1u);
          }
          umma_commit(&aempty[stage]);
          umma_commit(&bempty[bs]);
          if (c == nchunk - 1) umma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else if (warp == TG_PROD_WARP && lane == 0) {
    // ---------------- B' producer ----------------
    int bi = 0;
    for (int it = 0; it < nitems; ++it) {
      const int64_t w = w0 + it;
      const int64_t z = w / per_z;
      const int64_t nt = (w - z * per_z) % p.tiles_n;
      const float* src = p.bp + gemm_combo(p, z) * p.bp_combo_stride + nt * nchunk * 2 * cf;
      for (int c = 0; c < nchunk; ++c, ++bi) {
        const int bs = bi % TG_BSTAGES;
        mbar_wait(&bempty[bs], ((bi / TG_BSTAGES) & 1) ^ 1);
        unsigned char* dst = bring + (size_t)bs * 2 * cbytes;
        mbar_expect_tx(&bfull[bs], 2 * cbytes);
        bulk_g2s(dst, src + c * 2 * cf, 2 * cbytes, &bfull[bs]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

__host__ inline size_t tg_smem_bytes(int NT, int KC) {
  return (size_t)TG_BSTAGES * 2 * tg_chunk_floats(NT, KC) * 4 + 64 * 8 + 8 * TC_MAX_STAGES * 8 + 256;
}

// engine step on the GEMM path; returns 1 launched, 0 not applicable, -1 error
template <typename R>
int try_tc_gemm(const tnc_step_desc& d, cudaStream_t s) {
  if constexpr (sizeof(R) != 4) {
    return 0;
  } else {
    if (!d.a_rows_contig || d.K * d.N < 256) return 0;
    int KC;
    if (d.K % 16 == 0) KC = 16;
    else if (d.K == 8) KC = 8;
    else if (d.K == 4) KC = 4;
    else return 0;
    int64_t combos = 1;
    if (d.site.sel) {
      if (d.site.nvariants <= 0) return 0;
      combos = d.site.nvariants;
    }
    for (int j = 0; j < d.site.ncut; ++j) combos *= d.site.cut_ext[j];
    if (d.site.zstride != 0 || combos > 4096 || d.nf > TNC_MAX_LEGS) return 0;
    GemmDesc p;
    memset(&p, 0, sizeof p);
    p.Z = d.Z; p.M = d.M; p.K = d.K; p.N = d.N;
    p.NT = d.N >= 64 ? 64 : (int)((d.N + 7) / 8 * 8);
    p.tiles_n = (int)((d.N + p.NT - 1) / p.NT);
    p.KC = KC;
    p.nchunk = (int)(d.K / KC);
    p.tiles_m = (d.M + 127) / 128;
    p.a = reinterpret_cast<const float2*>(d.acc);
    p.a_zstride = d.acc_zstride;
    if ((((uintptr_t)p.a) % 16) || (d.K % 2) || (d.acc_zstride % 2)) return 0;   // float4 row loads
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
    const int64_t cf = tg_chunk_floats(p.NT, KC);
    p.bp_combo_stride = (int64_t)p.tiles_n * p.nchunk * 2 * cf;
    float* bp = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&bp), (size_t)combos * p.bp_combo_stride * 4, s) != cudaSuccess) return -1;
    p.bp = bp;
    {
      const int64_t work = combos * p.tiles_n * p.nchunk * p.NT * KC;
      int blocks = (int)std::min<int64_t>((work + 255) / 256, 148 * 16);
      k_bprime<<<blocks < 1 ? 1 : blocks, 256, 0, s>>>(p, combos);
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    p.items = p.Z * p.tiles_m * p.tiles_n;
    p.per_cta = (p.items + sms - 1) / sms;
    const int64_t grid = (p.items + p.per_cta - 1) / p.per_cta;
    const size_t smem = tg_smem_bytes(p.NT, KC);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_tc_gemm<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      cudaFuncSetAttribute(k_tc_gemm<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      cudaFuncSetAttribute(k_tc_gemm<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      attr = true;
    }
    if (KC == 16) k_tc_gemm<16><<<(unsigned)grid, TG_THREADS, smem, s>>>(p);
    else if (KC == 8) k_tc_gemm<8><<<(unsigned)grid, TG_THREADS, smem, s>>>(p);
    else k_tc_gemm<4><<<(unsigned)grid, TG_THREADS, smem, s>>>(p);
    const bool ok = cudaGetLastError() == cudaSuccess;
    cudaFreeAsync(bp, s);
    return ok ? 1 : -1;
  }
}

}  // namespace tnc
