// libtnc C ABI: argument validation, kernel selection, launches.
// Declarations and the reference interfaces each entry point replaces are in
// include/tnc.h.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <algorithm>
#include <string>
#include <vector>
#include "tnc_kernels.cuh"
#include "tnc_pair.cuh"
#include "tnc_tc.cuh"
#include "tnc_dmma.cuh"
#include "tnc_tcgemm.cuh"

namespace {

thread_local std::string g_err;

// TNC_KERNELS=simt disables the tensor-core paths (tests compare both);
// "tc-resident" / "tc-gemm" keep only one of them (precision probes).
int tc_mask() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TNC_KERNELS");
    v = 3;
    if (e && strcmp(e, "simt") == 0) v = 0;
    if (e && strcmp(e, "tc-resident") == 0) v = 1;
    if (e && strcmp(e, "tc-gemm") == 0) v = 2;
  }
  return v;
}
bool tc_enabled() { return tc_mask() != 0; }
// measured: K <= 4 stays on the SIMT column kernel (16-byte stores, 3.8 vs
// 3.5 TB/s at K=4, N=64); K >= 8 with K*N >= 256 goes to tcgen05
bool pair_use_tc(int64_t K, int64_t N) { return K * N >= 256 && K >= 8; }

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TNC_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return TNC_OK;
}

int grid_for(int64_t work, int threads, int64_t cap = 148LL * 64) {
  int64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (int)b;
}

template <typename R>
int launch_project(const tnc_project_desc& d, cudaStream_t s) {
  int64_t elems = 1;
  for (int j = 0; j < d.nd; ++j) elems *= d.dim[j];
  if (d.Z <= 0) return TNC_OK;
  tnc::k_project<R><<<grid_for(d.Z * elems, 256), 256, 0, s>>>(d, elems);
  return check_launch("tnc_project");
}

template <typename R, int NMAX>
void skinny_acc(const tnc_step_desc& d, cudaStream_t s) {
  const int64_t rows = d.Z * d.M;
  tnc::k_step_skinny_acc<R, NMAX><<<(unsigned)((rows + 127) / 128), 128, 0, s>>>(d);
}
template <typename R, int KMAX>
void skinny_row(const tnc_step_desc& d, cudaStream_t s) {
  const int64_t rows = d.Z * d.M;
  tnc::k_step_skinny_row<R, KMAX><<<(unsigned)((rows + 127) / 128), 128, 0, s>>>(d);
}

template <int L>
void warp_step(const tnc_step_desc& d, cudaStream_t s) {
  // grid: x over row groups of one z, y over z; about 16 warps-worth per SM in total
  const int64_t zb = std::min<int64_t>(d.Z, 65535);
  const int64_t warps_needed = (d.M + (32 / L) * 4 - 1) / ((32 / L) * 4);
  const int64_t bx = std::max<int64_t>(1, std::min<int64_t>((warps_needed + 7) / 8, (148 * 16 + zb - 1) / zb));
  const dim3 grid((unsigned)bx, (unsigned)zb);
  if (d.N <= 1) tnc::k_step_warp<L, 1><<<grid, 256, 0, s>>>(d);
  else if (d.N <= 2) tnc::k_step_warp<L, 2><<<grid, 256, 0, s>>>(d);
  else if (d.N <= 4) tnc::k_step_warp<L, 4><<<grid, 256, 0, s>>>(d);
  else if (d.N <= 8) tnc::k_step_warp<L, 8><<<grid, 256, 0, s>>>(d);
  else tnc::k_step_warp<L, 16><<<grid, 256, 0, s>>>(d);
}

template <typename R>
bool splitk(const tnc_step_desc& d, cudaStream_t s) {
  using C = typename tnc::cplx<R>::T;
  constexpr int BM = 64, BN = 32, BK = 16;
  const int64_t rows = d.Z * d.M;
  const int64_t tiles_n = (d.N + BN - 1) / BN;
  const int64_t tiles = ((rows + BM - 1) / BM) * tiles_n;
  int64_t splits = std::max<int64_t>(1, (148 * 8 + tiles - 1) / tiles);
  int64_t ks = (d.K + splits - 1) / splits;
  ks = (ks + BK - 1) / BK * BK;
  splits = (d.K + ks - 1) / ks;
  if (splits > 65535) return false;
  tnc::pool_keep();
  C* W = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&W), (size_t)splits * rows * d.N * sizeof(C), s) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  tnc::k_step_splitk<R, BM, BN, BK, 4, 2><<<dim3((unsigned)tiles, (unsigned)splits), (BM / 4) * (BN / 2), 0, s>>>(
      d, tiles_n, ks, W);
  tnc::k_splitk_reduce<R><<<grid_for(rows * d.N, 256), 256, 0, s>>>(d, splits, W);
  cudaFreeAsync(W, s);
  return true;
}

template <typename R>
bool try_skinny(const tnc_step_desc& d, cudaStream_t s, bool& fused_amax) {
  fused_amax = false;
  if (!d.a_rows_contig || !d.b_dense || d.conj_b) return false;
  if (d.Z * d.M > (int64_t)0x7fffffff * 128) return false;
  const int64_t N = d.N, K = d.K;
  // few rows with a long K and real work: split-K register-blocked partials
  // plus a fixed-order reduction (a warp per result re-reads the site block
  // once per row: 11 ms for M = 1024, K = 32768, N = 64)
  if (d.Z * d.M < 4096 && K >= 2048 && d.Z * d.M * N * K >= ((int64_t)1 << 26) &&
      (d.site.sel == nullptr || d.Z == 1) && d.site.ncut == 0 && d.site.zstride == 0) {
    if (splitk<R>(d, s)) return true;
  }
  // few rows (path ends: tiny M, large K or N): one thread per result element
  if (d.Z * d.M < 4096) {
    if (K >= 256 && d.Z * d.M * N <= (int64_t)148 * 64 * 8)   // long K: a warp per result
      tnc::k_step_dot<R><<<grid_for(d.Z * d.M * N * 32, 256), 256, 0, s>>>(d);
    else
      tnc::k_step_cols<R><<<grid_for(d.Z * d.M * N, 256), 256, 0, s>>>(d);
    return true;
  }
  // complex64, K = 2..64 (power of two), N <= 16: warp-cooperative coalesced rows
  if (sizeof(R) == 4 && N <= 16 && K * N < 256 && K >= 2 && K <= 64 && (K & (K - 1)) == 0 &&
      ((uintptr_t)d.acc % 16) == 0 && (d.acc_zstride % 2) == 0 && d.M < 0x7fffffffLL &&
      d.out_zstride < 0x7fffffffLL) {
    fused_amax = true;                           // k_step_warp records amax_out itself
    switch (K) {
      case 2: warp_step<1>(d, s); return true;
      case 4: warp_step<2>(d, s); return true;
      case 8: warp_step<4>(d, s); return true;
      case 16: warp_step<8>(d, s); return true;
      case 32: warp_step<16>(d, s); return true;
      default: warp_step<32>(d, s); return true;
    }
  }
  if (N <= 32) {
    if (N <= 1) skinny_acc<R, 1>(d, s);
    else if (N <= 2) skinny_acc<R, 2>(d, s);
    else if (N <= 4) skinny_acc<R, 4>(d, s);
    else if (N <= 8) skinny_acc<R, 8>(d, s);
    else if (N <= 16) skinny_acc<R, 16>(d, s);
    else skinny_acc<R, 32>(d, s);
    return true;
  }
  if (K <= 32) {
    if (K <= 1) skinny_row<R, 1>(d, s);
    else if (K <= 2) skinny_row<R, 2>(d, s);
    else if (K <= 4) skinny_row<R, 4>(d, s);
    else if (K <= 8) skinny_row<R, 8>(d, s);
    else if (K <= 16) skinny_row<R, 16>(d, s);
    else skinny_row<R, 32>(d, s);
    return true;
  }
  return false;
}

template <typename R>
void generic(const tnc_step_desc& d, cudaStream_t s) {
  constexpr int BM = 64, BN = 32, BK = 16, TM = 4, TN = 2;
  const int64_t tm = (d.M + BM - 1) / BM, tn = (d.N + BN - 1) / BN;
  tnc::k_step_generic<R, BM, BN, BK, TM, TN><<<(unsigned)(d.Z * tm * tn), (BM / TM) * (BN / TN), 0, s>>>(d, tm, tn);
}

// max |re|, |im| of out[z][0 .. M*N) for the kernels without a fused amax
int launch_amax(const tnc_step_desc& d, cudaStream_t s) {
  const int64_t count = d.M * d.N;
  const int64_t zb = d.Z < 65535 ? d.Z : 65535;
  int64_t bx = (count + 256 * 8 - 1) / (256 * 8);
  const int64_t cap = std::max<int64_t>(1, 148 * 8 / zb);
  if (bx > cap) bx = cap;
  tnc::k_amax<<<dim3((unsigned)bx, (unsigned)zb), 256, 0, s>>>(reinterpret_cast<const float2*>(d.out), d.Z,
                                                              d.out_zstride, count, d.amax_out);
  return check_launch("tnc_step[amax]");
}

template <typename R>
int launch_step_kernel(const tnc_step_desc& d, cudaStream_t s, bool& fused_amax) {
  int kernel = d.kernel;
  fused_amax = false;
  if (kernel == TNC_K_TC || (kernel == TNC_K_AUTO && tc_enabled())) {
    const int mask = kernel == TNC_K_TC ? 3 : tc_mask();
    int rc = 0;
    // with an input bound the fp16-split GEMM outruns the 3xTF32 resident kernel
    const bool gemm_first = sizeof(R) == 4 && d.amax_in != nullptr && (mask & 2) && tnc::tc16_enabled();
    if (gemm_first) {
      rc = tnc::try_tc_gemm<R>(d, s);
      if (rc == 1) fused_amax = true;
    }
    if (rc == 0 && (mask & 1)) rc = sizeof(R) == 8 ? tnc::try_dmma<R>(d, s) : tnc::try_tc<R>(d, s);
    if (rc == 0 && !gemm_first && (mask & 2) && sizeof(R) == 4) {
      rc = tnc::try_tc_gemm<R>(d, s);
      if (rc == 1) fused_amax = true;
    }
    if (rc == 1) return check_launch("tnc_step[tc]");
    if (rc < 0) return check_launch("tnc_step[tc] launch");
    if (kernel == TNC_K_TC) return fail(TNC_E_UNSUPPORTED, "tnc_step: shape outside the tensor-core kernel envelope");
  }
  if (kernel == TNC_K_SKINNY || kernel == TNC_K_AUTO) {
    if (try_skinny<R>(d, s, fused_amax)) return check_launch("tnc_step[skinny]");
    if (kernel == TNC_K_SKINNY) return fail(TNC_E_UNSUPPORTED, "tnc_step: shape outside the skinny kernel envelope");
  }
  if (d.a_koff == nullptr || d.b_koff == nullptr || d.b_noff == nullptr || d.c_noff == nullptr)
    return fail(TNC_E_INVALID, "tnc_step: generic kernel needs all four offset tables");
  generic<R>(d, s);
  return check_launch("tnc_step[generic]");
}

template <typename R>
int launch_step(const tnc_step_desc& d, cudaStream_t s) {
  if (d.Z <= 0 || d.M <= 0 || d.N <= 0) return TNC_OK;
  if (d.K <= 0) return fail(TNC_E_INVALID, "tnc_step: K must be >= 1");
  if (d.nf < 0 || d.nf > TNC_MAX_LEGS) return fail(TNC_E_INVALID, "tnc_step: nf=%d", d.nf);
  if (d.site.ncut < 0 || d.site.ncut > TNC_MAX_CUTS) return fail(TNC_E_INVALID, "tnc_step: ncut=%d", d.site.ncut);
  const bool want_amax = d.amax_out != nullptr && sizeof(R) == 4;
  if (want_amax && cudaMemsetAsync(d.amax_out, 0, (size_t)d.Z * sizeof(float), s) != cudaSuccess)
    return check_launch("tnc_step[amax zero]");
  bool fused = false;
  const int rc = launch_step_kernel<R>(d, s, fused);
  if (rc != TNC_OK || !want_amax || fused) return rc;
  return launch_amax(d, s);
}

template <typename R>
int launch_slice_sum(const tnc_slice_sum_desc& d, cudaStream_t s) {
  if (d.B <= 0) return TNC_OK;
  const int64_t threads = d.B * 32;
  tnc::k_slice_sum<R><<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(d);
  return check_launch("tnc_slice_sum");
}

bool dtype_ok(int dt) { return dt == TNC_C64 || dt == TNC_C128; }


template <typename R, typename KFN>
int launch_tiled_fn(KFN kern, const tnc::PairTile& p, int64_t batch, const void* a, const void* b, void* out,
                    cudaStream_t s) {
  using C = typename tnc::cplx<R>::T;
  const size_t smem = (size_t)(p.Kout * p.Lseg + p.K * p.N) * sizeof(C) + (size_t)p.K * 4;
  if (smem > 48 * 1024) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return check_launch("tnc_contract_pair: smem attribute");
  }
  const int64_t blocks = batch * p.U;
  if (blocks <= 0) return TNC_OK;
  if (blocks > 0x7fffffffLL) return fail(TNC_E_UNSUPPORTED, "tnc_contract_pair: grid too large");
  kern<<<(unsigned)blocks, 256, smem, s>>>(p, a, b, out);
  return check_launch("tnc_contract_pair[tiled]");
}

template <typename R, typename KFN>
int launch_pipe_fn(KFN kern, const tnc::PairTile& p, int64_t batch, const void* a, const void* b, void* out,
                   cudaStream_t s, bool cols = false, bool prod = false) {
  const int threads = prod ? tnc::PIPE_THREADS : 256;
  using C = typename tnc::cplx<R>::T;
  const size_t smem = cols ? 128 + (size_t)tnc::PIPE_STAGES * p.Kout * p.Lseg * sizeof(C) + (size_t)64 * 4 + (size_t)p.R * 4 + 16
                           : 128 + (size_t)tnc::PIPE_STAGES * p.Kout * p.Lseg * sizeof(C)
                             + (size_t)p.K * (p.N + 1) * sizeof(C) + (size_t)p.K * 4 + (size_t)p.R * 4 + 16;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return check_launch("tnc pair pipe: smem attribute");
  const int64_t total = batch * p.U;
  if (total <= 0) return TNC_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t ctas = std::min<int64_t>(total, (int64_t)sms * per_sm);
  const int64_t per = (total + ctas - 1) / ctas;
  const int64_t grid = (total + per - 1) / per;
  kern<<<(unsigned)grid, threads, smem, s>>>(p, a, b, out, total, per);
  return check_launch("tnc_contract_pair[pipe]");
}

bool pipe_eligible(const tnc::PairTile& p, size_t elem, const void* a) {
  if ((p.Lseg * elem) % 16 != 0 || (p.a_zstride * elem) % 16 != 0 || ((uintptr_t)a) % 16 != 0) return false;
  for (int j = 0; j < p.nfo; ++j) if ((p.fo_stride[j] * elem) % 16 != 0) return false;
  return true;   // segoff are sums of outer strides, multiples of Lseg
}

template <typename R>
int launch_pair_tiled(const tnc::PairTile& p, int64_t batch, const void* a, const void* b, void* out,
                      cudaStream_t s) {
  using C = typename tnc::cplx<R>::T;
  const int64_t N = p.N, K = p.K;
  if (p.pipe && pipe_eligible(p, sizeof(C), a)) {
    if (N >= 8 && N <= 256 && (256 % N) == 0 && K <= (sizeof(R) == 4 ? 64 : 16)) {
      // two columns per thread (16-byte stores) when the rows stay 16-byte aligned
      if (sizeof(R) == 4 && N >= 16 && ((uintptr_t)out % 16) == 0) {
        if (K <= 4) return launch_pipe_fn<R>(tnc::k_pair_pipe_cols<R, 4, 2>, p, batch, a, b, out, s, true);
        if (K <= 16) return launch_pipe_fn<R>(tnc::k_pair_pipe_cols<R, 16, 2>, p, batch, a, b, out, s, true);
      }
      if (K <= 4) return launch_pipe_fn<R>(tnc::k_pair_pipe_cols<R, 4>, p, batch, a, b, out, s, true);
      if (K <= 16) return launch_pipe_fn<R>(tnc::k_pair_pipe_cols<R, 16>, p, batch, a, b, out, s, true);
      if constexpr (sizeof(R) == 4) return launch_pipe_fn<R>(tnc::k_pair_pipe_cols<R, 64>, p, batch, a, b, out, s, true);
    }
    if (N <= 32) {
      // K >= 8: producer-warp variant (mbarrier stage release, no CTA barrier per tile)
      if (K >= 8 && N <= 4) {
        if (N <= 1) return launch_pipe_fn<R>(tnc::k_pair_pipe<R, 1, 0, true>, p, batch, a, b, out, s, false, true);
        if (N <= 2) return launch_pipe_fn<R>(tnc::k_pair_pipe<R, 2, 0, true>, p, batch, a, b, out, s, false, true);
        return launch_pipe_fn<R>(tnc::k_pair_pipe<R, 4, 0, true>, p, batch, a, b, out, s, false, true);
      }
      if (N <= 1) return launch_pipe_fn<R>(tnc::k_pair_pipe<R, 1, 0>, p, batch, a, b, out, s);
      if (N <= 2) return launch_pipe_fn<R>(tnc::k_pair_pipe<R, 2, 0>, p, batch, a, b, out, s);
      if (N <= 4) return launch_pipe_fn<R>(tnc::k_pair_pipe<R, 4, 0>, p, batch, a, b, out, s);
      if (N <= 8) return launch_pipe_fn<R>(tnc::k_pair_pipe<R, 8, 0>, p, batch, a, b, out, s);
      if (N <= 16) return launch_pipe_fn<R>(tnc::k_pair_pipe<R, 16, 0>, p, batch, a, b, out, s);
      return launch_pipe_fn<R>(tnc::k_pair_pipe<R, 32, 0>, p, batch, a, b, out, s);
    }
    if (K <= 1) return launch_pipe_fn<R>(tnc::k_pair_pipe<R, 1, 1>, p, batch, a, b, out, s);
    if (K <= 2) return launch_pipe_fn<R>(tnc::k_pair_pipe<R, 1, 2>, p, batch, a, b, out, s);
    if (K <= 4) return launch_pipe_fn<R>(tnc::k_pair_pipe<R, 1, 4>, p, batch, a, b, out, s);
    if (K <= 8) return launch_pipe_fn<R>(tnc::k_pair_pipe<R, 1, 8>, p, batch, a, b, out, s);
    return launch_pipe_fn<R>(tnc::k_pair_pipe<R, 1, 16>, p, batch, a, b, out, s);
  }
  if (N <= 32) {
    if (N <= 1) return launch_tiled_fn<R>(tnc::k_pair_tiled_acc<R, 1>, p, batch, a, b, out, s);
    if (N <= 2) return launch_tiled_fn<R>(tnc::k_pair_tiled_acc<R, 2>, p, batch, a, b, out, s);
    if (N <= 4) return launch_tiled_fn<R>(tnc::k_pair_tiled_acc<R, 4>, p, batch, a, b, out, s);
    if (N <= 8) return launch_tiled_fn<R>(tnc::k_pair_tiled_acc<R, 8>, p, batch, a, b, out, s);
    if (N <= 16) return launch_tiled_fn<R>(tnc::k_pair_tiled_acc<R, 16>, p, batch, a, b, out, s);
    return launch_tiled_fn<R>(tnc::k_pair_tiled_acc<R, 32>, p, batch, a, b, out, s);
  }
  if (K <= 1) return launch_tiled_fn<R>(tnc::k_pair_tiled_row<R, 1>, p, batch, a, b, out, s);
  if (K <= 2) return launch_tiled_fn<R>(tnc::k_pair_tiled_row<R, 2>, p, batch, a, b, out, s);
  if (K <= 4) return launch_tiled_fn<R>(tnc::k_pair_tiled_row<R, 4>, p, batch, a, b, out, s);
  if (K <= 8) return launch_tiled_fn<R>(tnc::k_pair_tiled_row<R, 8>, p, batch, a, b, out, s);
  return launch_tiled_fn<R>(tnc::k_pair_tiled_row<R, 16>, p, batch, a, b, out, s);
}

}  // namespace

extern "C" {

int tnc_version(void) { return 101; }

size_t tnc_struct_size(int which) {
  switch (which) {
    case 0: return sizeof(tnc_site);
    case 1: return sizeof(tnc_step_desc);
    case 2: return sizeof(tnc_project_desc);
    case 3: return sizeof(tnc_slice_sum_desc);
    case 4: return sizeof(tnc_path_desc);
    default: return 0;
  }
}

const char* tnc_last_error(void) { return g_err.c_str(); }

int tnc_device_check(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(TNC_E_NODEVICE, "no CUDA device");
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return fail(TNC_E_NODEVICE, "cudaGetDeviceProperties failed");
  if (p.major != 10) return fail(TNC_E_NODEVICE, "device %s is sm_%d%d, libtnc is built for sm_100a", p.name, p.major, p.minor);
  return TNC_OK;
}

int tnc_project(const tnc_project_desc* d, void* stream) {
  if (!d || !dtype_ok(d->dtype)) return fail(TNC_E_INVALID, "tnc_project: bad descriptor");
  if (d->nd < 0 || d->nd > TNC_MAX_LEGS) return fail(TNC_E_INVALID, "tnc_project: nd=%d", d->nd);
  if (d->slices_per_b <= 0) return fail(TNC_E_INVALID, "tnc_project: slices_per_b must be >= 1");
  cudaStream_t s = (cudaStream_t)stream;
  return d->dtype == TNC_C64 ? launch_project<float>(*d, s) : launch_project<double>(*d, s);
}

int tnc_step(const tnc_step_desc* d, void* stream) {
  if (!d || !dtype_ok(d->dtype)) return fail(TNC_E_INVALID, "tnc_step: bad descriptor");
  if (d->slices_per_b <= 0) return fail(TNC_E_INVALID, "tnc_step: slices_per_b must be >= 1");
  cudaStream_t s = (cudaStream_t)stream;
  return d->dtype == TNC_C64 ? launch_step<float>(*d, s) : launch_step<double>(*d, s);
}

int tnc_slice_sum(const tnc_slice_sum_desc* d, void* stream) {
  if (!d || !dtype_ok(d->dtype) || d->slices_per_b <= 0) return fail(TNC_E_INVALID, "tnc_slice_sum: bad descriptor");
  cudaStream_t s = (cudaStream_t)stream;
  return d->dtype == TNC_C64 ? launch_slice_sum<float>(*d, s) : launch_slice_sum<double>(*d, s);
}

int tnc_contract_path(const tnc_path_desc* d, void* stream) {
  if (!d || d->nsteps < 0 || (d->nsteps > 0 && !d->steps)) return fail(TNC_E_INVALID, "tnc_contract_path: bad descriptor");
  int rc = tnc_project(&d->first, stream);
  if (rc) return rc;
  for (int i = 0; i < d->nsteps; ++i) {
    rc = tnc_step(&d->steps[i], stream);
    if (rc) {
      std::string m = g_err;
      return fail(rc, "step %d: %s", i, m.c_str());
    }
  }
  return tnc_slice_sum(&d->reduce, stream);
}

// ---------------------------------------------------------------------------
// Pairwise contraction plans (tensor.py:103 contract_pair).  The host side
// computes the layout once -- which kernel, its tile geometry and offset
// tables -- into one byte blob; the blob lives either in caller workspace
// (one-shot tnc_contract_pair) or in plan-owned device memory.
// ---------------------------------------------------------------------------
}  // extern "C"

struct tnc_pair_plan {
  int dtype = 0;
  int kind = TNC_K_GENERIC;        // TNC_K_GENERIC or TNC_K_SKINNY (tiled)
  tnc_step_desc d;                 // generic launch template (tables patched)
  tnc::PairTile pt;                // tiled launch template (tables patched)
  std::vector<unsigned char> blob; // host copy of the tables
  size_t o_ak = 0, o_bk = 0, o_bn = 0, o_cn = 0, o_seg = 0, o_row = 0, o_k = 0;
  void* dmem = nullptr;            // plan-owned device copy (plan API)
  bool a_align_needed = false;     // tiled vec16 requires 16-byte aligned a
  bool tc_ok = false;              // tensor-core kernel envelope (complex64)
  tnc::TcDesc tc;                  // tensor-core launch template
  size_t o_lo = 0;                 // lo_off table (128 int64) in the blob
  size_t o_holo = 0, o_hohi = 0;   // two-level row-block base tables
  bool has_ho = false;
  size_t o_tcseg = 0, o_tckraw = 0; // tensor-core raw-ring tables
  size_t o_folo = 0, o_fohi = 0;   // two-level tile base tables (SIMT tiles)
  bool has_fo = false;
};

namespace {

void pair_layout(int a_rank, const int64_t* a_dims, int b_rank, const int64_t* b_dims,
                 int npairs, const int32_t* pa, const int32_t* pb,
                 std::vector<int>& fa, std::vector<int>& fb, int64_t& K, int64_t& N) {
  std::vector<char> ua(a_rank, 0), ub(b_rank, 0);
  for (int i = 0; i < npairs; ++i) { ua[pa[i]] = 1; ub[pb[i]] = 1; }
  fa.clear(); fb.clear();
  for (int i = 0; i < a_rank; ++i) if (!ua[i]) fa.push_back(i);
  for (int i = 0; i < b_rank; ++i) if (!ub[i]) fb.push_back(i);
  K = 1; N = 1;
  for (int i = 0; i < npairs; ++i) K *= a_dims[pa[i]];
  for (int i : fb) N *= b_dims[i];
}

int build_pair_plan(tnc_pair_plan& P, int dtype, int a_rank, const int64_t* a_dims, int b_rank,
                    const int64_t* b_dims, int npairs, const int32_t* pair_a, const int32_t* pair_b,
                    const int32_t* out_perm, int conj_b) {
  if (!dtype_ok(dtype)) return fail(TNC_E_INVALID, "contract_pair: bad dtype %d", dtype);
  if (a_rank < 0 || b_rank < 0 || a_rank > TNC_MAX_LEGS || b_rank > TNC_MAX_LEGS)
    return fail(TNC_E_INVALID, "contract_pair: rank out of range");
  if (npairs < 0 || npairs > a_rank || npairs > b_rank) return fail(TNC_E_INVALID, "contract_pair: bad npairs");
  std::vector<char> ua(a_rank, 0), ub(b_rank, 0);
  for (int i = 0; i < npairs; ++i) {
    if (pair_a[i] < 0 || pair_a[i] >= a_rank || pair_b[i] < 0 || pair_b[i] >= b_rank)
      return fail(TNC_E_INVALID, "axis pair (%d, %d) out of range", pair_a[i], pair_b[i]);
    if (ua[pair_a[i]] || ub[pair_b[i]]) return fail(TNC_E_INVALID, "axis repeated in pairs: (%d, %d)", pair_a[i], pair_b[i]);
    ua[pair_a[i]] = ub[pair_b[i]] = 1;
    if (a_dims[pair_a[i]] != b_dims[pair_b[i]])
      return fail(TNC_E_INVALID, "extent mismatch on pair (%d, %d)", pair_a[i], pair_b[i]);
  }
  for (int i = 0; i < a_rank; ++i) if (a_dims[i] < 1) return fail(TNC_E_INVALID, "axis extent < 1");
  for (int i = 0; i < b_rank; ++i) if (b_dims[i] < 1) return fail(TNC_E_INVALID, "axis extent < 1");
  std::vector<int> fa, fb;
  int64_t K, N;
  pair_layout(a_rank, a_dims, b_rank, b_dims, npairs, pair_a, pair_b, fa, fb, K, N);
  std::vector<int64_t> sa(a_rank), sb(b_rank);
  { int64_t s = 1; for (int i = a_rank - 1; i >= 0; --i) { sa[i] = s; s *= a_dims[i]; } }
  { int64_t s = 1; for (int i = b_rank - 1; i >= 0; --i) { sb[i] = s; s *= b_dims[i]; } }
  const int nout = (int)(fa.size() + fb.size());
  std::vector<int64_t> odims(nout);
  for (size_t i = 0; i < fa.size(); ++i) odims[i] = a_dims[fa[i]];
  for (size_t i = 0; i < fb.size(); ++i) odims[fa.size() + i] = b_dims[fb[i]];
  std::vector<int> perm(nout);
  for (int i = 0; i < nout; ++i) perm[i] = out_perm ? out_perm[i] : i;
  std::vector<char> seen(nout, 0);
  for (int i = 0; i < nout; ++i) {
    if (perm[i] < 0 || perm[i] >= nout || seen[perm[i]]) return fail(TNC_E_INVALID, "contract_pair: bad out_perm");
    seen[perm[i]] = 1;
  }
  std::vector<int64_t> ostr(nout);  // out stride of natural axis j
  { int64_t s = 1; for (int i = nout - 1; i >= 0; --i) { ostr[perm[i]] = s; s *= odims[perm[i]]; } }

  P.dtype = dtype;
  // generic tables: a_koff[K], b_koff[K], b_noff[N], c_noff[N]
  std::vector<int64_t> tab(2 * K + 2 * N);
  for (int64_t k = 0; k < K; ++k) {
    int64_t r = k, oa = 0, ob = 0;
    for (int i = npairs - 1; i >= 0; --i) {
      const int64_t dm = a_dims[pair_a[i]];
      oa += (r % dm) * sa[pair_a[i]];
      ob += (r % dm) * sb[pair_b[i]];
      r /= dm;
    }
    tab[k] = oa; tab[K + k] = ob;
  }
  for (int64_t n = 0; n < N; ++n) {
    int64_t r = n, obn = 0, ocn = 0;
    for (int i = (int)fb.size() - 1; i >= 0; --i) {
      const int64_t dm = b_dims[fb[i]];
      obn += (r % dm) * sb[fb[i]];
      ocn += (r % dm) * ostr[fa.size() + i];
      r /= dm;
    }
    tab[2 * K + n] = obn; tab[2 * K + N + n] = ocn;
  }
  tnc_step_desc& d = P.d;
  memset(&d, 0, sizeof d);
  d.dtype = dtype;
  d.kernel = TNC_K_GENERIC;
  d.slices_per_b = 1;
  d.conj_b = conj_b ? 1 : 0;
  d.nf = (int)fa.size();
  d.M = 1;
  for (size_t i = 0; i < fa.size(); ++i) {
    d.f_dim[i] = a_dims[fa[i]];
    d.f_astride[i] = sa[fa[i]];
    d.f_cstride[i] = ostr[i];
    d.M *= a_dims[fa[i]];
  }
  d.K = K; d.N = N;

  bool identity_a = true;
  for (size_t i = 0; i < fa.size(); ++i) identity_a = identity_a && perm[i] == (int)i;
  const int64_t tile_max = dtype == TNC_C64 ? 4096 : 2048;   // one ring stage: 32 KiB
  std::vector<int64_t> segoff, folo, fohi;
  std::vector<int32_t> rowoff, koff;
  P.kind = TNC_K_GENERIC;
  if (identity_a && K * N <= 4096 && (N <= 32 || K <= 16) && a_rank > 0) {
    std::vector<char> shared(a_rank, 0);
    for (int i = 0; i < npairs; ++i) shared[pair_a[i]] = 1;
    int t = a_rank;
    int64_t lseg = 1, kout = K;
    while (t > 0) {
      const int64_t dm = a_dims[t - 1];
      const int64_t nl = lseg * dm, nk = shared[t - 1] ? kout / dm : kout;
      if (nk * nl > tile_max) break;
      lseg = nl; kout = nk; --t;
    }
    const int64_t tile = kout * lseg, R = tile / K;
    if (tile <= tile_max && R >= 1) {
      tnc::PairTile& pt = P.pt;
      memset(&pt, 0, sizeof pt);
      std::vector<int> of, os, inf;
      for (int i = 0; i < a_rank; ++i) {
        if (i < t) (shared[i] ? os : of).push_back(i);
        else if (!shared[i]) inf.push_back(i);
      }
      pt.nfo = (int)of.size();
      pt.U = 1;
      for (size_t j = 0; j < of.size(); ++j) { pt.fo_dim[j] = a_dims[of[j]]; pt.fo_stride[j] = sa[of[j]]; pt.U *= a_dims[of[j]]; }
      pt.conj_b = conj_b ? 1 : 0;
      pt.Kout = kout; pt.Lseg = lseg; pt.R = R; pt.K = K; pt.N = N;
      {
        const int nfo = pt.nfo;
        int split = nfo;
        int64_t plo = 1;
        while (split > 0 && plo * pt.fo_dim[split - 1] <= 4096) { plo *= pt.fo_dim[split - 1]; --split; }
        int64_t phi = 1;
        for (int i = 0; i < split; ++i) phi *= pt.fo_dim[i];
        if (nfo > 1 && phi <= (1 << 20)) {
          auto fill = [&](int from, int to, int64_t count, std::vector<int64_t>& outv) {
            outv.resize(count);
            for (int64_t m = 0; m < count; ++m) {
              int64_t r = m, off = 0;
              for (int i = to - 1; i >= from; --i) { off += (r % pt.fo_dim[i]) * pt.fo_stride[i]; r /= pt.fo_dim[i]; }
              outv[m] = off;
            }
          };
          fill(split, nfo, plo, folo);
          fill(0, split, phi, fohi);
          pt.f_plo = plo;
        }
      }
      segoff.resize(kout);
      std::vector<int64_t> segw(a_rank, 0);
      { int64_t w = 1; for (int j = (int)os.size() - 1; j >= 0; --j) { segw[os[j]] = w; w *= a_dims[os[j]]; } }
      for (int64_t j = 0; j < kout; ++j) {
        int64_t r = j, off = 0;
        for (int q = (int)os.size() - 1; q >= 0; --q) { off += (r % a_dims[os[q]]) * sa[os[q]]; r /= a_dims[os[q]]; }
        segoff[j] = off;
      }
      rowoff.resize(R);
      koff.resize(K);
      for (int64_t r0 = 0; r0 < R; ++r0) {
        int64_t r = r0, off = 0;
        for (int q = (int)inf.size() - 1; q >= 0; --q) { off += (r % a_dims[inf[q]]) * sa[inf[q]]; r /= a_dims[inf[q]]; }
        rowoff[r0] = (int32_t)off;
      }
      for (int64_t k0 = 0; k0 < K; ++k0) {
        int64_t r = k0, seg = 0, inner = 0;
        for (int i = npairs - 1; i >= 0; --i) {
          const int ax = pair_a[i];
          const int64_t dm = a_dims[ax], dg = r % dm;
          r /= dm;
          if (ax < t) seg += dg * segw[ax]; else inner += dg * sa[ax];
        }
        koff[k0] = (int32_t)(seg * lseg + inner);
      }
      bool v16 = dtype == TNC_C64 && (lseg % 2 == 0);
      for (int64_t j = 0; j < kout && v16; ++j) v16 = (segoff[j] % 2 == 0);
      pt.vec16 = v16 ? 1 : 0;
      pt.pipe = 1;
      P.a_align_needed = v16;
      P.kind = TNC_K_SKINNY;
    }
  }
  // tensor-core envelope: complex64, identity result layout, a 128-row block
  // made of the innermost free legs
  std::vector<int64_t> looff, holo, hohi, tcseg;
  std::vector<int32_t> tckraw;
  {
    bool identity = true;
    for (int i = 0; i < nout; ++i) identity = identity && perm[i] == i;
    if (dtype == TNC_C64 && identity && tnc::tc_shape_ok(K, N, d.M)) {
      std::vector<char> shared(a_rank, 0);
      for (int i = 0; i < npairs; ++i) shared[pair_a[i]] = 1;
      int64_t prod_in = 1;
      int t = a_rank;
      std::vector<int> inner;
      while (t > 0 && prod_in < 128) {
        --t;
        if (!shared[t]) { inner.insert(inner.begin(), t); prod_in *= a_dims[t]; }
      }
      if (prod_in == 128) {
        tnc::TcDesc& c = P.tc;
        memset(&c, 0, sizeof c);
        c.M = d.M; c.K = K; c.N = N;
        c.conj_b = conj_b ? 1 : 0;
        c.slices_per_b = 1;
        int nho = 0;
        for (int i = 0; i < t; ++i) if (!shared[i]) { c.ho_dim[nho] = a_dims[i]; c.ho_stride[nho] = sa[i]; ++nho; }
        c.nho = nho;
        // two-level row-block base tables over the outer free legs
        {
          int split = nho;                 // legs [split, nho) form the low group
          int64_t plo = 1;
          while (split > 0 && plo * c.ho_dim[split - 1] <= 4096) { plo *= c.ho_dim[split - 1]; --split; }
          int64_t phi = 1;
          for (int i = 0; i < split; ++i) phi *= c.ho_dim[i];
          if (phi <= (1 << 20) && plo * phi < (1LL << 31)) {
            auto fill = [&](int from, int to, int64_t count, std::vector<int64_t>& outv) {
              outv.resize(count);
              for (int64_t m = 0; m < count; ++m) {
                int64_t r = m, off = 0;
                for (int i = to - 1; i >= from; --i) { off += (r % c.ho_dim[i]) * c.ho_stride[i]; r /= c.ho_dim[i]; }
                outv[m] = off;
              }
            };
            fill(split, nho, plo, holo);
            fill(0, split, phi, hohi);
            c.p_lo = plo;
          }
        }
        // raw-ring geometry: span = legs [t, a_rank) (the 7 row legs + inner shared legs)
        {
          int64_t lseg = 1;
          for (int i = t; i < a_rank; ++i) lseg *= a_dims[i];
          std::vector<int> outer_sh;
          for (int i = 0; i < t; ++i) if (shared[i]) outer_sh.push_back(i);
          int64_t kout = 1;
          for (int i : outer_sh) kout *= a_dims[i];
          std::vector<int64_t> segw(a_rank, 0);
          { int64_t w = 1; for (int j = (int)outer_sh.size() - 1; j >= 0; --j) { segw[outer_sh[j]] = w; w *= a_dims[outer_sh[j]]; } }
          tcseg.resize(kout);
          for (int64_t j = 0; j < kout; ++j) {
            int64_t r = j, off = 0;
            for (int q = (int)outer_sh.size() - 1; q >= 0; --q) { off += (r % a_dims[outer_sh[q]]) * sa[outer_sh[q]]; r /= a_dims[outer_sh[q]]; }
            tcseg[j] = off;
          }
          tckraw.resize(K);
          for (int64_t k0 = 0; k0 < K; ++k0) {
            int64_t r = k0, seg = 0, inner = 0;
            for (int i = npairs - 1; i >= 0; --i) {
              const int ax = pair_a[i];
              const int64_t dm = a_dims[ax], dg = r % dm;
              r /= dm;
              if (ax < t) seg += dg * segw[ax]; else inner += dg * sa[ax];
            }
            tckraw[k0] = (int32_t)(seg * lseg + inner);
          }
          c.Kout = kout;
          c.Lseg = lseg;
          c.raw_ok = (kout * lseg == 128 * K && (lseg * 8) % 16 == 0) ? 1 : 0;
        }
        looff.resize(128);
        for (int r0 = 0; r0 < 128; ++r0) {
          int64_t r = r0, off = 0;
          for (int q = (int)inner.size() - 1; q >= 0; --q) { off += (r % a_dims[inner[q]]) * sa[inner[q]]; r /= a_dims[inner[q]]; }
          looff[r0] = off;
        }
        // converter bank spreading: when kraw is XOR-linear within a chunk, pick
        // per-row-bit k XORs so each half-warp's 16 rows hit 16 distinct 8-byte
        // bank slots (row bit i alone, or row bit i plus one k bit)
        {
          const int64_t KC = tnc::tc_kc(K);
          bool lin = (KC & (KC - 1)) == 0 && (int64_t)tckraw.size() == K;
          for (int64_t q = 0; q < K && lin; ++q)
            for (int64_t x = 0; x < KC && lin; ++x) lin = tckraw[q ^ x] == (tckraw[q] ^ tckraw[x]);
          if (lin) {
            uint32_t span = 1u;                  // GF(2) span of the chosen 4-bit slot vectors
            auto add = [&](int u) {
              uint32_t t2 = span;
              for (int v = 0; v < 16; ++v) if ((span >> v) & 1) t2 |= 1u << (v ^ u);
              span = t2;
            };
            for (int i = 0; i < 4; ++i) {
              const int u = (int)((looff[1 << i] - looff[0]) & 15);
              if (!((span >> u) & 1)) { add(u); continue; }
              for (int jb = 0; (1 << jb) < KC; ++jb) {
                const int w = (int)(tckraw[1 << jb] & 15);
                if (!((span >> (u ^ w)) & 1)) { P.tc.kx_row[i] = 1 << jb; add(u ^ w); break; }
              }
            }
            if (getenv("TNC_TC_NOXOR")) memset(P.tc.kx_row, 0, sizeof P.tc.kx_row);
          }
        }
        P.tc_ok = true;
      }
    }
  }
  // blob layout (8-byte aligned sections)
  size_t o = 0;
  P.o_ak = o; o += K * 8;
  P.o_bk = o; o += K * 8;
  P.o_bn = o; o += N * 8;
  P.o_cn = o; o += N * 8;
  P.o_seg = o; o += segoff.size() * 8;
  P.o_row = o; o += rowoff.size() * 4;
  o = (o + 7) & ~(size_t)7;
  P.o_k = o; o += koff.size() * 4;
  o = (o + 7) & ~(size_t)7;
  P.o_lo = o; o += looff.size() * 8;
  P.o_holo = o; o += holo.size() * 8;
  P.o_hohi = o; o += hohi.size() * 8;
  P.has_ho = !holo.empty();
  P.o_tcseg = o; o += tcseg.size() * 8;
  P.o_tckraw = o; o += tckraw.size() * 4;
  o = (o + 7) & ~(size_t)7;
  P.o_folo = o; o += folo.size() * 8;
  P.o_fohi = o; o += fohi.size() * 8;
  P.has_fo = !folo.empty();
  P.blob.assign(o + 8, 0);
  memcpy(P.blob.data() + P.o_ak, tab.data(), 2 * K * 8);                    // a_koff, b_koff
  memcpy(P.blob.data() + P.o_bn, tab.data() + 2 * K, N * 8 * 2);             // b_noff, c_noff
  if (!segoff.empty()) memcpy(P.blob.data() + P.o_seg, segoff.data(), segoff.size() * 8);
  if (!rowoff.empty()) memcpy(P.blob.data() + P.o_row, rowoff.data(), rowoff.size() * 4);
  if (!koff.empty()) memcpy(P.blob.data() + P.o_k, koff.data(), koff.size() * 4);
  if (!looff.empty()) memcpy(P.blob.data() + P.o_lo, looff.data(), looff.size() * 8);
  if (!holo.empty()) memcpy(P.blob.data() + P.o_holo, holo.data(), holo.size() * 8);
  if (!hohi.empty()) memcpy(P.blob.data() + P.o_hohi, hohi.data(), hohi.size() * 8);
  if (!tcseg.empty()) memcpy(P.blob.data() + P.o_tcseg, tcseg.data(), tcseg.size() * 8);
  if (!tckraw.empty()) memcpy(P.blob.data() + P.o_tckraw, tckraw.data(), tckraw.size() * 4);
  if (!folo.empty()) memcpy(P.blob.data() + P.o_folo, folo.data(), folo.size() * 8);
  if (!fohi.empty()) memcpy(P.blob.data() + P.o_fohi, fohi.data(), fohi.size() * 8);
  return TNC_OK;
}

void bind_tables(tnc_pair_plan& P, void* dev) {
  unsigned char* w = reinterpret_cast<unsigned char*>(dev);
  P.d.a_koff = reinterpret_cast<const int64_t*>(w + P.o_ak);
  P.d.b_koff = reinterpret_cast<const int64_t*>(w + P.o_bk);
  P.d.b_noff = reinterpret_cast<const int64_t*>(w + P.o_bn);
  P.d.c_noff = reinterpret_cast<const int64_t*>(w + P.o_cn);
  P.pt.b_koff = P.d.b_koff;
  P.pt.b_noff = P.d.b_noff;
  P.pt.segoff = reinterpret_cast<const int64_t*>(w + P.o_seg);
  P.pt.rowoff = reinterpret_cast<const int32_t*>(w + P.o_row);
  P.pt.koff = reinterpret_cast<const int32_t*>(w + P.o_k);
  P.tc.akoff = P.d.a_koff;
  P.tc.lo_off = reinterpret_cast<const int64_t*>(w + P.o_lo);
  P.tc.segoff = reinterpret_cast<const int64_t*>(w + P.o_tcseg);
  P.tc.kraw = reinterpret_cast<const int32_t*>(w + P.o_tckraw);
  P.pt.fo_lo = P.has_fo ? reinterpret_cast<const int64_t*>(w + P.o_folo) : nullptr;
  P.pt.fo_hi = P.has_fo ? reinterpret_cast<const int64_t*>(w + P.o_fohi) : nullptr;
  P.tc.ho_lo = P.has_ho ? reinterpret_cast<const int64_t*>(w + P.o_holo) : nullptr;
  P.tc.ho_hi = P.has_ho ? reinterpret_cast<const int64_t*>(w + P.o_hohi) : nullptr;
  P.tc.b_koff = P.d.b_koff;
  P.tc.b_noff = P.d.b_noff;
}

int execute_pair_plan(const tnc_pair_plan& P, int64_t batch, const void* a, int64_t a_zstride, const void* b,
                      int64_t b_zstride, void* out, int64_t out_zstride, cudaStream_t s) {
  if (batch <= 0) return TNC_OK;
  if (P.tc_ok && (tc_mask() & 1) && pair_use_tc(P.tc.K, P.tc.N)) {
    tnc::TcDesc c = P.tc;
    c.a = reinterpret_cast<const float2*>(a);
    c.a_zstride = a_zstride;
    c.site.ptr = b;
    c.site.zstride = b_zstride;
    c.out = reinterpret_cast<float2*>(out);
    c.out_zstride = out_zstride;
    if (tnc::launch_tc(c, batch, s) != 0) return check_launch("contract_pair[tc]");
    return TNC_OK;
  }
  if (P.kind == TNC_K_SKINNY) {
    tnc::PairTile pt = P.pt;
    pt.a_zstride = a_zstride; pt.b_zstride = b_zstride; pt.out_zstride = out_zstride;
    if (pt.vec16 && ((((uintptr_t)a) % 16) != 0 || (a_zstride % 2) != 0)) pt.vec16 = 0;
    return P.dtype == TNC_C64 ? launch_pair_tiled<float>(pt, batch, a, b, out, s)
                              : launch_pair_tiled<double>(pt, batch, a, b, out, s);
  }
  tnc_step_desc d = P.d;
  d.Z = batch;
  d.acc = a; d.acc_zstride = a_zstride;
  d.out = out; d.out_zstride = out_zstride;
  d.site.ptr = b; d.site.zstride = b_zstride;
  return tnc_step(&d, (void*)s);
}

}  // namespace

extern "C" {

size_t tnc_contract_pair_workspace(int a_rank, const int64_t* a_dims, int b_rank, const int64_t* b_dims,
                                   int npairs, const int32_t* pair_a, const int32_t* pair_b) {
  tnc_pair_plan P;
  if (build_pair_plan(P, TNC_C64, a_rank, a_dims, b_rank, b_dims, npairs, pair_a, pair_b, nullptr, 0) != TNC_OK)
    return 0;
  tnc_pair_plan Q;
  if (build_pair_plan(Q, TNC_C128, a_rank, a_dims, b_rank, b_dims, npairs, pair_a, pair_b, nullptr, 0) != TNC_OK)
    return 0;
  return std::max(P.blob.size(), Q.blob.size()) + 256;
}

int tnc_contract_pair(int dtype, int64_t batch,
                      const void* a, int a_rank, const int64_t* a_dims, int64_t a_zstride,
                      const void* b, int b_rank, const int64_t* b_dims, int64_t b_zstride,
                      int npairs, const int32_t* pair_a, const int32_t* pair_b,
                      const int32_t* out_perm, int conj_b,
                      void* out, int64_t out_zstride,
                      void* workspace, size_t workspace_bytes, void* stream) {
  tnc_pair_plan P;
  int rc = build_pair_plan(P, dtype, a_rank, a_dims, b_rank, b_dims, npairs, pair_a, pair_b, out_perm, conj_b);
  if (rc) return rc;
  if (workspace_bytes < P.blob.size()) return fail(TNC_E_INVALID, "tnc_contract_pair: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemcpyAsync(workspace, P.blob.data(), P.blob.size(), cudaMemcpyHostToDevice, s) != cudaSuccess)
    return check_launch("tnc_contract_pair: table upload");
  bind_tables(P, workspace);
  rc = execute_pair_plan(P, batch, a, a_zstride, b, b_zstride, out, out_zstride, s);
  if (rc) return rc;
  // the host blob must outlive the async upload
  if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("tnc_contract_pair: sync");
  return TNC_OK;
}

int tnc_pair_plan_create(int dtype, int a_rank, const int64_t* a_dims, int b_rank, const int64_t* b_dims,
                         int npairs, const int32_t* pair_a, const int32_t* pair_b,
                         const int32_t* out_perm, int conj_b, tnc_pair_plan** plan) {
  if (!plan) return fail(TNC_E_INVALID, "tnc_pair_plan_create: null plan pointer");
  *plan = nullptr;
  tnc_pair_plan* P = new tnc_pair_plan();
  int rc = build_pair_plan(*P, dtype, a_rank, a_dims, b_rank, b_dims, npairs, pair_a, pair_b, out_perm, conj_b);
  if (rc) { delete P; return rc; }
  if (cudaMalloc(&P->dmem, P->blob.size()) != cudaSuccess) {
    delete P;
    return check_launch("tnc_pair_plan_create: cudaMalloc");
  }
  if (cudaMemcpy(P->dmem, P->blob.data(), P->blob.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(P->dmem);
    delete P;
    return check_launch("tnc_pair_plan_create: upload");
  }
  bind_tables(*P, P->dmem);
  *plan = P;
  return TNC_OK;
}

int tnc_pair_plan_execute(const tnc_pair_plan* plan, int64_t batch, const void* a, int64_t a_zstride,
                          const void* b, int64_t b_zstride, void* out, int64_t out_zstride, void* stream) {
  if (!plan) return fail(TNC_E_INVALID, "tnc_pair_plan_execute: null plan");
  return execute_pair_plan(*plan, batch, a, a_zstride, b, b_zstride, out, out_zstride, (cudaStream_t)stream);
}

int tnc_pair_plan_kernel(const tnc_pair_plan* plan) {
  if (!plan) return TNC_E_INVALID;
  if (plan->tc_ok && (tc_mask() & 1) && pair_use_tc(plan->tc.K, plan->tc.N)) return TNC_K_TC;
  return plan->kind;
}

void tnc_pair_plan_destroy(tnc_pair_plan* plan) {
  if (!plan) return;
  if (plan->dmem) cudaFree(plan->dmem);
  delete plan;
}

}  // extern "C"
