// Microbenchmark: issue rate of tcgen05.mma variants (one CTA per SM, one
// thread issuing NITER MMAs into one TMEM accumulator).  Prints cycles/MMA
// and the implied per-SM MAC rate.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
//   -std=c++17 -I paper_2011_02621_b200/csrc -I include tools/mma_bench.cu -o tools/_mma_bench
#include <cstdio>
#include "tnc_tc.cuh"
using namespace tnc;

__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int MODE, int N>
__global__ void __launch_bounds__(128, 1) k_bench(int niter, unsigned long long* out) {
  // MODE 0: tf32 A in TMEM; 1: tf32 A in smem; 2: bf16 A in TMEM; 3: tf32 ts, 2 accumulators alternating
  __shared__ __align__(1024) unsigned char sm[40 * 1024];
  __shared__ uint64_t bar, bar2[4];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 40 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int q = 0; q < 4; ++q) mbar_init(&bar2[q], 1); mbar_fence_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    uint32_t idesc;
    if (MODE == 2 || MODE == 7) idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    else idesc = tf32_idesc(N);
    const uint32_t b0 = smem_u32(sm);
    const uint64_t bd = umma_desc(b0, 128, 512);
    const uint64_t ad = umma_desc(b0 + 32768, 128, 512);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < niter; ++i) {
      const uint32_t acc = i == 0 ? 0u : 1u;
      if (MODE == 0) mma_tf32_ts(tmem, tmem + 256, bd, idesc, acc);
      else if (MODE == 1) mma_tf32(tmem, ad, bd, idesc, acc);
      else if (MODE == 2) mma_f16_ts(tmem, tmem + 256, bd, idesc, acc);
      else if (MODE == 7) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
      else if (MODE == 3) mma_tf32_ts(tmem + (i & 1) * N, tmem + 256 + 8 * (i & 3), bd, idesc, i < 2 ? 0u : 1u);
      else if (MODE >= 4 && MODE <= 6) {
        // chunk-shaped: 12 MMAs per group of 12 iterations, commit(s) every 12
        mma_tf32_ts(tmem + ((i >> 1) & 1) * N, tmem + 256 + 8 * (i & 7), bd + ((i & 3) * 64), idesc, i < 4 ? 0u : 1u);
        if (MODE == 5 && (i % 12) == 11) { umma_commit(&bar2[0]); umma_commit(&bar2[1]); }
        if (MODE == 6 && (i % 24) == 23) { umma_commit(&bar2[0]); umma_commit(&bar2[1]); }
      }
      if (MODE == 8 && (i % 12) == 11) {     // chunk round trip: 12 MMAs, commit, wait
        mma_tf32_ts(tmem, tmem + 256, bd, idesc, 1u);
        umma_commit(&bar2[2]);
        mbar_wait_spin(&bar2[2], (uint32_t)((i / 12) & 1));
      } else if (MODE == 8) mma_tf32_ts(tmem, tmem + 256, bd, idesc, acc);
      if (MODE == 10) {                       // single-MMA round trip: mma, commit, wait
        mma_tf32_ts(tmem, tmem + 256, bd, idesc, acc);
        umma_commit(&bar2[2]);
        mbar_wait_spin(&bar2[2], (uint32_t)(i & 1));
      }
      if (MODE == 9) mma_tf32_ts(tmem + (i & 3) * 32, tmem + 256, bd, idesc, i < 4 ? 0u : 1u);   // 4 independent accumulators
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// MMA chain (thread 0, N columns, A in TMEM) while warps 4-7 stream tcgen05.st
// (ST=1) or tcgen05.ld (ST=2) into their own TMEM columns: does TMEM traffic
// from other warps slow the MMA issue?
template <int ST, int N>
__global__ void __launch_bounds__(256, 1) k_contend(int niter, unsigned long long* out) {
  __shared__ __align__(1024) unsigned char sm[40 * 1024];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 40 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_fence_init(); stop = 0; }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = tf32_idesc(N);
    const uint64_t bd = umma_desc(smem_u32(sm), 128, 512);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < niter; ++i) mma_tf32_ts(tmem, tmem + 256, bd, idesc, i == 0 ? 0u : 1u);
    umma_commit(&bar);
    mbar_wait_spin(&bar, 0);
    const unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    stop = 1;
  } else if (warp >= 4 && ST) {
    const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t v[16];
    for (int q = 0; q < 16; ++q) v[q] = threadIdx.x * q;
    int it = 0;
    while (!stop) {
      const uint32_t col = 320 + (uint32_t)((it & 7) * 16);
      if (ST == 1) { tmem_st<16>(tmem + lb + col, v); tmem_wait_st(); }
      else { tmem_ld16(tmem + lb + col, v); tmem_wait_ld(); v[0] += 1; }
      ++it;
    }
    if (v[0] == 12345) out[0] = 0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int ST, int N>
void run_contend(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int niter = 4096;
  k_contend<ST, N><<<148, 256>>>(niter, d);
  k_contend<ST, N><<<148, 256>>>(niter, d);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  printf("%-28s N=%3d: %7.1f cycles/MMA %s\n", name, N, avg / 148 / niter, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

template <int MODE, int N>
void run(const char* name, int K) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int niter = 4096;
  k_bench<MODE, N><<<148, 128>>>(niter, d);
  k_bench<MODE, N><<<148, 128>>>(niter, d);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double cyc = avg / niter;
  printf("%-28s N=%3d: %7.1f cycles/MMA  %7.0f MAC/cycle/SM  %s\n", name, N, cyc, 128.0 * N * K / cyc,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0, 64>("tf32 ts", 8);
  run<0, 128>("tf32 ts", 8);
  run<0, 256>("tf32 ts", 8);
  run<1, 64>("tf32 ss", 8);
  run<1, 128>("tf32 ss", 8);
  run<1, 256>("tf32 ss", 8);
  run<2, 64>("bf16 ts", 16);
  run<2, 128>("bf16 ts", 16);
  run<2, 256>("bf16 ts", 16);
  run<7, 64>("bf16 ss", 16);
  run<7, 128>("bf16 ss", 16);
  run<7, 256>("bf16 ss", 16);
  run<3, 64>("tf32 ts 2acc", 8);
  run<3, 128>("tf32 ts 2acc", 8);
  run<4, 64>("tf32 ts chunk nocommit", 8);
  run<5, 64>("tf32 ts commit/12", 8);
  run<6, 64>("tf32 ts commit/24", 8);
  run<5, 128>("tf32 ts commit/12", 8);
  run<0, 16>("tf32 ts", 8);
  run<0, 32>("tf32 ts", 8);
  run<9, 16>("tf32 ts 4acc", 8);
  run<9, 32>("tf32 ts 4acc", 8);
  run<2, 16>("bf16 ts", 16);
  run<2, 32>("bf16 ts", 16);
  run<8, 16>("tf32 ts chunk+wait/12", 8);
  run<8, 64>("tf32 ts chunk+wait/12", 8);
  run_contend<0, 16>("tf32 ts, idle warps");
  run_contend<1, 16>("tf32 ts, 4 warps tcgen05.st");
  run_contend<2, 16>("tf32 ts, 4 warps tcgen05.ld");
  run_contend<1, 64>("tf32 ts, 4 warps tcgen05.st");
  run<10, 16>("tf32 ts 1 mma+commit+wait", 8);
  run<10, 128>("tf32 ts 1 mma+commit+wait", 8);
  return 0;
}
