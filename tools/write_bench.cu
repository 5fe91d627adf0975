// Microbenchmark: HBM write bandwidth by store mechanism and warps per SM.
// One CTA per SM (148), WARPS warps each streaming 4 KB blocks of a 4 GiB
// buffer: (0) STG.128 from registers, (1) cp.async.bulk smem -> global with
// DEPTH 4 KB bulk stores in flight per warp.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 tools/write_bench.cu -o tools/_write_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE, int DEPTH>
__global__ void k_write(float4* out, size_t nblk) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  unsigned char* buf = sm + (size_t)warp * DEPTH * 4096;
  for (int i = threadIdx.x; i < wpb * DEPTH * 256; i += blockDim.x) reinterpret_cast<float4*>(sm)[i] = make_float4(1.f, 2.f, 3.f, 4.f);
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  size_t b = (size_t)blockIdx.x * wpb + warp;
  const size_t stride = (size_t)gridDim.x * wpb;
  int k = 0;
  for (; b < nblk; b += stride, ++k) {
    float4* dst = out + b * 256;                  // 4 KB block = 256 float4
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dst[i * 32 + lane] = make_float4(b, i, lane, 0.f);
    } else if (MODE == 2 || MODE == 3) {
      // result layout [n][f] (f extent F = 2^22, complex64): block = 32 f x 16 n,
      // f fastest across blocks; MODE 2: STG.64 per lane (lane = f), MODE 3: STG.128 (2 f per lane, 8 n per instr)
      const size_t F = 1ull << 22;
      const size_t fb = b % (F / 32), nb = b / (F / 32);
      float2* o2 = reinterpret_cast<float2*>(out);
      if (MODE == 2) {
#pragma unroll
        for (int c = 0; c < 16; ++c) o2[(nb * 16 + c) * F + fb * 32 + lane] = make_float2(c, lane);
      } else {
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
          const int cc = c + (lane >> 4);
          reinterpret_cast<float4*>(o2 + (nb * 16 + cc) * F + fb * 32)[lane & 15] = make_float4(c, lane, 0.f, 1.f);
        }
      }
    } else if (lane == 0) {
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(DEPTH - 1) : "memory");
      const uint32_t src = (uint32_t)__cvta_generic_to_shared(buf + (k % DEPTH) * 4096);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;" ::"l"(dst), "r"(src) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (MODE == 1 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int MODE, int DEPTH>
void run(const char* name, int warps, float4* out, size_t nblk) {
  const size_t smem = (size_t)warps * DEPTH * 4096;
  cudaFuncSetAttribute(k_write<MODE, DEPTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_write<MODE, DEPTH><<<148, warps * 32, smem>>>(out, nblk);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k_write<MODE, DEPTH><<<148, warps * 32, smem>>>(out, nblk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const cudaError_t err = cudaGetLastError();
  printf("%-26s warps/SM=%2d depth=%d: %7.1f GB/s %s\n", name, warps, DEPTH, 5.0 * nblk * 4096 / (ms * 1e-3) / 1e9,
         err == cudaSuccess ? "" : cudaGetErrorString(err));
}

int main() {
  const size_t bytes = 4ull << 30, nblk = bytes / 4096;
  float4* out;
  cudaMalloc(&out, bytes);
  run<2, 1>("[n][f] STG.64 lanes=f", 8, out, nblk);
  run<3, 1>("[n][f] STG.128", 8, out, nblk);
  run<2, 1>("[n][f] STG.64 lanes=f", 16, out, nblk);
  run<0, 1>("STG.128", 4, out, nblk);
  run<0, 1>("STG.128", 8, out, nblk);
  run<0, 1>("STG.128", 16, out, nblk);
  run<0, 1>("STG.128", 32, out, nblk);
  run<1, 2>("bulk 4KB", 4, out, nblk);
  run<1, 2>("bulk 4KB", 8, out, nblk);
  run<1, 4>("bulk 4KB", 8, out, nblk);
  run<1, 4>("bulk 4KB", 4, out, nblk);
  run<1, 6>("bulk 4KB", 8, out, nblk);
  return 0;
}
