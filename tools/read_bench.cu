// Microbenchmark: HBM read bandwidth of cp.async.bulk (TMA 1-D) copies into
// shared memory as a function of segment size, for segments laid out like the
// GEMM path's A boxes (one SEG-byte piece per 2 KB row, rows consecutive).
// One CTA per SM, one producer thread keeping DEPTH 16 KB stages in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 tools/read_bench.cu -o tools/_read_bench
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int SEG>
__global__ void k_read(const unsigned char* in, size_t nstage, size_t row_bytes, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  constexpr int DEPTH = 8, STAGE = 16384, PIECES = STAGE / SEG;
  __shared__ __align__(8) uint64_t bar[DEPTH];
  if (threadIdx.x == 0) {
    for (int i = 0; i < DEPTH; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  // stage s covers PIECES rows x SEG bytes: rows r0 .. r0+PIECES-1, column block cb
  const size_t cols = row_bytes / SEG;
  uint32_t phase[DEPTH] = {0};
  size_t k = 0;
  for (size_t s = blockIdx.x; s < nstage; s += gridDim.x, ++k) {
    const int slot = (int)(k % DEPTH);
    if (k >= DEPTH) {
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                     : "=r"(done) : "r"(su32(&bar[slot])), "r"(phase[slot]));
      phase[slot] ^= 1;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[slot])), "r"(STAGE));
    // tile = row block; column block fastest (like the K chunks of one row tile)
    const size_t cb = s % cols, rb = s / cols;
    for (int p = 0; p < PIECES; ++p) {
      const unsigned char* src = in + (rb * PIECES + p) * row_bytes + cb * SEG;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(sm + slot * STAGE + p * SEG)), "l"(src), "r"(SEG), "r"(su32(&bar[slot])) : "memory");
    }
  }
  for (int slot = 0; slot < DEPTH; ++slot) {
    uint32_t done = 0;
    if ((size_t)slot >= k) continue;
    while (!done)
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                   : "=r"(done) : "r"(su32(&bar[slot])), "r"(phase[slot]));
  }
  sink[blockIdx.x] = sm[0];
}

template <int SEG>
void run(const unsigned char* in, size_t bytes, size_t row_bytes, unsigned long long* sink) {
  const size_t nstage = bytes / 16384;
  cudaFuncSetAttribute(k_read<SEG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_read<SEG><<<148, 32, 8 * 16384>>>(in, nstage, row_bytes, sink);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k_read<SEG><<<148, 32, 8 * 16384>>>(in, nstage, row_bytes, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const cudaError_t err = cudaGetLastError();
  printf("segment %5d B, row %5zu B: %7.1f GB/s %s\n", SEG, row_bytes, 5.0 * bytes / (ms * 1e-3) / 1e9,
         err == cudaSuccess ? "" : cudaGetErrorString(err));
}

// TMA tensor loads: 2-D box [32 floats x 128 rows] (128B swizzle) from a
// [rows][row_floats] fp32 tensor, box column fastest (the GEMM path's A chunks)
__global__ void k_read_tma(const __grid_constant__ CUtensorMap tm, size_t nbox, int colboxes, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  constexpr int DEPTH = 8, STAGE = 16384;
  __shared__ __align__(8) uint64_t bar[DEPTH];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  if (threadIdx.x == 0) {
    for (int i = 0; i < DEPTH; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t phase[DEPTH] = {0};
  size_t k = 0;
  for (size_t s = blockIdx.x; s < nbox; s += gridDim.x, ++k) {
    const int slot = (int)(k % DEPTH);
    if (k >= DEPTH) {
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                     : "=r"(done) : "r"(su32(&bar[slot])), "r"(phase[slot]));
      phase[slot] ^= 1;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[slot])), "r"(STAGE));
    const int cb = (int)(s % colboxes), rb = (int)(s / colboxes);
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su32(base + slot * STAGE)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(cb * 32), "r"(rb * 128),
                   "r"(su32(&bar[slot])) : "memory");
  }
  for (int slot = 0; slot < DEPTH; ++slot) {
    uint32_t done = 0;
    if ((size_t)slot >= k) continue;
    while (!done)
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                   : "=r"(done) : "r"(su32(&bar[slot])), "r"(phase[slot]));
  }
  sink[blockIdx.x] = base[0];
}

typedef CUresult (*enc_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                           const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

void run_tma(unsigned char* in, size_t bytes, size_t row_floats, unsigned long long* sink, CUtensorMapL2promotion prom) {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  enc_fn enc = reinterpret_cast<enc_fn>(f);
  const size_t rows = bytes / (row_floats * 4);
  CUtensorMap tm;
  const cuuint64_t gdim[2] = {row_floats, rows};
  const cuuint64_t gstr[1] = {row_floats * 4};
  const cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, in, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode failed\n"); return; }
  const int colboxes = (int)(row_floats / 32);
  const size_t nbox = (rows / 128) * colboxes;
  cudaFuncSetAttribute(k_read_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384 + 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_read_tma<<<148, 32, 8 * 16384 + 1024>>>(tm, nbox, colboxes, sink);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k_read_tma<<<148, 32, 8 * 16384 + 1024>>>(tm, nbox, colboxes, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const cudaError_t err = cudaGetLastError();
  printf("TMA box 128B x 128 rows, row %5zu B, promo %d: %7.1f GB/s %s\n", row_floats * 4, (int)prom,
         5.0 * nbox * 16384 / (ms * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
}

int main() {
  const size_t bytes = 4ull << 30;
  unsigned char* in;
  unsigned long long* sink;
  cudaMalloc(&in, bytes);
  cudaMalloc(&sink, 148 * 8);
  cudaMemset(in, 1, bytes);
  run<128>(in, bytes, 2048, sink);
  run<256>(in, bytes, 2048, sink);
  run<512>(in, bytes, 2048, sink);
  run<2048>(in, bytes, 2048, sink);
  run<128>(in, bytes, 1024, sink);
  run<128>(in, bytes, 128, sink);
  run<16384>(in, bytes, 16384, sink);
  for (size_t rf : {32ul, 128ul, 256ul, 512ul}) {
    run_tma(in, bytes, rf, sink, CU_TENSOR_MAP_L2_PROMOTION_NONE);
    run_tma(in, bytes, rf, sink, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  }
  return 0;
}
