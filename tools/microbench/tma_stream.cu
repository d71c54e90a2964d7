// Micro-benchmark: HBM read bandwidth of a TMA ring (one CTA per SM, one producer thread, one
// consumer warp that immediately releases stages), with the split kernel's box shape
// (64 rows x 128 B, 128B swizzle) over a [rows, 128] bf16 tensor.  Varies stage count / size.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok) asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(smem_u32(b)), "r"(par));
}

template <int STAGES, int BOXES_PER_STAGE>
__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap tm, int rows_total, int iters_per_cta) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * BOXES_PER_STAGE * 8192);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  __syncthreads();
  // each CTA streams a contiguous chunk of 64-row blocks
  const int blocks_total = rows_total / 64;
  const int per = blocks_total / gridDim.x;
  const int b0 = blockIdx.x * per;
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters_per_cta; ++i) {
      const int s = i % STAGES;
      wait(empty + s, ((i / STAGES) & 1) ^ 1);
      asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(smem_u32(full + s)), "r"(BOXES_PER_STAGE * 8192));
      for (int b = 0; b < BOXES_PER_STAGE; ++b) {
        const int blk = b0 + (i * BOXES_PER_STAGE / 2 + b / 2) % per;
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                     ::"r"(smem_u32(sm + (s * BOXES_PER_STAGE + b) * 8192)), "l"((uint64_t)&tm), "r"((b & 1) * 64), "r"(blk * 64), "r"(smem_u32(full + s)) : "memory");
      }
    }
  } else if (threadIdx.x == 32) {
    for (int i = 0; i < iters_per_cta; ++i) {
      const int s = i % STAGES;
      wait(full + s, (i / STAGES) & 1);
      asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(empty + s)));
    }
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int S, int B>
void run(CUtensorMap& tm, int rows, EncFn) {
  int smem = S * B * 8192 + 1024;
  cudaFuncSetAttribute(stream<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int iters = 2000 / B * 2;
  stream<S, B><<<148, 64, smem>>>(tm, rows, 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  stream<S, B><<<148, 64, smem>>>(tm, rows, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double bytes = 148.0 * iters * B * 8192;
  printf("stages=%d stage_KB=%3d in_flight_KB=%4d: %.0f GB/s (%s)\n", S, B * 8, S * B * 8, bytes / ms / 1e6,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int rows = 16 * 1024 * 1024;   // 4 GiB of [rows, 128] bf16
  void* p; cudaMalloc(&p, (size_t)rows * 256);
  cudaMemset(p, 0, (size_t)rows * 256);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncFn enc = (EncFn)fn;
  CUtensorMap tm;
  cuuint64_t dims[2] = {128, (cuuint64_t)rows}; cuuint64_t str[1] = {256};
  cuuint32_t box[2] = {64, 64}; cuuint32_t es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  run<2, 4>(tm, rows, enc);
  run<3, 4>(tm, rows, enc);
  run<4, 4>(tm, rows, enc);
  run<6, 4>(tm, rows, enc);
  run<2, 8>(tm, rows, enc);
  run<3, 8>(tm, rows, enc);
  run<5, 4>(tm, rows, enc);
  run<8, 2>(tm, rows, enc);
  run<12, 2>(tm, rows, enc);
  run<24, 1>(tm, rows, enc);
  return 0;
}
