// Micro-benchmark: HBM read bandwidth of a TMA ring (one CTA per SM, one producer thread, one
// consumer warp that releases stages at once) for the split kernel's access pattern: 32 KB
// stages = 2 x (64 rows x 128 B, SW128) boxes x 2 column halves, i.e. two 16 KB (page, kv head)
// blocks of a [rows, 128] bf16 tensor; blocks visited sequentially or in a random permutation,
// from one tensor or alternating between two (K and V).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok) asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(smem_u32(b)), "r"(par));
}

__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                                                const int* __restrict__ order, int per_cta, int stages, int two) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * 32768);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  __syncthreads();
  const int* ord = order + (size_t)blockIdx.x * per_cta;
  const int iters = per_cta / 2;               // two 16 KB blocks per stage
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % stages;
      wait(empty + s, ((i / stages) & 1) ^ 1);
      asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(smem_u32(full + s)), "r"(32768));
      const CUtensorMap* m = (two == 1 && (i & 1)) ? &tb : &ta;
      for (int b = 0; b < 4; ++b) {
        // two == 2: one 32 KB run (two consecutive 64-row blocks) per stage, e.g. K and V of one
        // (page, kv head) interleaved; otherwise two independent 16 KB blocks
        const int blk = two == 2 ? (ord[2 * i] & ~1) + (b >> 1) : ord[2 * i + (b >> 1)];
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                     ::"r"(smem_u32(sm + s * 32768 + b * 8192)), "l"((uint64_t)m), "r"((b & 1) * 64), "r"(blk * 64), "r"(smem_u32(full + s)) : "memory");
      }
    }
  } else if (threadIdx.x == 32) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % stages;
      wait(full + s, (i / stages) & 1);
      asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(empty + s)));
    }
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  // argv[1] = working set in 16 KB blocks (0: the whole 2 GiB per tensor; e.g. 2048 = 32 MB, L2-resident)
  const int ws = argc > 1 ? atoi(argv[1]) : 0;
  const int rows = 8 * 1024 * 1024;   // 2 GiB per tensor of [rows, 128] bf16
  const int blocks = rows / 64;       // 16 KB blocks
  void *pa, *pb;
  cudaMalloc(&pa, (size_t)rows * 256); cudaMalloc(&pb, (size_t)rows * 256);
  cudaMemset(pa, 1, (size_t)rows * 256); cudaMemset(pb, 2, (size_t)rows * 256);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncFn enc = (EncFn)fn;
  CUtensorMap ta, tb;
  cuuint64_t dims[2] = {128, (cuuint64_t)rows}; cuuint64_t str[1] = {256};
  cuuint32_t box[2] = {64, 64}; cuuint32_t es[2] = {1, 1};
  enc(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, pa, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, pb, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int per_cta = (blocks / 148) & ~1;
  std::vector<int> seq(148 * per_cta), rnd(148 * per_cta);
  for (int i = 0; i < 148 * per_cta; ++i) seq[i] = ws ? i % ws : i;
  std::vector<int> perm(blocks);
  for (int i = 0; i < blocks; ++i) perm[i] = i;
  std::shuffle(perm.begin(), perm.end(), std::mt19937(7));
  for (int i = 0; i < 148 * per_cta; ++i) rnd[i] = ws ? perm[i] % ws : perm[i];
  int *dseq, *drnd;
  cudaMalloc(&dseq, seq.size() * 4); cudaMalloc(&drnd, rnd.size() * 4);
  cudaMemcpy(dseq, seq.data(), seq.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(drnd, rnd.data(), rnd.size() * 4, cudaMemcpyHostToDevice);
  for (int stages : {2, 3, 4, 5, 6}) {
    const int smem = stages * 32768 + 1024;
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int two = 0; two < 3; ++two)
      for (int r = 0; r < 2; ++r) {
        const int* o = r ? drnd : dseq;
        stream<<<148, 64, smem>>>(ta, tb, o, 64, stages, two);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        stream<<<148, 64, smem>>>(ta, tb, o, per_cta, stages, two);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = 148.0 * per_cta * 16384;
        printf("stages=%d (%3d KB in flight) %s %s: %.0f GB/s (%s)\n", stages, stages * 32, r ? "random" : "seq   ",
               two == 2 ? "32 KB runs      " : two ? "K/V alternating" : "one tensor     ", bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
      }
  }
  return 0;
}
