// Micro-benchmark: tcgen05.mma issue->completion latency and throughput for the split kernel's
// shapes (M=128; QK: SS N=64; PV: TS N=128; l: TS N=16), bf16 -> fp32, one CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int m, int n, bool bmn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((bmn ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(b)));
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok) asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(smem_u32(b)), "r"(par));
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) k(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;\n"); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  uint32_t tm = tslot;
  uint32_t base = smem_u32(sm);
  unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    uint64_t dq = sw128_desc(base, 16, 1024), dk = sw128_desc(base + 32768, 16, 1024), dv = sw128_desc(base + 65536, 8192, 1024);
    for (int i = 0; i < iters; ++i) {
      if (MODE == 0 || MODE == 2) {
        for (int ks = 0; ks < 8; ++ks) mma_ss(tm + (i & 1) * 64, dq + ((ks >> 2) * 16384 + (ks & 3) * 32) / 16, dk + ((ks >> 2) * 8192 + (ks & 3) * 32) / 16, idesc(128, 64, false), ks > 0);
      }
      if (MODE == 1 || MODE == 2) {
        for (int kt = 0; kt < 4; ++kt) {
          mma_ts(tm + 256, tm + 128 + kt * 8, dv + (kt * 2048) / 16, idesc(128, 128, true), 1);
          mma_ts(tm + 192, tm + 128 + kt * 8, dq + (kt * 32) / 16, idesc(128, 16, false), 1);
        }
      }
      if (MODE == 3) {  // latency: commit and wait each iteration (QK only)
        for (int ks = 0; ks < 8; ++ks) mma_ss(tm, dq + ((ks >> 2) * 16384 + (ks & 3) * 32) / 16, dk + ((ks >> 2) * 8192 + (ks & 3) * 32) / 16, idesc(128, 64, false), ks > 0);
        commit(&bar);
        wait(&bar, i & 1);
      }
    }
    if (MODE != 3) { commit(&bar); wait(&bar, 0); }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm));
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 148);
  const char* names[] = {"QK 8x(128x64x16) SS", "PV 4x(128x128x16)+4x(128x16x16) TS", "QK+PV per tile", "QK + commit/wait latency"};
  for (int mode = 0; mode < 4; ++mode) {
    auto f = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : k<3>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    int iters = 2000;
    f<<<148, 128, 100000>>>(d, 10);
    f<<<148, 128, 100000>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("%-40s: %.1f cycles per iteration (%s)\n", names[mode], (double)h[0] / iters, cudaGetErrorString(e));
  }
  return 0;
}
