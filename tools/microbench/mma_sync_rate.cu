// Micro-benchmark: legacy mma.sync m16n8k16 bf16->fp32 throughput on sm_100a.
// Decides whether the shared-page attention tiles can stay on mma.sync (SURVEY §7 hard part 2).
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

template <int NACC>
__global__ void mma_loop(float* out, int iters) {
  unsigned a0 = threadIdx.x * 3u + 1u, a1 = a0 ^ 0x5555u, a2 = a0 + 7u, a3 = a0 * 5u;
  unsigned b0 = threadIdx.x + 11u, b1 = b0 * 3u;
  float acc[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
          : "+f"(acc[i][0]), "+f"(acc[i][1]), "+f"(acc[i][2]), "+f"(acc[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps : {4, 8, 16}) for (int bps : {1, 2, 4}) {
    int threads = warps * 32, blocks = sms * bps;
    mma_loop<8><<<blocks, threads>>>(out, 64);
    cudaEventRecord(e0);
    mma_loop<8><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 16 * 8.0 * iters * (double)blocks * warps;
    printf("mma.sync bf16 m16n8k16: warps/blk=%d blk/SM=%d -> %.1f TFLOP/s (%.3f ms)\n", warps, bps, flops / ms / 1e9, ms);
  }
  cudaError_t err = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
