// Micro-benchmark: MUFU.EX2 throughput per SM with full warps vs partially active warps, and the
// packed ex2.approx.f16x2 variant.  Decides how to spread softmax work over SM sub-partitions.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

template <int ACTIVE, int MODE>
__global__ void k(float* out, int iters) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 0.1f, x2 = x0 + 0.2f, x3 = x0 + 0.3f;
  unsigned h0 = 0x3c003c00u + threadIdx.x, h1 = h0 ^ 0x1, h2 = h0 ^ 0x2, h3 = h0 ^ 0x3;
  if ((threadIdx.x & 31) < ACTIVE) {
    for (int i = 0; i < iters; ++i) {
      if (MODE == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x2)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x3));
      } else {
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h0)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h1));
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h2)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h3));
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + __uint_as_float(h0 ^ h1 ^ h2 ^ h3);
}

template <int A, int M>
void run(const char* name, int warps) {
  float* o; cudaMalloc(&o, 148 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  k<A, M><<<148, warps * 32>>>(o, 10);
  cudaEventRecord(e0);
  k<A, M><<<148, warps * 32>>>(o, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double instr = 4.0 * iters * warps * 148;   // warp-instructions
  printf("%-28s warps/SM=%2d: %.2f warp-instr/clk/SM @1.9GHz  (%.3f ms)\n", name, warps, instr / (ms * 1e-3) / 1.9e9 / 148, ms);
  cudaFree(o);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<32, 0>("ex2.f32 32 lanes", w);
    run<8, 0>("ex2.f32 8 lanes", w);
    run<16, 0>("ex2.f32 16 lanes", w);
    run<32, 1>("ex2.f16x2 32 lanes", w);
  }
  return 0;
}
