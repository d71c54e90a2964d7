// Issue-rate microbenchmark of the softmax's instruction kinds on one SM: MUFU.EX2, F2FP bf16x2
// pack, the mixed-precision add (add.rn.f32.bf16), FFMA, FMNMX3.  W warps per CTA (W/4 per SM
// sub-partition), 8 independent chains per thread, cycles per warp-instruction per SMSP.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

template <int KIND>
__global__ void bench(float* out, long long* cyc, int iters) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = -0.001f * (threadIdx.x + i);
  uint32_t u[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) u[i] = 0x3f803f80u + i;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
      if (KIND == 1) {
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v[i]), "f"(v[(i + 1) & 7]));
        v[i] = __uint_as_float(r ^ u[i]);
      }
      if (KIND == 2) asm volatile("add.rn.f32.bf16 %0, %1, %0;" : "+f"(v[i]) : "h"((unsigned short)(u[i] & 0xffff)));
      if (KIND == 3) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3A83126F;" : "+f"(v[i]));
      if (KIND == 4) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(v[(i + 3) & 7]), "f"(v[(i + 5) & 7]));
      if (KIND == 5) {   // 2 ex2 + 1 bf16x2 pack: shares a pipe if the cost is the sum
        float a = v[i], b = v[(i + 4) & 7];
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b));
        v[i] = __uint_as_float(r ^ u[i]);
      }
      if (KIND == 6) {   // integer round-to-nearest-even bf16x2 pack
        const uint32_t a = __float_as_uint(v[i]), b = __float_as_uint(v[(i + 1) & 7]);
        const uint32_t ra = a + 0x7fffu + ((a >> 16) & 1u), rb = b + 0x7fffu + ((b >> 16) & 1u);
        uint32_t r;
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(ra), "r"(rb));
        v[i] = __uint_as_float(r ^ u[i]);
      }
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int KIND>
void run(const char* name, int warps) {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  bench<KIND><<<148, warps * 32>>>(out, cyc, iters);
  bench<KIND><<<148, warps * 32>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double instr_per_smsp = (double)iters * 8 * warps / 4;
  printf("%-10s warps/SM %2d: %.2f cycles per warp-instr per SMSP (%.1f lanes/clk/SM)\n", name, warps,
         c / instr_per_smsp, 32.0 * 4 / (c / instr_per_smsp));
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("ex2", w); run<1>("f2fp.bf16", w); run<2>("add.f32.bf16", w); run<3>("ffma", w); run<4>("max3", w);
    run<5>("2ex2+f2fp", w); run<6>("int-rn-pack", w);
  }
  return 0;
}
