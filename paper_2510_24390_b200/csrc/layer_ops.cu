// layer_ops.cu — the non-GEMM steps of a decoder layer around the expansion attention
// (oracle O7, oracle/decoder.py): fused residual add + RMSNorm, RoPE fused
// into the KV append, SiLU(gate) * up.  All HBM-bound row / element operations: 128-bit accesses,
// fp32 arithmetic, bf16 storage (reading M1).  GEMMs are plain library calls (cuBLAS) made by the
// caller.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>

#include "../../include/orion.h"
#include "nvtx_range.h"
#include "split_tc.h"

namespace orion {
namespace {

__device__ __forceinline__ float2 bf2_to_f2(uint32_t v) {
  return make_float2(__uint_as_float(v << 16), __uint_as_float(v & 0xFFFF0000u));
}
__device__ __forceinline__ uint32_t f2_to_bf2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float bf16_round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// One block per row.  r = bf16(a + b) (b nullable: r = a), residual_out = r (nullable),
// out = bf16(r * rsqrt(mean(r^2) + eps) * w) (nullable).
__global__ void __launch_bounds__(256) rmsnorm_kernel(const __nv_bfloat16* __restrict__ a,
                                                      const __nv_bfloat16* __restrict__ b,
                                                      const __nv_bfloat16* __restrict__ w,
                                                      __nv_bfloat16* __restrict__ out,
                                                      __nv_bfloat16* __restrict__ residual_out,
                                                      int hidden, float eps) {
  pdl_trigger();
  pdl_wait();
  const size_t row = blockIdx.x;
  const int n8 = hidden / 8;
  const uint4* a8 = reinterpret_cast<const uint4*>(a + row * hidden);
  const uint4* b8 = b ? reinterpret_cast<const uint4*>(b + row * hidden) : nullptr;
  extern __shared__ float red_smem[];
  constexpr int kMax = 4;                            // up to 4 x 8 elements per thread (hidden <= 8192)
  uint4 rv[kMax];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < kMax; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
    if (c < n8) {
      uint4 x = __ldg(a8 + c);
      if (b8) {
        const uint4 y = __ldg(b8 + c);
        uint32_t* xs = reinterpret_cast<uint32_t*>(&x);
        const uint32_t* ys = reinterpret_cast<const uint32_t*>(&y);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 p = bf2_to_f2(xs[j]), q = bf2_to_f2(ys[j]);
          xs[j] = f2_to_bf2(p.x + q.x, p.y + q.y);
        }
      }
      rv[i] = x;
      const uint32_t* xs = reinterpret_cast<const uint32_t*>(&x);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 p = bf2_to_f2(xs[j]);
        ss = fmaf(p.x, p.x, fmaf(p.y, p.y, ss));
      }
      if (residual_out) reinterpret_cast<uint4*>(residual_out + row * hidden)[c] = x;
    }
  }
  if (!out) return;
#pragma unroll
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red_smem[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red_smem[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red_smem[32] = rsqrtf(v / hidden + eps);
  }
  __syncthreads();
  const float inv = red_smem[32];
  const uint4* w8 = reinterpret_cast<const uint4*>(w);
#pragma unroll
  for (int i = 0; i < kMax; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
    if (c < n8) {
      const uint4 wv = __ldg(w8 + c);
      const uint32_t* xs = reinterpret_cast<const uint32_t*>(&rv[i]);
      const uint32_t* ws = reinterpret_cast<const uint32_t*>(&wv);
      uint4 o4;
      uint32_t* os = reinterpret_cast<uint32_t*>(&o4);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 p = bf2_to_f2(xs[j]), q = bf2_to_f2(ws[j]);
        os[j] = f2_to_bf2(p.x * inv * q.x, p.y * inv * q.y);
      }
      reinterpret_cast<uint4*>(out + row * hidden)[c] = o4;
    }
  }
}

// One block per branch.  qkv row = [q (hq d) | k (hkv d) | v (hkv d)]; token position
// pos = pos_base[b] + slot, slot = own_len (ADVANCE) or own_len - 1 (REWRITE).  q and k are rotated
// (rotate_half convention, inv_freq_i = theta^(-2i/d)), q written to q_out [b][hq][d], k and v
// written to the slot of b's own run in the paged caches; ADVANCE then increments own_len.
template <int D>
__global__ void __launch_bounds__(128) rope_append_kernel(
    const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ q_out,
    __nv_bfloat16* __restrict__ k_cache, __nv_bfloat16* __restrict__ v_cache,
    const int32_t* __restrict__ own_pt_off, const int32_t* __restrict__ own_cap,
    const int32_t* __restrict__ page_table, int32_t* __restrict__ own_len,
    const int32_t* __restrict__ pos_base, int hq, int hkv, int page_shift, int kvs, int mode,
    float log2_theta, int num_pages, int* err) {
  constexpr int HALF = D / 2;
  __shared__ int s_slot, s_page, s_len;
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x;
  if (threadIdx.x == 0) {
    const int len = own_len[b];
    const int slot = mode == ORION_APPEND_REWRITE ? len - 1 : len;
    const bool ok = slot >= 0 && slot < own_cap[b];
    s_len = len;
    s_slot = slot;
    int page = ok ? page_table[own_pt_off[b] + (slot >> page_shift)] : -1;
    if (page >= num_pages || (ok && page < 0)) {     // outside the caches: never written
      if (err) atomicCAS(err, 0, b + 1);
      page = -1;
    }
    s_page = page;
  }
  __syncthreads();
  const int slot = s_slot;
  const float pos = static_cast<float>(__ldg(pos_base + b) + slot);
  const __nv_bfloat16* row = qkv + static_cast<size_t>(b) * (hq + 2 * hkv) * D;
  // rotate pairs (i, i + D/2) of every q and k head: (hq + hkv) heads x HALF pairs
  for (int idx = threadIdx.x; idx < (hq + hkv) * HALF; idx += blockDim.x) {
    const int h = idx / HALF, i = idx % HALF;
    const float inv_freq = exp2f(-2.0f * i / D * log2_theta);
    float sn, cs;
    sincosf(pos * inv_freq, &sn, &cs);
    const float x1 = __bfloat162float(row[h * D + i]), x2 = __bfloat162float(row[h * D + i + HALF]);
    const __nv_bfloat16 o1 = __float2bfloat16_rn(x1 * cs - x2 * sn);
    const __nv_bfloat16 o2 = __float2bfloat16_rn(x2 * cs + x1 * sn);
    if (h < hq) {
      q_out[(static_cast<size_t>(b) * hq + h) * D + i] = o1;
      q_out[(static_cast<size_t>(b) * hq + h) * D + i + HALF] = o2;
    } else if (s_page >= 0) {
      const int g = h - hq;
      const size_t dst = ((((static_cast<size_t>(s_page) * hkv + g) * kvs) << page_shift) +
                          (slot & ((1 << page_shift) - 1))) * D;
      k_cache[dst + i] = o1;
      k_cache[dst + i + HALF] = o2;
    }
  }
  if (s_page >= 0) {
    for (int idx = threadIdx.x; idx < hkv * D / 8; idx += blockDim.x) {
      const int g = idx / (D / 8), c = idx % (D / 8);
      const size_t dst = ((((static_cast<size_t>(s_page) * hkv + g) * kvs) << page_shift) +
                          (slot & ((1 << page_shift) - 1))) * D + c * 8;
      *reinterpret_cast<uint4*>(v_cache + dst) =
          *reinterpret_cast<const uint4*>(row + (hq + hkv + g) * D + c * 8);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && mode == ORION_APPEND_ADVANCE && s_page >= 0) own_len[b] = s_len + 1;
}

// a = bf16(SiLU(g) * u) for gu = [g (inter) | u (inter)] per row, SiLU(g) = g / (1 + e^-g).
__global__ void __launch_bounds__(256) silu_mul_kernel(const __nv_bfloat16* __restrict__ gu,
                                                       __nv_bfloat16* __restrict__ out, int rows,
                                                       int inter) {
  pdl_trigger();
  pdl_wait();
  const int n8 = inter / 8;
  const size_t total = static_cast<size_t>(rows) * n8;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = i / n8, c = i % n8;
    const uint4 g = __ldg(reinterpret_cast<const uint4*>(gu + r * 2 * inter) + c);
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(gu + r * 2 * inter + inter) + c);
    const uint32_t* gs = reinterpret_cast<const uint32_t*>(&g);
    const uint32_t* us = reinterpret_cast<const uint32_t*>(&u);
    uint4 o4;
    uint32_t* os = reinterpret_cast<uint32_t*>(&o4);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 gf = bf2_to_f2(gs[j]), uf = bf2_to_f2(us[j]);
      os[j] = f2_to_bf2(gf.x / (1.f + __expf(-gf.x)) * uf.x, gf.y / (1.f + __expf(-gf.y)) * uf.y);
    }
    reinterpret_cast<uint4*>(out + r * inter)[c] = o4;
  }
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace
}  // namespace orion

using namespace orion;

extern "C" orion_status orion_rmsnorm(int32_t n_rows, int32_t hidden, const void* a, const void* b,
                                      const void* weight, float eps, void* out, void* residual_out,
                                      void* stream) {
  const orion::NvtxRange nvtx_range("orion_rmsnorm");
  if (n_rows < 0 || hidden < 8 || hidden % 8 || hidden > 8192)
    return fail(ORION_ERR_UNSUPPORTED, "rmsnorm: hidden %d must be a multiple of 8 in [8, 8192]", hidden);
  if (!a || (out && !weight) || (!out && !residual_out))
    return fail(ORION_ERR_INVALID_ARG, "rmsnorm: null pointer");
  if (!al16(a) || (b && !al16(b)) || (weight && !al16(weight)) || (out && !al16(out)) ||
      (residual_out && !al16(residual_out)))
    return fail(ORION_ERR_INVALID_ARG, "rmsnorm: pointers must be 16-byte aligned");
  if (n_rows == 0) return ORION_OK;
  cudaError_t e = launch_pdl(rmsnorm_kernel, dim3(n_rows), dim3(256), 33 * sizeof(float),
                             static_cast<cudaStream_t>(stream), static_cast<const __nv_bfloat16*>(a),
                             static_cast<const __nv_bfloat16*>(b), static_cast<const __nv_bfloat16*>(weight),
                             static_cast<__nv_bfloat16*>(out), static_cast<__nv_bfloat16*>(residual_out),
                             static_cast<int>(hidden), eps);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ORION_ERR_CUDA, "rmsnorm_kernel: %s", cudaGetErrorString(e));
  return ORION_OK;
}

extern "C" orion_status orion_rope_append(const orion_attn_shape* shape, int32_t n_branches,
                                          const void* qkv, void* q_out, void* k_cache, void* v_cache,
                                          const int32_t* own_pt_off, const int32_t* own_cap,
                                          const int32_t* page_table, int32_t num_pages,
                                          int32_t* own_len, const int32_t* pos_base, float rope_theta,
                                          int32_t mode, void* stream) {
  const orion::NvtxRange nvtx_range("orion_rope_append");
  orion_status st = check_shape_public(shape);
  if (st != ORION_OK) return st;
  if (n_branches < 0) return fail(ORION_ERR_INVALID_ARG, "n_branches < 0");
  if (mode != ORION_APPEND_ADVANCE && mode != ORION_APPEND_REWRITE)
    return fail(ORION_ERR_INVALID_ARG, "bad append mode %d", mode);
  if (!qkv || !q_out || !k_cache || !v_cache || !own_pt_off || !own_cap || !page_table || !own_len ||
      !pos_base)
    return fail(ORION_ERR_INVALID_ARG, "rope_append: null pointer");
  if (!al16(qkv) || !al16(q_out) || !al16(k_cache) || !al16(v_cache))
    return fail(ORION_ERR_INVALID_ARG, "rope_append: pointers must be 16-byte aligned");
  if (!(rope_theta > 1.f)) return fail(ORION_ERR_INVALID_ARG, "rope_theta must be > 1");
  if (num_pages < 1) return fail(ORION_ERR_INVALID_ARG, "rope_append: num_pages < 1");
  if (n_branches == 0) return ORION_OK;
  int shift = 0;
  while ((1 << shift) < shape->page_size) ++shift;
  const float lt = std::log2(rope_theta);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int* err = append_check_begin(s);
  cudaError_t e = launch_pdl(
      shape->head_dim == 128 ? rope_append_kernel<128> : rope_append_kernel<64>, dim3(n_branches), dim3(128), 0, s,
      static_cast<const __nv_bfloat16*>(qkv), static_cast<__nv_bfloat16*>(q_out),
      static_cast<__nv_bfloat16*>(k_cache), static_cast<__nv_bfloat16*>(v_cache), own_pt_off, own_cap,
      page_table, own_len, pos_base, shape->num_q_heads, shape->num_kv_heads, shift,
      1 + shape->kv_interleaved, mode, lt, num_pages, err);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ORION_ERR_CUDA, "rope_append_kernel: %s", cudaGetErrorString(e));
  return append_check_end(s, "rope_append");
}

extern "C" orion_status orion_silu_mul(int32_t n_rows, int32_t inter, const void* gate_up, void* out,
                                       void* stream) {
  const orion::NvtxRange nvtx_range("orion_silu_mul");
  if (n_rows < 0 || inter < 8 || inter % 8) return fail(ORION_ERR_UNSUPPORTED, "silu_mul: inter %d", inter);
  if (!gate_up || !out) return fail(ORION_ERR_INVALID_ARG, "silu_mul: null pointer");
  if (!al16(gate_up) || !al16(out)) return fail(ORION_ERR_INVALID_ARG, "silu_mul: pointers must be 16-byte aligned");
  if (n_rows == 0) return ORION_OK;
  const size_t total = static_cast<size_t>(n_rows) * inter / 8;
  const int grid = static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 16));
  cudaError_t e = launch_pdl(silu_mul_kernel, dim3(grid), dim3(256), 0, static_cast<cudaStream_t>(stream),
                             static_cast<const __nv_bfloat16*>(gate_up), static_cast<__nv_bfloat16*>(out),
                             static_cast<int>(n_rows), static_cast<int>(inter));
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ORION_ERR_CUDA, "silu_mul_kernel: %s", cudaGetErrorString(e));
  return ORION_OK;
}
