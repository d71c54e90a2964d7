// merge16.h — the LSE merge of one output row's fp16 partials (K3), shared by the combine kernel
// (kernels.cu) and the split kernels if the merge is ever fused into them.
// Product-side only.
//
// A row's partials i (plan_format.h fp16 format: o_i = acc_i / l_i, lse2_i = m_i + log2 l_i) are
// listed in plan order by the combine CSR (comb_off / comb_slot):
//   out = sum_i 2^(lse2_i - M) o_i / sum_i 2^(lse2_i - M),  lse = (M + log2 sum) ln 2,  M = max lse2_i.
// One row per group of kMergeLanes consecutive lanes (16 at D = 128, 8 at D = 64: one 16-B load per
// lane and partial); every lane of the warp calls it (the shuffles use the full mask; a group
// without a row passes valid = false).  Lane `sub` of the group owns D / kMergeLanes consecutive
// elements.  Lane j of a row's group holds the slot and lse of partials j, j + kMergeLanes, ... in
// turn, so the dependent chain comb_off -> comb_slot -> part_lse -> part_o is walked once per
// chunk of kMergeLanes partials and the o loads of 4 partials issue together.
// The weighted sum runs in the fixed plan order: a row's result does not depend on which kernel or
// CTA merges it (the combine kernel and the split kernel's merge phase agree bitwise).  Loads use
// ld.global.cg: in the merge phase the partials were written by other CTAs of the same kernel, so
// the incoherent read-only path must not serve them (hence .cg on the hinted loads).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <type_traits>

namespace orion {

#ifndef ORION_MERGE_LANES
#define ORION_MERGE_LANES 16
#endif
// lanes per row: at least one 16-byte load (8 halves) per lane and partial
template <int D> constexpr int merge_lanes() { return (D / ORION_MERGE_LANES) >= 4 ? ORION_MERGE_LANES : D / 4; }

// Cache policies of the merge's loads: the plan's combine CSR is re-read by every layer's combine
// (evict_last keeps it resident); a partial is dead once merged (evict_first).
__device__ __forceinline__ uint64_t merge_policy(bool last) {
  uint64_t pol;
  if (last) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ int32_t ld_hint(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.cg.L2::cache_hint.b32 %0, [%1], %2;\n" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_hint(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.cg.L2::cache_hint.f32 %0, [%1], %2;\n" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint2 ld_hint(const uint2* p, uint64_t pol) {
  uint2 v;
  asm volatile("ld.global.cg.L2::cache_hint.v2.b32 {%0, %1}, [%2], %3;\n" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint4 ld_hint(const uint4* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.cg.L2::cache_hint.v4.b32 {%0, %1, %2, %3}, [%4], %5;\n"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

template <int D, int kMergeLanes = merge_lanes<D>()>
__device__ __forceinline__ void merge_row16(const int32_t* __restrict__ comb_off, const int32_t* __restrict__ comb_slot,
                                            const __half* part_o, const float* part_lse,
                                            __nv_bfloat16* __restrict__ out, float* __restrict__ lse, int row,
                                            bool valid, int sub) {
  constexpr int E = D / kMergeLanes;  // elements per lane (4 or more)
  constexpr int EV = E >= 8 ? 8 : 4;  // halves per vector load: 16 B, or 8 B at 4 elements per lane
  constexpr int U = E / EV;           // vector loads per lane per partial
  using Vec = typename std::conditional<(EV == 8), uint4, uint2>::type;
  const unsigned full = 0xffffffffu;
  const uint64_t keep = merge_policy(true), drop = merge_policy(false);
  const int e0 = valid ? ld_hint(comb_off + row, keep) : 0;
  const int n = valid ? ld_hint(comb_off + row + 1, keep) - e0 : 0;
  int nmax = n;  // the warp walks chunks uniformly (shuffles need every lane)
#pragma unroll
  for (int o = 16; o >= kMergeLanes; o >>= 1) nmax = max(nmax, __shfl_xor_sync(full, nmax, o));
  // Pass 1: M = max lse2 of the row; chunk 0's slot / lse stay in registers.
  const int slot0 = sub < n ? ld_hint(comb_slot + e0 + sub, keep) : 0;
  const float lse0 = sub < n ? ld_hint(part_lse + slot0, drop) : -INFINITY;
  float M = lse0;
  for (int c = kMergeLanes; c < nmax; c += kMergeLanes)
    if (c + sub < n) M = fmaxf(M, ld_hint(part_lse + ld_hint(comb_slot + e0 + c + sub, keep), drop));
#pragma unroll
  for (int o = kMergeLanes / 2; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(full, M, o, kMergeLanes));
  const float base = M == -INFINITY ? 0.f : M;
  float acc[E];
#pragma unroll
  for (int i = 0; i < E; ++i) acc[i] = 0.f;
  float L = 0.f;
  // Pass 2: weights and the weighted sum of o, chunk by chunk, 4 partials per batch.
  for (int c = 0; c < nmax; c += kMergeLanes) {
    int slot_l = slot0;
    float lse_l = lse0;
    if (c > 0) {
      slot_l = c + sub < n ? ld_hint(comb_slot + e0 + c + sub, keep) : 0;
      lse_l = c + sub < n ? ld_hint(part_lse + slot_l, drop) : -INFINITY;
    }
    float w_l = 0.f;
    if (c + sub < n) asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(w_l) : "f"(lse_l - base));
    const int cn = min(nmax - c, kMergeLanes);
    for (int j0 = 0; j0 < cn; j0 += 4) {
      Vec x[4][U];
      float wt[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int s = __shfl_sync(full, slot_l, (j0 + j) & (kMergeLanes - 1), kMergeLanes);
        wt[j] = __shfl_sync(full, w_l, (j0 + j) & (kMergeLanes - 1), kMergeLanes);
        if (c + j0 + j < n) {
          const Vec* src = reinterpret_cast<const Vec*>(part_o + static_cast<size_t>(s) * D + sub * E);
#pragma unroll
          for (int u = 0; u < U; ++u) x[j][u] = ld_hint(src + u, drop);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (c + j0 + j < n) {
          L += wt[j];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const __half2* h2 = reinterpret_cast<const __half2*>(&x[j][u]);
#pragma unroll
            for (int i = 0; i < EV / 2; ++i) {
              const float2 f = __half22float2(h2[i]);
              acc[u * EV + 2 * i] += wt[j] * f.x;
              acc[u * EV + 2 * i + 1] += wt[j] * f.y;
            }
          }
        }
      }
    }
  }
  if (!valid) return;
  const float inv = L > 0.f ? 1.f / L : 0.f;
  uint32_t* o = reinterpret_cast<uint32_t*>(out + static_cast<size_t>(row) * D + sub * E);
  uint32_t pk[E / 2];
#pragma unroll
  for (int i = 0; i < E / 2; ++i) {
    __nv_bfloat162 b = __floats2bfloat162_rn(acc[2 * i] * inv, acc[2 * i + 1] * inv);
    pk[i] = *reinterpret_cast<uint32_t*>(&b);
  }
  if constexpr (EV == 8) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      reinterpret_cast<uint4*>(o)[u] = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
  } else {
    *reinterpret_cast<uint2*>(o) = make_uint2(pk[0], pk[1]);
  }
  if (lse && sub == 0) lse[row] = L > 0.f ? (M + log2f(L)) * 0.6931471805599453f : -INFINITY;
}

}  // namespace orion
