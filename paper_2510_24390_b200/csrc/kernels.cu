// kernels.cu — device side of the Orion expansion decode step for sm_100a.
//
//   K1 kv_append_kernel   one block per branch; 128-bit bit-exact copy of the new token's K/V
//                         into slot own_len of the branch's own page run.
//   K2 split_kernel       one work item = (shared piece, kv head, token chunk, <=64 query rows).
//                         The chunk's K/V tokens are gathered page-by-page with 16-byte cp.async
//                         into an XOR-swizzled 3-stage shared-memory ring, so every token of a
//                         shared prefix/ancestor piece is read from HBM once for all the rows
//                         (branches x GQA heads) that attend to it.  Q.K^T and P.V run on the
//                         tensor cores (mma.sync m16n8k16 bf16 -> fp32), with an fp32 online
//                         softmax in the log2 domain (row max / sum by warp shuffles).  Each
//                         row's partial (m, l, acc) goes to the fp32 workspace.
//   K3 combine_kernel     one warp (fp32 partials) or 8 lanes (fp16 partials) per (branch, q head):
//                         LSE-merge of its partials in plan order,
//                         out = acc / l rounded to bf16 (RNE), lse = ln-sum-exp.
//
// Semantics: include/orion.h.  Design and rooflines: DESIGN.md §"Kernels".
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <map>
#include <mutex>

#include "../../include/orion.h"
#include "plan_format.h"
#include "merge16.h"
#include "nvtx_range.h"
#include "split_tc.h"

namespace orion {
orion_status check_shape_public(const orion_attn_shape* s);
}  // namespace orion

using namespace orion;

namespace {

constexpr int kStages = 3;
constexpr int kThreads = 128;   // 4 warps, 16 query rows each
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// ------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async_16(uint32_t dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;  // n == 0: zero-fill, nothing read
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float2 unpack_bf16(uint32_t v) {
  return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&v));
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

// Byte offset of 16-byte chunk `c` of row `r` in a [rows][D] bf16 tile; XOR swizzle on the low
// three chunk bits makes the 8 rows of every ldmatrix phase hit 8 distinct bank groups.
template <int D>
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return static_cast<uint32_t>(r * (D * 2) + ((c ^ (r & 7)) << 4));
}

struct SplitArgs {
  const WorkItem* items;
  const int32_t* readers;
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  const int32_t* page_table;
  const int32_t* own_len;
  float* part_acc;
  float2* part_ml;
  int32_t hq, hkv, group, page_shift;
  int32_t kvs;  // (page, kv head) block stride: 1 separate K/V caches, 2 interleaved
  float scale_log2;
};

// ------------------------------------------------------------------------------ K2 split
template <int D>
__global__ void __launch_bounds__(kThreads, 2) split_kernel(const SplitArgs a) {
  constexpr int CH = D / 8;                 // 16-byte chunks per token row
  constexpr int TILE_BYTES = kTileTokens * D * 2;
  constexpr int NB_S = kTileTokens / 8;     // n-blocks of S per tile (8 tokens each)
  constexpr int NB_O = D / 8;               // n-blocks of the output accumulator
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sK = smem + kRowsPerItem * D * 2;
  uint8_t* sV = sK + kStages * TILE_BYTES;

  const WorkItem w = a.items[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int end = w.t1;
  if (w.dyn >= 0) end = min(end, __ldg(a.own_len + w.dyn));
  const int ntok = max(0, end - w.t0);
  const int ntiles = (ntok + kTileTokens - 1) / kTileTokens;
  const int pmask = (1 << a.page_shift) - 1;
  const size_t head_stride = (static_cast<size_t>(D) << a.page_shift) * a.kvs;  // (page, kv head) block stride

  // Q rows of this item -> sQ (zero rows past n_rows).
  for (int i = tid; i < kRowsPerItem * CH; i += kThreads) {
    const int r = i / CH, c = i % CH;
    const bool ok = r < w.n_rows;
    const __nv_bfloat16* src = a.q;
    if (ok) {
      const int rr = w.row_begin + r;
      const int b = __ldg(a.readers + w.readers_off + rr / a.group);
      const int h = w.kv_head * a.group + rr % a.group;
      src = a.q + (static_cast<size_t>(b) * a.hq + h) * D + c * 8;
    }
    cp_async_16(smem_addr(sQ + swz<D>(r, c)), src, ok);
  }
  cp_async_commit();

  auto load_tile = [&](int tile, int stage) {
    const int tbase = w.t0 + tile * kTileTokens;
    uint8_t* dk = sK + stage * TILE_BYTES;
    uint8_t* dv = sV + stage * TILE_BYTES;
#pragma unroll 4
    for (int i = tid; i < kTileTokens * CH; i += kThreads) {
      const int tt = i / CH, c = i % CH;
      const int pos = tbase + tt;
      const bool ok = pos < end;
      size_t off = 0;
      if (ok) {
        const int page = __ldg(a.page_table + w.pt_off + (pos >> a.page_shift));
        off = (static_cast<size_t>(page) * a.hkv + w.kv_head) * head_stride +
              static_cast<size_t>(pos & pmask) * D + c * 8;
      }
      cp_async_16(smem_addr(dk + swz<D>(tt, c)), a.k + off, ok);
      cp_async_16(smem_addr(dv + swz<D>(tt, c)), a.v + off, ok);
    }
  };

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < ntiles) load_tile(s, s);
    cp_async_commit();
  }

  const int wr0 = warp * 16;
  const bool active = wr0 < w.n_rows;
  uint32_t qf[D / 16][4];
  float acc[NB_O][4];
#pragma unroll
  for (int n = 0; n < NB_O; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  for (int it = 0; it < ntiles; ++it) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    {
      const int nt = it + kStages - 1;
      if (nt < ntiles) load_tile(nt, nt % kStages);
      cp_async_commit();
    }
    if (!active) continue;
    if (it == 0) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const int m = lane >> 3;
        const int r = wr0 + (m & 1) * 8 + (lane & 7);
        ldsm_x4(smem_addr(sQ + swz<D>(r, kk * 2 + (m >> 1))), qf[kk][0], qf[kk][1], qf[kk][2],
                qf[kk][3]);
      }
    }
    const uint8_t* tk = sK + (it % kStages) * TILE_BYTES;
    const uint8_t* tv = sV + (it % kStages) * TILE_BYTES;

    // S = Q K^T for this warp's 16 rows x 64 tokens.
    float s[NB_S][4];
#pragma unroll
    for (int n = 0; n < NB_S; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < NB_S / 2; ++np) {
        const int m = lane >> 3;
        const int tok = np * 16 + (m >> 1) * 8 + (lane & 7);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(smem_addr(tk + swz<D>(tok, kk * 2 + (m & 1))), b0, b1, b2, b3);
        mma_bf16(s[2 * np], qf[kk], b0, b1);
        mma_bf16(s[2 * np + 1], qf[kk], b2, b3);
      }
    }
    // Scale into the log2 domain and mask tokens past the end.
    const int tbase = w.t0 + it * kTileTokens;
    const bool tail = tbase + kTileTokens > end;
#pragma unroll
    for (int n = 0; n < NB_S; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float x = s[n][e] * a.scale_log2;
        if (tail && tbase + n * 8 + 2 * (lane & 3) + (e & 1) >= end) x = -INFINITY;
        s[n][e] = x;
      }
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int n = 0; n < NB_S; ++n) {
      mx0 = fmaxf(mx0, fmaxf(s[n][0], s[n][1]));
      mx1 = fmaxf(mx1, fmaxf(s[n][2], s[n][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float nm0 = fmaxf(m0, mx0), nm1 = fmaxf(m1, mx1);
    const float base0 = nm0 == -INFINITY ? 0.f : nm0;
    const float base1 = nm1 == -INFINITY ? 0.f : nm1;
    const float al0 = fast_exp2(m0 - base0), al1 = fast_exp2(m1 - base1);
    m0 = nm0;
    m1 = nm1;
    // P = exp2(S - m), rounded to bf16 for the PV MMA; l sums the SAME rounded values.
    uint32_t p[NB_S][2];
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int n = 0; n < NB_S; ++n) {
      p[n][0] = pack_bf16(fast_exp2(s[n][0] - base0), fast_exp2(s[n][1] - base0));
      p[n][1] = pack_bf16(fast_exp2(s[n][2] - base1), fast_exp2(s[n][3] - base1));
      const float2 u = unpack_bf16(p[n][0]), v = unpack_bf16(p[n][1]);
      rs0 += u.x + u.y;
      rs1 += v.x + v.y;
    }
    l0 = l0 * al0 + rs0;
    l1 = l1 * al1 + rs1;
#pragma unroll
    for (int n = 0; n < NB_O; ++n) {
      acc[n][0] *= al0; acc[n][1] *= al0;
      acc[n][2] *= al1; acc[n][3] *= al1;
    }
    // O += P V.
#pragma unroll
    for (int kt = 0; kt < kTileTokens / 16; ++kt) {
      const uint32_t pa[4] = {p[2 * kt][0], p[2 * kt][1], p[2 * kt + 1][0], p[2 * kt + 1][1]};
#pragma unroll
      for (int np = 0; np < NB_O / 2; ++np) {
        const int m = lane >> 3;
        const int tok = kt * 16 + (m & 1) * 8 + (lane & 7);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(smem_addr(tv + swz<D>(tok, np * 2 + (m >> 1))), b0, b1, b2, b3);
        mma_bf16(acc[2 * np], pa, b0, b1);
        mma_bf16(acc[2 * np + 1], pa, b2, b3);
      }
    }
  }
  cp_async_wait<0>();
  if (!active) return;
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const int r0 = wr0 + (lane >> 2), r1 = r0 + 8;
  const int c0 = 2 * (lane & 3);
  if (r0 < w.n_rows) {
    float* dst = a.part_acc + static_cast<size_t>(w.slot0 + r0) * D;
#pragma unroll
    for (int n = 0; n < NB_O; ++n)
      *reinterpret_cast<float2*>(dst + n * 8 + c0) = make_float2(acc[n][0], acc[n][1]);
    if ((lane & 3) == 0) a.part_ml[w.slot0 + r0] = make_float2(m0, l0);
  }
  if (r1 < w.n_rows) {
    float* dst = a.part_acc + static_cast<size_t>(w.slot0 + r1) * D;
#pragma unroll
    for (int n = 0; n < NB_O; ++n)
      *reinterpret_cast<float2*>(dst + n * 8 + c0) = make_float2(acc[n][2], acc[n][3]);
    if ((lane & 3) == 0) a.part_ml[w.slot0 + r1] = make_float2(m1, l1);
  }
}

// ------------------------------------------------------------------------------ K3 combine
template <int D>
__global__ void __launch_bounds__(256) combine_kernel(const int32_t* __restrict__ comb_off,
                                                      const int32_t* __restrict__ comb_slot,
                                                      const float* __restrict__ part_acc,
                                                      const float2* __restrict__ part_ml,
                                                      __nv_bfloat16* __restrict__ out,
                                                      float* __restrict__ lse, int n_rows) {
  constexpr int V = D / 32;  // floats per lane
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  const int e0 = __ldg(comb_off + row), e1 = __ldg(comb_off + row + 1);
  float M = -INFINITY;
  for (int e = e0 + lane; e < e1; e += 32) M = fmaxf(M, part_ml[__ldg(comb_slot + e)].x);
#pragma unroll
  for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  const float base = M == -INFINITY ? 0.f : M;
  float acc[V];
#pragma unroll
  for (int i = 0; i < V; ++i) acc[i] = 0.f;
  float L = 0.f;
  for (int e = e0; e < e1; ++e) {  // fixed plan order -> deterministic
    const int slot = __ldg(comb_slot + e);
    const float2 ml = part_ml[slot];
    const float wgt = fast_exp2(ml.x - base);
    L += wgt * ml.y;
    const float* src = part_acc + static_cast<size_t>(slot) * D + lane * V;
    if constexpr (V == 4) {
      const float4 x = *reinterpret_cast<const float4*>(src);
      acc[0] += wgt * x.x; acc[1] += wgt * x.y; acc[2] += wgt * x.z; acc[3] += wgt * x.w;
    } else {
      const float2 x = *reinterpret_cast<const float2*>(src);
      acc[0] += wgt * x.x; acc[1] += wgt * x.y;
    }
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  __nv_bfloat16* o = out + static_cast<size_t>(row) * D + lane * V;
  if constexpr (V == 4) {
    uint2 pk;
    pk.x = pack_bf16(acc[0] * inv, acc[1] * inv);
    pk.y = pack_bf16(acc[2] * inv, acc[3] * inv);
    *reinterpret_cast<uint2*>(o) = pk;
  } else {
    *reinterpret_cast<uint32_t*>(o) = pack_bf16(acc[0] * inv, acc[1] * inv);
  }
  if (lse && lane == 0) lse[row] = L > 0.f ? (M + log2f(L)) * kLn2 : -INFINITY;
}

// K3 for the fp16 partial format (plan_format.h): partial i = (o_i = acc_i / l_i, lse2_i), so
// out = sum_i 2^(lse2_i - M) o_i / sum_i 2^(lse2_i - M) and lse = (M + log2 sum) ln 2.
// merge_lanes<D>() lanes per row (16 at D = 128: two rows per warp; merge16.h): each lane owns
// D/16 consecutive elements (one 16-B load per partial).  Lane j of a row's group holds the slot
// and lse of partials j, j+16, ... in turn, so the dependent chain comb_off -> comb_slot ->
// part_lse -> part_o is walked once per chunk of 16 partials (c4: ~4.4 partials per row, one
// chunk) and the o loads of 4 partials issue together.  16 lanes per row measured +2.8 % on c4's
// 8-query share over 8 (4 lanes: -6 %; 32 lanes with 8-byte loads: +0.2 % more), c4 +0.3 %.  Accumulation is in the fixed plan
// order (deterministic, and the same expression sequence as a serial loop).
#ifndef ORION_COMB_THREADS
#define ORION_COMB_THREADS 128
#endif
constexpr int kCombThreads = ORION_COMB_THREADS;

template <int D>
__global__ void __launch_bounds__(kCombThreads) combine16_kernel(const int32_t* __restrict__ comb_off,
                                                                 const int32_t* __restrict__ comb_slot,
                                                                 const __half* __restrict__ part_o,
                                                                 const float* __restrict__ part_lse,
                                                                 __nv_bfloat16* __restrict__ out,
                                                                 float* __restrict__ lse, int n_rows) {
  constexpr int kCombLanes = merge_lanes<D>();
  const int row = blockIdx.x * (kCombThreads / kCombLanes) + (threadIdx.x / kCombLanes);
  pdl_trigger();
  pdl_wait();
  merge_row16<D>(comb_off, comb_slot, part_o, part_lse, out, lse, row < n_rows ? row : 0, row < n_rows,
                 threadIdx.x & (kCombLanes - 1));
}

// ------------------------------------------------------------------------------ K1 append
template <int D>
__global__ void __launch_bounds__(128) kv_append_kernel(
    const __nv_bfloat16* __restrict__ k_new, const __nv_bfloat16* __restrict__ v_new,
    __nv_bfloat16* __restrict__ k_cache, __nv_bfloat16* __restrict__ v_cache,
    const int32_t* __restrict__ own_pt_off, const int32_t* __restrict__ own_cap,
    const int32_t* __restrict__ page_table, int32_t* __restrict__ own_len, int hkv,
    int page_shift, int mode, int kvs, int num_pages, int* err) {
  constexpr int CH = D / 8;
  __shared__ int s_pos, s_page, s_len;
  const int b = blockIdx.x;
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) {
    const int len = own_len[b];
    const int pos = mode == ORION_APPEND_REWRITE ? len - 1 : len;
    const bool ok = pos >= 0 && pos < own_cap[b];
    s_len = len;
    s_pos = pos;
    int page = ok ? page_table[own_pt_off[b] + (pos >> page_shift)] : -1;
    if (page >= num_pages || (ok && page < 0)) {     // outside the caches: never written
      if (err) atomicCAS(err, 0, b + 1);
      page = -1;
    }
    s_page = page;
  }
  __syncthreads();
  const int page = s_page, pos = s_pos;
  if (page < 0) return;
  const size_t row = static_cast<size_t>(pos & ((1 << page_shift) - 1)) * D;
  for (int i = threadIdx.x; i < hkv * CH; i += blockDim.x) {
    const int g = i / CH, c = i % CH;
    const size_t dst = (((static_cast<size_t>(page) * hkv + g) * kvs) << page_shift) * D + row + c * 8;
    const size_t src = (static_cast<size_t>(b) * hkv + g) * D + c * 8;
    *reinterpret_cast<uint4*>(k_cache + dst) = *reinterpret_cast<const uint4*>(k_new + src);
    *reinterpret_cast<uint4*>(v_cache + dst) = *reinterpret_cast<const uint4*>(v_new + src);
  }
  if (threadIdx.x == 0 && mode == ORION_APPEND_ADVANCE) own_len[b] = s_len + 1;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

std::mutex g_setup_mu;
std::map<int, int> g_sms;                                   // device -> SM count
std::map<std::pair<int, const void*>, cudaError_t> g_smem;  // (device, kernel) -> attribute status
}  // namespace

namespace orion {
int current_device_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lk(g_setup_mu);
  auto f = g_sms.find(dev);
  if (f != g_sms.end()) return f->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  g_sms[dev] = n;
  return n;
}

// SMs available to the context that owns `stream`, or -1 for a green-context stream (a partition:
// fewer SMs than the device) or when the driver cannot say.  Cached per context.
int stream_context_sms(cudaStream_t stream) {
  // the entry point's default version (12.5+) is cuStreamGetCtx_v2: (stream, context, green context)
  typedef CUresult (*StreamGetCtxFn)(CUstream, CUcontext*, CUgreenCtx*);
  typedef CUresult (*CtxGetDevResourceFn)(CUcontext, CUdevResource*, CUdevResourceType);
  static const StreamGetCtxFn get_ctx = []() -> StreamGetCtxFn {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPointByVersion("cuStreamGetCtx", &p, 12050, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess
               ? reinterpret_cast<StreamGetCtxFn>(p)
               : nullptr;
  }();
  static const CtxGetDevResourceFn get_res = []() -> CtxGetDevResourceFn {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPointByVersion("cuCtxGetDevResource", &p, 12040, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess
               ? reinterpret_cast<CtxGetDevResourceFn>(p)
               : nullptr;
  }();
  static std::map<CUcontext, int> cache;
  if (!get_ctx || !get_res) return -1;
  CUcontext ctx = nullptr;
  CUgreenCtx gctx = nullptr;
  if (get_ctx(reinterpret_cast<CUstream>(stream), &ctx, &gctx) != CUDA_SUCCESS || !ctx) return -1;
  if (gctx) return -1;   // a green-context stream: pctx is the primary context, not the partition
  std::lock_guard<std::mutex> lk(g_setup_mu);
  auto f = cache.find(ctx);
  if (f != cache.end()) return f->second;
  CUdevResource r;
  int n = -1;
  if (get_res(ctx, &r, CU_DEV_RESOURCE_TYPE_SM) == CUDA_SUCCESS) n = static_cast<int>(r.sm.smCount);
  cache[ctx] = n;
  return n;
}

cudaError_t ensure_dynamic_smem(const void* func, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_setup_mu);
  auto key = std::make_pair(dev, func);
  auto f = g_smem.find(key);
  if (f != g_smem.end()) return f->second;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  g_smem[key] = e;
  return e;
}
}  // namespace orion

namespace {

int log2i(int x) {
  int s = 0;
  while ((1 << s) < x) ++s;
  return s;
}

template <int D>
size_t split_smem_bytes() {
  return static_cast<size_t>(kRowsPerItem) * D * 2 + 2ull * kStages * kTileTokens * D * 2;
}

#ifdef ORION_CHECK
// Debug build only (`make check` -> liborion_check.so, selected with ORION_LIB): the content
// checks include/orion.h leaves out of the release library.  Before every split launch, each work
// item's token ranges are walked as the kernels will walk them (tokens [t0, min(t1, own_len[dyn])),
// plan_format.h) and every page id they read must lie in [0, num_pages); a dynamic range's branch
// must exist and its own_len be >= 0.  The release kernels read pages through TMA, which
// zero-fills out-of-range boxes instead of faulting, so a bad page table would otherwise give
// silently wrong output.  The check synchronises the stream (not capturable in a CUDA graph).
__device__ int g_check_err[4];  // first failing item + 1, what, value, index

__device__ void check_report(int item, int what, int value, int index) {
  if (atomicCAS(&g_check_err[0], 0, item + 1) == 0) {
    g_check_err[1] = what;
    g_check_err[2] = value;
    g_check_err[3] = index;
  }
}

__global__ void check_plan_kernel(const WorkItem* __restrict__ items, const Range* __restrict__ ranges,
                                  int n_items, const int32_t* __restrict__ page_table,
                                  const int32_t* __restrict__ own_len, int n_branches, int num_pages,
                                  int page_shift) {
  const int it = blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= n_items) return;
  const WorkItem w = items[it];
  const int nr = (w.flags & kItemRanges) ? w.n_ranges : 1;
  for (int r = 0; r < nr; ++r) {
    int pt_off = w.pt_off, t0 = w.t0, t1 = w.t1, dyn = w.dyn;
    if (w.flags & kItemRanges) {
      const Range R = ranges[w.pt_off + r];
      pt_off = R.pt_off; t0 = R.t0; t1 = R.t1; dyn = R.dyn;
    }
    int end = t1;
    if (dyn >= 0) {
      if (dyn >= n_branches) return check_report(it, 1, dyn, r);
      const int ol = own_len[dyn];
      if (ol < 0) return check_report(it, 2, ol, dyn);
      end = min(end, ol);
    }
    for (int t = t0 & ~((1 << page_shift) - 1); t < end; t += 1 << page_shift) {
      const int pg = page_table[pt_off + (t >> page_shift)];
      if (pg < 0 || pg >= num_pages) return check_report(it, 3, pg, pt_off + (t >> page_shift));
    }
  }
}

orion_status check_plan_contents(const PlanHeader* h, const char* dplan, const int32_t* page_table,
                                 const int32_t* own_len, int num_pages, cudaStream_t st) {
  static const int zero[4] = {0, 0, 0, 0};
  int res[4] = {0, 0, 0, 0};
  {   // the device plan must be a copy of this host plan (not a stale or foreign one)
    PlanHeader dh;
    cudaError_t ce = cudaMemcpyAsync(&dh, dplan, sizeof dh, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) return fail(ORION_ERR_CUDA, "ORION_CHECK plan read-back: %s", cudaGetErrorString(ce));
    if (dh.magic != h->magic || dh.plan_id != h->plan_id || dh.n_items != h->n_items ||
        dh.n_partials != h->n_partials)
      return fail(ORION_ERR_INVALID_ARG, "ORION_CHECK: d_plan is not a copy of h_plan (plan id %llx vs %llx)",
                  (unsigned long long)dh.plan_id, (unsigned long long)h->plan_id);
  }
  cudaError_t e = cudaMemcpyToSymbolAsync(g_check_err, zero, sizeof zero, 0, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    check_plan_kernel<<<(h->n_items + 127) / 128, 128, 0, st>>>(
        reinterpret_cast<const WorkItem*>(dplan + h->items_off),
        reinterpret_cast<const Range*>(dplan + h->ranges_off), h->n_items, page_table, own_len,
        h->n_branches, num_pages, log2i(h->page_size));
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyFromSymbolAsync(res, g_check_err, sizeof res, 0, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fail(ORION_ERR_CUDA, "ORION_CHECK: %s", cudaGetErrorString(e));
  static const char* what[4] = {"", "dynamic range names a branch >= n_branches", "own_len < 0",
                                "page id outside [0, num_pages)"};
  if (res[0])
    return fail(ORION_ERR_INVALID_ARG, "ORION_CHECK: work item %d: %s (value %d, index %d)", res[0] - 1,
                what[res[1] & 3], res[2], res[3]);
  return ORION_OK;
}
#endif

}  // namespace

namespace orion {
// Append page-id check of the debug build (ORION_CHECK): the append kernels record the first
// branch whose target page lies outside [0, num_pages) (they skip its write in every build); the
// debug build reads the record back (synchronising) and reports INVALID_ARG.
#ifdef ORION_CHECK
__device__ int g_append_err;
int* append_check_begin(cudaStream_t st) {
  int* p = nullptr;
  if (cudaGetSymbolAddress(reinterpret_cast<void**>(&p), g_append_err) != cudaSuccess) return nullptr;
  cudaMemsetAsync(p, 0, sizeof(int), st);
  return p;
}
orion_status append_check_end(cudaStream_t st, const char* what) {
  int v = 0;
  cudaError_t e = cudaMemcpyFromSymbolAsync(&v, g_append_err, sizeof v, 0, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fail(ORION_ERR_CUDA, "ORION_CHECK %s: %s", what, cudaGetErrorString(e));
  if (v) return fail(ORION_ERR_INVALID_ARG, "ORION_CHECK %s: branch %d's own-run page id is outside [0, num_pages)", what, v - 1);
  return ORION_OK;
}
#else
int* append_check_begin(cudaStream_t) { return nullptr; }
orion_status append_check_end(cudaStream_t, const char*) { return ORION_OK; }
#endif
}  // namespace orion

namespace {

template <int D>
orion_status launch_split(const PlanHeader* h, const char* dplan, const void* q, const void* k,
                          const void* v, int32_t num_pages, const int32_t* page_table,
                          const int32_t* own_len, void* ws, cudaStream_t st, int kvs, void* out = nullptr,
                          float* lse = nullptr, const FusedAppend* app = nullptr) {
#ifdef ORION_CHECK
  {
    const orion_status cs = check_plan_contents(h, dplan, page_table, own_len, num_pages, st);
    if (cs != ORION_OK) return cs;
  }
#endif
  if (h->variant == kVariantTC || h->variant == kVariantTCT) {
    TcArgs t;
    t.out = static_cast<__nv_bfloat16*>(out);      // direct output (point-prefill plans only)
    t.lse = lse;
    t.items = reinterpret_cast<const WorkItem*>(dplan + h->items_off);
    t.ranges = reinterpret_cast<const Range*>(dplan + h->ranges_off);
    t.readers = reinterpret_cast<const int32_t*>(dplan + h->readers_off);
    t.q = static_cast<const __nv_bfloat16*>(q);
    t.page_table = page_table;
    t.own_len = own_len;
    t.part_acc = static_cast<float*>(ws);
    t.part_ml = reinterpret_cast<float2*>(static_cast<char*>(ws) + h->acc_bytes);
    t.part_o = static_cast<__half*>(ws);
    t.part_lse = reinterpret_cast<float*>(static_cast<char*>(ws) + h->acc_bytes);
    t.n_items = h->n_items;
    t.hq = h->num_q_heads;
    t.hkv = h->num_kv_heads;
    t.group = h->group;
    t.page_shift = log2i(h->page_size);
    t.kvs = kvs;
    t.scale_log2 = h->sm_scale * kLog2e;
    t.lc = h->prefill_rows > 0 ? h->prefill_rows : 1;
    t.work_counter = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + h->counter_off);
    t.part16 = 0;
    t.pdl_late = 0;
    t.app = FusedAppend{};
    if (app) {   // only on the swap-AB kernel of a plan without big items (orion_expand_step)
      if (h->variant != kVariantTCT || h->n_big > 0) return fail(ORION_ERR_UNSUPPORTED, "fused append on a hybrid plan");
      t.app = *app;
      t.app.epoch = t.work_counter + kAppendEpochWord;
      t.app.flags = t.work_counter + kCounterBytes / 4;
      t.app.enabled = 1;
    }
    if (h->variant == kVariantTCT) {
      if (D != 128) return fail(ORION_ERR_UNSUPPORTED, "transposed split kernel needs head_dim 128");
      if (h->n_big > 0) {
        // hybrid plan: items [0, n_big) (65..128 rows) on the rows-on-lanes kernel, writing the
        // fp16 partial format, then [n_big, n_items) on the swap-AB kernel with its own counter
        TcArgs tb = t;
        tb.n_items = h->n_big;
        tb.part16 = 1;
        const orion_status s1 = launch_split_tc<D>(h, tb, k, v, num_pages, st);
        if (s1 != ORION_OK || h->n_big == h->n_items) return s1;
        t.items += h->n_big;
        t.n_items = h->n_items - h->n_big;
        t.work_counter += 4;
        t.pdl_late = 1;
      }
      return launch_split_tct(h, t, k, v, num_pages, st);
    }
    return launch_split_tc<D>(h, t, k, v, num_pages, st);
  }
  const cudaError_t attr_err =
      ensure_dynamic_smem(reinterpret_cast<const void*>(split_kernel<D>), (int)split_smem_bytes<D>());
  if (attr_err != cudaSuccess)
    return fail(ORION_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(attr_err));
  SplitArgs a;
  a.items = reinterpret_cast<const WorkItem*>(dplan + h->items_off);
  a.readers = reinterpret_cast<const int32_t*>(dplan + h->readers_off);
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.k = static_cast<const __nv_bfloat16*>(k);
  a.v = static_cast<const __nv_bfloat16*>(v);
  a.page_table = page_table;
  a.own_len = own_len;
  a.part_acc = static_cast<float*>(ws);
  a.part_ml = reinterpret_cast<float2*>(static_cast<char*>(ws) + h->acc_bytes);
  a.hq = h->num_q_heads;
  a.hkv = h->num_kv_heads;
  a.group = h->group;
  a.page_shift = log2i(h->page_size);
  a.kvs = kvs;
  a.scale_log2 = h->sm_scale * kLog2e;
  split_kernel<D><<<h->n_items, kThreads, split_smem_bytes<D>(), st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ORION_ERR_CUDA, "split_kernel: %s", cudaGetErrorString(e));
  return ORION_OK;
}

template <int D>
orion_status launch_combine(const PlanHeader* h, const char* dplan, void* out, float* lse,
                            const void* ws, cudaStream_t st) {
  const int nb = (h->n_rows + 7) / 8;
  if (partials_fp16(h->variant)) {
    cudaError_t e = launch_pdl(
        combine16_kernel<D>, dim3((h->n_rows + kCombThreads / merge_lanes<D>() - 1) / (kCombThreads / merge_lanes<D>())),
        dim3(kCombThreads), 0, st,
        reinterpret_cast<const int32_t*>(dplan + h->comb_off_off),
        reinterpret_cast<const int32_t*>(dplan + h->comb_slot_off), static_cast<const __half*>(ws),
        reinterpret_cast<const float*>(static_cast<const char*>(ws) + h->acc_bytes),
        static_cast<__nv_bfloat16*>(out), lse, h->n_rows);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ORION_ERR_CUDA, "combine16_kernel: %s", cudaGetErrorString(e));
    return ORION_OK;
  }
  const float* acc = static_cast<const float*>(ws);
  const float2* ml = reinterpret_cast<const float2*>(static_cast<const char*>(ws) + h->acc_bytes);
  combine_kernel<D><<<nb, 256, 0, st>>>(reinterpret_cast<const int32_t*>(dplan + h->comb_off_off),
                                        reinterpret_cast<const int32_t*>(dplan + h->comb_slot_off),
                                        acc, ml, static_cast<__nv_bfloat16*>(out), lse, h->n_rows);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ORION_ERR_CUDA, "combine_kernel: %s", cudaGetErrorString(e));
  return ORION_OK;
}

// Shared validation of the attention entry points.
orion_status check_attn(const orion_attn_shape* shape, int32_t n_branches, const void* h_plan,
                        const void* d_plan, const void* workspace, size_t workspace_bytes,
                        const PlanHeader** hp) {
  orion_status st = check_shape_public(shape);
  if (st != ORION_OK) return st;
  if (!h_plan || !d_plan || !workspace) return fail(ORION_ERR_INVALID_ARG, "null plan/workspace");
  if (!aligned16(d_plan) || !aligned16(workspace))
    return fail(ORION_ERR_INVALID_ARG, "d_plan / workspace must be 16-byte aligned");
  const PlanHeader* h = static_cast<const PlanHeader*>(h_plan);
  if (h->magic != kPlanMagic || h->version != kPlanVersion)
    return fail(ORION_ERR_INVALID_ARG, "h_plan is not an orion plan");
  if (h->n_branches != n_branches || h->num_q_heads != shape->num_q_heads ||
      h->num_kv_heads != shape->num_kv_heads || h->head_dim != shape->head_dim ||
      h->page_size != shape->page_size)
    return fail(ORION_ERR_INVALID_ARG, "plan was built for another shape / branch count");
  if (workspace_bytes < static_cast<size_t>(h->workspace_bytes))
    return fail(ORION_ERR_INVALID_ARG, "workspace %zu < %lld bytes", workspace_bytes,
                (long long)h->workspace_bytes);
  if (h->n_items < 1) return fail(ORION_ERR_INVALID_ARG, "empty plan");
  *hp = h;
  return ORION_OK;
}

}  // namespace

extern "C" orion_status orion_kv_append(const orion_attn_shape* shape, int32_t n_branches,
                                        const void* k_new, const void* v_new, void* k_cache,
                                        void* v_cache, const int32_t* own_pt_off,
                                        const int32_t* own_cap, const int32_t* page_table,
                                        int32_t num_pages, int32_t* own_len, int32_t mode,
                                        void* stream) {
  const orion::NvtxRange nvtx_range("orion_kv_append");
  orion_status st = check_shape_public(shape);
  if (st != ORION_OK) return st;
  if (n_branches < 0) return fail(ORION_ERR_INVALID_ARG, "n_branches < 0");
  if (mode != ORION_APPEND_ADVANCE && mode != ORION_APPEND_REWRITE)
    return fail(ORION_ERR_INVALID_ARG, "bad append mode %d", mode);
  if (!k_new || !v_new || !k_cache || !v_cache || !own_pt_off || !own_cap || !page_table ||
      !own_len)
    return fail(ORION_ERR_INVALID_ARG, "null device pointer");
  if (!aligned16(k_new) || !aligned16(v_new) || !aligned16(k_cache) || !aligned16(v_cache))
    return fail(ORION_ERR_INVALID_ARG, "K/V pointers must be 16-byte aligned");
  if (num_pages < 1) return fail(ORION_ERR_INVALID_ARG, "num_pages < 1");
  if (n_branches == 0) return ORION_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int shift = log2i(shape->page_size);
  int* err = append_check_begin(s);
  cudaError_t e = launch_pdl(
      shape->head_dim == 128 ? kv_append_kernel<128> : kv_append_kernel<64>, dim3(n_branches), dim3(128), 0, s,
      static_cast<const __nv_bfloat16*>(k_new), static_cast<const __nv_bfloat16*>(v_new),
      static_cast<__nv_bfloat16*>(k_cache), static_cast<__nv_bfloat16*>(v_cache), own_pt_off,
      own_cap, page_table, own_len, shape->num_kv_heads, shift, mode, 1 + shape->kv_interleaved, num_pages, err);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ORION_ERR_CUDA, "kv_append_kernel: %s", cudaGetErrorString(e));
  return append_check_end(s, "kv_append");
}

extern "C" orion_status orion_expand_split(const orion_attn_shape* shape, int32_t n_branches,
                                           const void* q, const void* k_cache,
                                           const void* v_cache, int32_t num_pages,
                                           const int32_t* page_table, const int32_t* own_len,
                                           const void* h_plan, const void* d_plan,
                                           void* workspace, size_t workspace_bytes,
                                           void* stream) {
  const orion::NvtxRange nvtx_range("orion_expand_split");
  const PlanHeader* h = nullptr;
  orion_status st = check_attn(shape, n_branches, h_plan, d_plan, workspace, workspace_bytes, &h);
  if (st != ORION_OK) return st;
  if (!q || !k_cache || !v_cache || !page_table || !own_len)
    return fail(ORION_ERR_INVALID_ARG, "null pointer");
  if (!aligned16(q) || !aligned16(k_cache) || !aligned16(v_cache))
    return fail(ORION_ERR_INVALID_ARG, "device pointers must be 16-byte aligned");
  if (num_pages < 1) return fail(ORION_ERR_INVALID_ARG, "num_pages < 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const char* dp = static_cast<const char*>(d_plan);
  if (shape->head_dim == 128)
    return launch_split<128>(h, dp, q, k_cache, v_cache, num_pages, page_table, own_len, workspace, s,
                             1 + shape->kv_interleaved);
  return launch_split<64>(h, dp, q, k_cache, v_cache, num_pages, page_table, own_len, workspace, s,
                          1 + shape->kv_interleaved);
}

extern "C" orion_status orion_expand_combine(const orion_attn_shape* shape, int32_t n_branches,
                                             void* out, float* lse, const void* h_plan,
                                             const void* d_plan, const void* workspace,
                                             size_t workspace_bytes, void* stream) {
  const orion::NvtxRange nvtx_range("orion_expand_combine");
  const PlanHeader* h = nullptr;
  orion_status st = check_attn(shape, n_branches, h_plan, d_plan, workspace, workspace_bytes, &h);
  if (st != ORION_OK) return st;
  if (!out) return fail(ORION_ERR_INVALID_ARG, "null out");
  if (!aligned16(out)) return fail(ORION_ERR_INVALID_ARG, "out must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const char* dp = static_cast<const char*>(d_plan);
  if (shape->head_dim == 128) return launch_combine<128>(h, dp, out, lse, workspace, s);
  return launch_combine<64>(h, dp, out, lse, workspace, s);
}

extern "C" orion_status orion_expand_attn(const orion_attn_shape* shape, int32_t n_branches,
                                          const void* q, void* out, float* lse,
                                          const void* k_cache, const void* v_cache,
                                          int32_t num_pages, const int32_t* page_table,
                                          const int32_t* own_len, const void* h_plan,
                                          const void* d_plan, void* workspace,
                                          size_t workspace_bytes, void* stream) {
  const orion::NvtxRange nvtx_range("orion_expand_attn");
  if (!out) return fail(ORION_ERR_INVALID_ARG, "null out");
  if (h_plan && static_cast<const PlanHeader*>(h_plan)->magic == kPlanMagic &&
      static_cast<const PlanHeader*>(h_plan)->prefill_rows > 0)
    return fail(ORION_ERR_INVALID_ARG, "a point-prefill plan needs orion_point_prefill_attn");
  orion_status st = orion_expand_split(shape, n_branches, q, k_cache, v_cache, num_pages, page_table, own_len,
                                       h_plan, d_plan, workspace, workspace_bytes, stream);
  if (st != ORION_OK) return st;
  return orion_expand_combine(shape, n_branches, out, lse, h_plan, d_plan, workspace,
                              workspace_bytes, stream);
}

namespace {
#ifndef ORION_FUSE_TOKENS_PER_SM
#define ORION_FUSE_TOKENS_PER_SM 2048
#endif
constexpr int64_t kFuseTokensPerSm = ORION_FUSE_TOKENS_PER_SM;
bool step_fuses(const PlanHeader* h) {
#ifdef ORION_CHECK
  return false;
#else
  return h->variant == kVariantTCT && h->n_big == 0 && h->head_dim == 128 &&
         h->streamed_tokens <= kFuseTokensPerSm * current_device_sms();
#endif
}
}  // namespace

extern "C" orion_status orion_step_launches(const void* h_plan, int32_t* launches) {
  if (!h_plan || !launches) return fail(ORION_ERR_INVALID_ARG, "null pointer");
  const PlanHeader* h = static_cast<const PlanHeader*>(h_plan);
  if (h->magic != kPlanMagic || h->version != kPlanVersion) return fail(ORION_ERR_INVALID_ARG, "not an orion plan");
  if (h->prefill_rows > 0) { *launches = 1; return ORION_OK; }   // point prefill: the split kernel only
  if (step_fuses(h)) { *launches = 1; return ORION_OK; }
  const bool hybrid2 = h->variant == kVariantTCT && h->n_big > 0 && h->n_big < h->n_items;
  *launches = 3 + (hybrid2 ? 1 : 0);
  return ORION_OK;
}

extern "C" orion_status orion_expand_step(const orion_attn_shape* shape, int32_t n_branches,
                                          const void* q, const void* k_new, const void* v_new, void* out,
                                          float* lse, void* k_cache, void* v_cache, int32_t num_pages,
                                          const int32_t* page_table, const int32_t* own_pt_off,
                                          const int32_t* own_cap, int32_t* own_len, int32_t mode,
                                          const void* h_plan, const void* d_plan, void* workspace,
                                          size_t workspace_bytes, void* stream) {
  const orion::NvtxRange nvtx_range("orion_expand_step");
  const PlanHeader* h = nullptr;
  orion_status st = check_attn(shape, n_branches, h_plan, d_plan, workspace, workspace_bytes, &h);
  if (st != ORION_OK) return st;
  if (h->prefill_rows > 0) return fail(ORION_ERR_INVALID_ARG, "a point-prefill plan needs orion_point_prefill_attn");
  // K1 fused into the swap-AB split launch when the plan has no rows-on-lanes items and the step
  // is short (<= kFuseTokensPerSm streamed tokens per SM: there the saved launch and kernel
  // boundary dominate -- c4 with 2 queries 20.4k -> 26.8k tok/s -- while on longer steps the
  // separate append kernel, overlapping the split's prologue through PDL, measured 1-2 % faster:
  // c4 with 8 and 64 queries).  The release library only (the debug build checks every append and
  // plan separately).  Otherwise the two calls it stands for, with the same results.
  // The fused launch's CTAs wait on each other (append flags, the merge's grid barrier), so every
  // CTA must be resident at once: only on a stream of the whole device's context (a green-context
  // partition -- fewer SMs -- or a driver that cannot say runs the two calls).
  bool fuse = step_fuses(h) && shape->head_dim == 128 &&
              stream_context_sms(static_cast<cudaStream_t>(stream)) == current_device_sms();
  if (!fuse) {
    st = orion_kv_append(shape, n_branches, k_new, v_new, k_cache, v_cache, own_pt_off, own_cap, page_table,
                         num_pages, own_len, mode, stream);
    if (st != ORION_OK) return st;
    return orion_expand_attn(shape, n_branches, q, out, lse, k_cache, v_cache, num_pages, page_table, own_len,
                             h_plan, d_plan, workspace, workspace_bytes, stream);
  }
  if (mode != ORION_APPEND_ADVANCE && mode != ORION_APPEND_REWRITE)
    return fail(ORION_ERR_INVALID_ARG, "bad append mode %d", mode);
  if (!q || !out || !k_new || !v_new || !k_cache || !v_cache || !page_table || !own_pt_off || !own_cap || !own_len)
    return fail(ORION_ERR_INVALID_ARG, "null pointer");
  if (!aligned16(q) || !aligned16(out) || !aligned16(k_new) || !aligned16(v_new) || !aligned16(k_cache) ||
      !aligned16(v_cache))
    return fail(ORION_ERR_INVALID_ARG, "device pointers must be 16-byte aligned");
  if (num_pages < 1) return fail(ORION_ERR_INVALID_ARG, "num_pages < 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const char* dp = static_cast<const char*>(d_plan);
  FusedAppend ap{};
  ap.k_new = static_cast<const __nv_bfloat16*>(k_new);
  ap.v_new = static_cast<const __nv_bfloat16*>(v_new);
  ap.k_cache = static_cast<__nv_bfloat16*>(k_cache);
  ap.v_cache = static_cast<__nv_bfloat16*>(v_cache);
  ap.own_pt_off = own_pt_off;
  ap.own_cap = own_cap;
  ap.own_len = own_len;
  ap.err = nullptr;
  ap.n_branches = n_branches;
  ap.mode = mode;
  ap.num_pages = num_pages;
  ap.merge = 1;                                     // K3 as the split launch's last phase
  ap.n_rows = h->n_rows;
  ap.comb_off = reinterpret_cast<const int32_t*>(dp + h->comb_off_off);
  ap.comb_slot = reinterpret_cast<const int32_t*>(dp + h->comb_slot_off);
  ap.out = static_cast<__nv_bfloat16*>(out);
  ap.lse = lse;
  st = launch_split<128>(h, dp, q, k_cache, v_cache, num_pages, page_table, own_len, workspace, s,
                         1 + shape->kv_interleaved, nullptr, nullptr, &ap);
  return st;
}

extern "C" orion_status orion_point_prefill_attn(const orion_attn_shape* shape, int32_t n_branches,
                                                 const void* q, void* out, float* lse,
                                                 const void* k_cache, const void* v_cache,
                                                 int32_t num_pages, const int32_t* page_table,
                                                 const int32_t* own_len, const void* h_plan,
                                                 const void* d_plan, void* workspace,
                                                 size_t workspace_bytes, void* stream) {
  const orion::NvtxRange nvtx_range("orion_point_prefill_attn");
  if (!out) return fail(ORION_ERR_INVALID_ARG, "null out");
  if (!h_plan || static_cast<const PlanHeader*>(h_plan)->magic != kPlanMagic ||
      static_cast<const PlanHeader*>(h_plan)->prefill_rows <= 0)
    return fail(ORION_ERR_INVALID_ARG, "orion_point_prefill_attn needs a point-prefill plan");
  // A prefill plan's items are reader-stationary (one partial per row): the split kernel writes
  // out / lse itself and no combine pass runs.
  const PlanHeader* h = nullptr;
  orion_status st = check_attn(shape, n_branches, h_plan, d_plan, workspace, workspace_bytes, &h);
  if (st != ORION_OK) return st;
  if (!q || !k_cache || !v_cache || !page_table || !own_len)
    return fail(ORION_ERR_INVALID_ARG, "null pointer");
  if (!aligned16(q) || !aligned16(k_cache) || !aligned16(v_cache) || !aligned16(out))
    return fail(ORION_ERR_INVALID_ARG, "device pointers must be 16-byte aligned");
  if (num_pages < 1) return fail(ORION_ERR_INVALID_ARG, "num_pages < 1");
  if (h->variant != kVariantTC) return fail(ORION_ERR_INVALID_ARG, "prefill plan with a decode kernel variant");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const char* dp = static_cast<const char*>(d_plan);
  if (shape->head_dim == 128)
    return launch_split<128>(h, dp, q, k_cache, v_cache, num_pages, page_table, own_len, workspace, s,
                             1 + shape->kv_interleaved, out, lse);
  return launch_split<64>(h, dp, q, k_cache, v_cache, num_pages, page_table, own_len, workspace, s,
                          1 + shape->kv_interleaved, out, lse);
}

extern "C" const char* orion_version(void) {
  return "orion-b200 0.5 (sm_100a; K1 append (fused into the split launch on short steps: orion_expand_step); K2 split: hybrid decode plans -- tcgen05.mma + TMEM + TMA swap-AB "
         "for items of <= 64 rows, rows-on-lanes tcgen05 for 65..128-row (masked) block items, two PDL-chained "
         "launches | rows-on-lanes (d = 64, point prefill; K/V-sharing item pairs with ORION_PLAN_PAIR) | "
         "mma.sync m16n8k16 (ORION_PLAN_MMA_SYNC); K3 combine)";
}
