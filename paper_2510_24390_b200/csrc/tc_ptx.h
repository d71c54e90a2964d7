// tc_ptx.h — PTX wrappers (mbarrier, TMA, tcgen05 MMA / commit / fences, UMMA descriptors) and
// the range geometry of multi-range work items, shared by the rows-on-lanes tcgen05 split kernels
// (split_tc.cu, split_pair.cu).  Product-side only.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

#include "plan_format.h"
#include "split_tc.h"

namespace orion {
namespace tc {

constexpr int kTok = 64;       // tokens per S tile / ring stage
constexpr int kBox = 16;       // token rows per TMA box of a partial tile

// ------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(
                   smem_u32(b)),
               "r"(bytes)
               : "memory");
}
// Blocking wait on a phase parity.  try_wait carries a suspend-time hint, so a waiting warp sleeps
// instead of spinning and resumes as soon as the phase completes.  Release builds wait without a
// bound; the debug builds (ORION_WATCHDOG: `make check`, `make trace`) trap after ~2^22 polls so a
// protocol bug shows up as a kernel error instead of a hung GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = smem_u32(b);
#ifdef ORION_WATCHDOG
  for (uint32_t spin = 0;; ++spin) {
#else
  for (;;) {
#endif
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity), "r"(20000u)
        : "memory");
    if (ok) return;
#ifdef ORION_WATCHDOG
    if (spin == (1u << 22))
      printf("orion watchdog: mbarrier wait blk %d warp %d lane %d bar smem 0x%x parity %u\n", blockIdx.x,
             threadIdx.x >> 5, threadIdx.x & 31, a, parity);
    if (spin > (1u << 22) + (1u << 20)) __trap();
#endif
  }
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
#ifdef ORION_TC_TRACE
#define TRACE_DECL unsigned long long tr_[12] = {0}; const unsigned long long tr_t0 = clock64();
#define TW(slot, stmt) do { const unsigned long long t_ = clock64(); stmt; tr_[slot] += clock64() - t_; } while (0)
#define TRACE_DUMP(role) do { if (blockIdx.x < 2 && (threadIdx.x & 31) == 0) printf( \
    "TRACE blk %d warp %2d %-8s tot %llu | %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu\n", blockIdx.x, \
    threadIdx.x >> 5, role, clock64() - tr_t0, tr_[0], tr_[1], tr_[2], tr_[3], tr_[4], tr_[5], tr_[6], tr_[7], \
    tr_[8], tr_[9], tr_[10], tr_[11]); } while (0)
#else
#define TRACE_DECL
#define TW(slot, stmt) stmt
#define TRACE_DUMP(role) do {} while (0)
#endif

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n .reg .b32 rx;\n .reg .pred px;\n elect.sync rx|px, %1;\n @px mov.s32 %0, 1;\n}\n"
      : "+r"(pred)
      : "r"(0xFFFFFFFFu));
  return pred != 0;
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
// tcgen05.cp 128x256b: 128 rows x 32 bytes of a shared-memory matrix (described like an MMA
// operand) into TMEM lanes 0..127, 8 columns.  Runs in the issuing thread's tcgen05 pipeline order
// with its MMAs (an MMA issued after it reads the copied data; one issued before it has read its
// own operands first), and tcgen05.commit tracks it.
__device__ __forceinline__ void tc_cp_128x256b(uint32_t taddr, uint64_t s_desc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n" ::"r"(taddr), "l"(s_desc) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// The same with an L2 cache policy (createpolicy), e.g. evict_first for a K/V stream read once.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// L2 eviction-priority hints: the split kernels' partials are written with evict_last so that
// the combine pass finds them in L2 (the K/V stream of the same launch would otherwise push them
// out to DRAM); `pol` from createpolicy.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_global_hint(__half* ptr, __half v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.b16 [%0], %1, %2;\n" ::"l"(ptr), "h"(__half_as_ushort(v)), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_global_hint(float* ptr, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;\n" ::"l"(ptr), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_global_hint(uint4* ptr, uint4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;\n" ::"l"(ptr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0));
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}
// acc + lo + hi of a packed bf16x2 word in fp32 without unpacking: two mixed-precision adds
// (add.rn.f32.bf16, sm_100; SASS FHADD.BF16 with a half selector) instead of shift, and, 2 FADD.
__device__ __forceinline__ float add_bf16x2_f32(uint32_t pk, float acc) {
  float r;
  asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %1;\n\tadd.rn.f32.bf16 %0, lo, %2;\n\t"
      "add.rn.f32.bf16 %0, hi, %0;\n\t}"
      : "=f"(r) : "r"(pk), "f"(acc));
  return r;
}
// Three-input max (sm_100 FMNMX3), and the max of N values as four independent FMNMX3 chains: a
// softmax row max in ~N/8 dependent steps instead of N (the latency of a 64-long fmaxf chain was a
// quarter of a tile's softmax time).  Same result as a sequential fmaxf fold (max is exact).
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
template <int N>
__device__ __forceinline__ float max_tree(const uint32_t (&v)[N]) {
  static_assert(N % 8 == 0, "max_tree: N multiple of 8");
  float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
#pragma unroll
  for (int c = 0; c < N; c += 8) {
    m0 = fmax3(m0, __uint_as_float(v[c]), __uint_as_float(v[c + 1]));
    m1 = fmax3(m1, __uint_as_float(v[c + 2]), __uint_as_float(v[c + 3]));
    m2 = fmax3(m2, __uint_as_float(v[c + 4]), __uint_as_float(v[c + 5]));
    m3 = fmax3(m3, __uint_as_float(v[c + 6]), __uint_as_float(v[c + 7]));
  }
  return fmaxf(fmax3(m0, m1, m2), m3);
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// UMMA shared-memory descriptor (sm_100 format, version 1), 128-byte swizzle.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;   // descriptor version (Blackwell)
  d |= static_cast<uint64_t>(2) << 61;   // SWIZZLE_128B
  return d;
}
// Instruction descriptor, kind::f16: bf16 A/B, fp32 D.
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n, bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

// Geometry of one token range of an item: the item itself, or range r of a multi-range item
// (kItemRanges, point-prefill plans).  Tiles sit on the 64-token grid of the range's page run.
struct RangeG {
  int32_t pt_off, t0, end, base, ntiles, causal, masked;
  uint32_t mask;   // kRangeMasked: bit i = the item's i-th reader reads this range
};
__device__ __forceinline__ int item_nranges(const WorkItem& w) {
  return (w.flags & kItemRanges) ? w.n_ranges : 1;
}
__device__ __forceinline__ RangeG range_geom(const TcArgs& a, const WorkItem& w, int r) {
  int32_t t1, dyn, fl;
  RangeG g;
  g.mask = 0xffffffffu;
  if (w.flags & kItemRanges) {
    const Range R = a.ranges[w.pt_off + r];
    g.pt_off = R.pt_off; g.t0 = R.t0; t1 = R.t1; dyn = R.dyn; fl = R.flags;
    if (fl & kRangeMasked) g.mask = static_cast<uint32_t>(R.pad_[0]);
  } else {
    g.pt_off = w.pt_off; g.t0 = w.t0; t1 = w.t1; dyn = w.dyn; fl = w.flags & ~kRangeMasked;
  }
  g.masked = (fl & kRangeMasked) != 0;
  g.end = t1;
  if (dyn >= 0) g.end = min(g.end, __ldg(a.own_len + dyn));
  g.base = g.t0 & ~(kTok - 1);
  g.ntiles = g.end > g.t0 ? (g.end - g.base + kTok - 1) / kTok : 0;
  g.causal = (fl & kItemCausal) != 0;
  return g;
}
__device__ __forceinline__ int item_tiles(const TcArgs& a, const WorkItem& w) {
  int n = 0;
  for (int r = 0; r < item_nranges(w); ++r) n += range_geom(a, w, r).ntiles;
  return n;
}

__device__ __forceinline__ int next_nonempty(const TcArgs& a, int it) {
  while (it < a.n_items && item_tiles(a, a.items[it]) == 0) it += gridDim.x;
  return it;
}

}  // namespace tc
}  // namespace orion
