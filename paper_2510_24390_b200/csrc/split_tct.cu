// split_tct.cu — K2 split attention, transposed ("swap-AB") tcgen05 formulation (default, d=128).
//
// Decode attention has few query rows per shared piece (G heads x the piece's readers: 4..64 in
// the paper's workloads) but long token runs.  Putting query rows on the MMA M dimension (the
// classic orientation, split_tc.cu) leaves most TMEM lanes / softmax threads idle and funnels the
// exponentials of a small item through one SM sub-partition.  Here tokens are the M dimension:
//
//   S^T[128 tok x N]  = K_tile[128 x d] . Q^T            (A = K smem K-major, B = Q smem K-major)
//   O^T[d x N]       += V_tile^T[d x 128] . P^T[128 x N] (A = V smem MN-major, B = P^T smem MN-major)
// with N = 16/32/64 (query rows, padded).  One softmax thread per token row of S^T; the two
// softmax warpgroups split every tile's columns (query rows) in half, so each thread handles N/2
// scores: a warpgroup-wide "is any running max unset or grown by > 2^8" vote (bar.red.or), and
// only on that rare path a column max (redux.sync.max.f32 + smem) that moves the reference and
// rescales this warpgroup's O^T columns.  Row sums l are accumulated per thread from the bf16 P
// and reduced over the 128 token rows at item end.  The exponentials of a tile are spread over all
// four sub-partitions whatever the row count.
//
// Roles (384 threads, one persistent CTA per SM, items strided over CTAs):
//   warp 0  TMEM allocation, then the V TMA producer (ring 3 x 32 KB, released at PV completion)
//   warp 1  per-CTA scheduler: item geometry into an 8-entry smem ring, Q rows gathered with
//           cp.async into a double buffer
//   warp 2  K TMA producer (ring 2 x 32 KB, released at QK completion)
//   warp 3  MMA issuer (QK up to three tiles ahead of PV; zeroes a partial tile's V edge rows once
//           the tile has landed, so 0 x NaN from never-written slots cannot reach O)
//   warps 4-7 / 8-11  softmax warpgroups 0 / 1 (query columns [0, N/2) / [N/2, N)); O^T is
//           double-buffered by item parity, so an item's epilogue (fp16 o = acc / l and fp32
//           log2-sum-exp per row, plan_format.h) overlaps the next item's first PVs.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <cstdio>

#include "../../include/orion.h"
#include "merge16.h"
#include "plan_format.h"
#include "split_tc.h"
#include "tc_ptx.h"
#include "tmem_ops.h"

namespace orion {
namespace tct {

constexpr int D = 128;
constexpr int kTok = 128;                 // tokens per tile = MMA M of S^T
constexpr int kBox = 16;                  // token rows of a partial-tile TMA box
constexpr int kSK = 2, kSV = 3;           // K / V ring depth (32 KB stages)
constexpr int kThreads = 384;
constexpr int kWarpAlloc = 0, kWarpSched = 1, kWarpTMA = 2, kWarpMMA = 3;
constexpr int kWarpTMAV = 0;              // the TMEM-alloc warp streams V once allocation is done
// TMEM columns
constexpr int kSB = 3;                    // S^T buffers: tile j uses j % 3
__device__ __forceinline__ uint32_t colS(uint32_t b) { return b * 64; }
__device__ __forceinline__ uint32_t colO(uint32_t i) { return 192 + i * 64; }   // O^T of item parity i

struct L {
  static constexpr int QB = 64 * D * 2;          // 16 KB: [2 halves][64 rows][128 B]
  static constexpr int HALF_Q = 64 * 128;
  static constexpr int KVB = kTok * D * 2;       // 32 KB: [2 halves][128 tokens][128 B]
  static constexpr int HALF_KV = kTok * 128;
  static constexpr int PB = kTok * 128;          // 16 KB: P^T [128 tokens][64 rows] bf16, MN-major
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = 2 * QB;
  static constexpr int OFF_V = OFF_K + kSK * KVB;
  static constexpr int OFF_P = OFF_V + kSV * KVB;
  // per-warpgroup column state, indexed by the warpgroup's local column (< 32): the column split
  // moves with npad from item to item while the two warpgroups may be on different tiles
  static constexpr int OFF_M = OFF_P + 2 * PB;      // running max m: [wg 2][32]
  static constexpr int OFF_SH = OFF_M + 2 * 32 * 4; // growth-path shifts: [wg 2][32]
  static constexpr int OFF_RED = OFF_SH + 2 * 32 * 4;  // growth-path column max scratch: [wg 2][4 warps][32]
  static constexpr int OFF_LI = OFF_RED + 2 * 4 * 32 * 4;  // 1 / l of the pending item: [wg 2][32]
  static constexpr int OFF_SCHED = OFF_LI + 2 * 32 * 4;    // item schedule ring: 8 x 64 B
  static constexpr int OFF_MI = OFF_SCHED + 8 * 64;        // MMA warp's entry geometry: 8 x 32 B
  static constexpr int OFF_BAR = OFF_MI + 8 * 32;
  static constexpr int N_BAR = 2 * kSK + 2 * kSV + 3 + 3 + 2 + 2 + 2 + 2 + 2 + 2 + 2 * 8;
  static constexpr int BYTES = OFF_BAR + N_BAR * 8 + 16;
};
static_assert(L::BYTES <= 232448, "shared memory budget");

// PTX helpers shared with the rows-on-lanes kernels (tc_ptx.h): mbarrier, TMA, tcgen05.
using tc::smem_u32;
using tc::mbar_init;
using tc::l2_policy_evict_last;
using tc::l2_policy_evict_first;
using tc::st_global_hint;
using tc::mbar_arrive;
using tc::mbar_expect_tx;
using tc::mbar_wait;
using tc::elect_one;
using tc::fence_proxy_async;
using tc::tc_fence_before;
using tc::tc_fence_after;
using tc::tc_commit;
using tc::tc_wait_ld;
using tc::tc_wait_st;
using tc::mma_ss;
using tc::tma_load_2d;
using tc::cp_async16;
using tc::ex2;
using tc::pack_bf16;
using tc::sw128_desc;

#undef TRACE_DECL
#undef TW
#undef TRACE_DUMP
#ifdef ORION_TC_TRACE
#define TRACE_DECL unsigned long long tr_[12] = {0}; const unsigned long long tr_t0 = clock64();
#define TRP tr_
#define TW(slot, stmt) do { const unsigned long long t_ = clock64(); stmt; tr_[slot] += clock64() - t_; } while (0)
#define TRACE_DUMP(role) do { if (blockIdx.x < 2 && (threadIdx.x & 31) == 0) printf( \
    "TRACE blk %d warp %2d %-8s tot %llu | %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu\n", blockIdx.x, \
    threadIdx.x >> 5, role, clock64() - tr_t0, tr_[0], tr_[1], tr_[2], tr_[3], tr_[4], tr_[5], tr_[6], tr_[7], \
    tr_[8], tr_[9], tr_[10], tr_[11]); } while (0)
#else
#define TRACE_DECL
#define TRP nullptr
#define TW(slot, stmt) stmt
#define TRACE_DUMP(role) do {} while (0)
#endif
#ifdef ORION_TC_TRACE
#define STW(slot, stmt) do { const unsigned long long t_ = clock64(); stmt; trp[slot] += clock64() - t_; } while (0)
#else
#define STW(slot, stmt) stmt
#endif

__device__ __forceinline__ float warp_max(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;\n" : "=f"(r) : "f"(v));
  return r;
}
// Block-level OR over the 128 threads of one softmax warpgroup (named barrier `id`).
__device__ __forceinline__ bool wg_any(bool v, int id) {
  int r;
  asm volatile("{\n .reg .pred a, b;\n setp.ne.s32 a, %1, 0;\n barrier.red.or.pred b, %2, 128, a;\n selp.s32 %0, 1, 0, b;\n}\n"
               : "=r"(r)
               : "r"(v ? 1 : 0), "r"(id)
               : "memory");
  return r != 0;
}
__device__ __forceinline__ void wg_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ uint32_t idesc(int n, bool a_mn, bool b_mn) {   // M = 128, bf16 -> fp32
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}

// Geometry of range r of an item (the item itself unless kItemRanges).
struct RangeT {
  int32_t pt_off, t0, end, base, ntiles, dyn;
};
// (a, b) += (lo, hi) of a packed bf16x2 word, each in fp32: bit-identical to unpacking and adding
// (bf16 -> f32 is exact), in two instructions (add.rn.f32.bf16 -> FHADD.BF16 with a half selector).
__device__ __forceinline__ void add_bf16x2_f32x2(uint32_t pk, float& a, float& b) {
  asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\tadd.rn.f32.bf16 %0, lo, %0;\n\t"
      "add.rn.f32.bf16 %1, hi, %1;\n\t}"
      : "+f"(a), "+f"(b) : "r"(pk));
}
__device__ __forceinline__ int item_nranges(const WorkItem& w) { return (w.flags & kItemRanges) ? w.n_ranges : 1; }
// Fused append: branch d's flag word carries (epoch + 1) << 20 | own_len once its append is done
// (12 epoch bits suffice: every fused launch rewrites every branch's flag; own_len < 2^20);
// the range reads its length from the flag (one acquire load: no separate own_len load), after
// which the appended K/V rows may be read.  Lane 0 spins; the warp follows.
__device__ __forceinline__ int appended_len(const TcArgs& a, int d, uint32_t seq) {
  int v = 0;
  if ((threadIdx.x & 31) == 0) {
    for (;;) {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(a.app.flags + d) : "memory");
      if ((static_cast<uint32_t>(v) >> 20) == (seq & 0xfffu)) break;
      __nanosleep(64);
    }
  }
  return __shfl_sync(0xffffffffu, v, 0) & 0xfffff;
}
__device__ __forceinline__ RangeT range_of(const TcArgs& a, const WorkItem& w, int r, uint32_t seq) {
  RangeT g;
  int32_t t1, dyn;
  if (w.flags & kItemRanges) {
    const Range R = a.ranges[w.pt_off + r];
    g.pt_off = R.pt_off; g.t0 = R.t0; t1 = R.t1; dyn = R.dyn;
  } else {
    g.pt_off = w.pt_off; g.t0 = w.t0; t1 = w.t1; dyn = w.dyn;
  }
  g.end = t1;
  g.dyn = dyn;
  if (dyn >= 0) {
    if (a.app.enabled) {
      g.end = min(g.end, appended_len(a, dyn, seq));   // written in this launch
    } else {
      g.end = min(g.end, __ldg(a.own_len + dyn));
    }
  }
  g.base = g.t0 & ~(kTok - 1);
  g.ntiles = g.end > g.t0 ? (g.end - g.base + kTok - 1) / kTok : 0;
  return g;
}
__device__ __forceinline__ int npad_of(int n_rows) { return n_rows <= 16 ? 16 : (n_rows <= 32 ? 32 : 64); }

// One softmax tile for one warpgroup's half of the query columns: thread t owns token row t of S^T
// and columns [c0, c0 + NH) (NH = padded query rows / 2); mrow / shs / red are this warpgroup's
// arrays indexed by local column.  Writes its columns of P^T row t; on the
// rare growth path (first tile of an item, or a running max grown by more than 2^8) it moves the
// per-column reference m and rescales its columns of O^T / L^T.
template <int NH>
__device__ __forceinline__ void softmax_tile(uint32_t tmem, uint32_t lane_base, int p, int t, uint32_t scol,
                                             uint8_t* pbuf, int c0, int tb, int lo, int hi, float* mrow,
                                             float* shs, float* red, bool had, uint32_t ocol, float (&ls)[NH],
                                             float scale_log2, uint64_t* sfree, bool need_pv, uint64_t* pv_free,
                                             uint32_t pv_free_par, uint64_t* pv_prev, uint32_t pv_prev_par,
                                             unsigned long long* trp) {
  uint32_t s[NH];
#ifdef ORION_TC_TRACE
  unsigned long long tq_ = clock64();
#define SLOT_END(i) do { trp[i] += clock64() - tq_; tq_ = clock64(); } while (0)
#else
#define SLOT_END(i) do {} while (0)
#endif
  if constexpr (NH == 8) tmem_ld32x8(tmem + lane_base + scol, s);
  if constexpr (NH == 16) tmem_ld32x16(tmem + lane_base + scol, s);
  if constexpr (NH == 32) tmem_ld32x32(tmem + lane_base + scol, s);
  tc_wait_ld();
  SLOT_END(7);
  tc_fence_before();
  mbar_arrive(sfree);                                // QK(j+3) may overwrite this S^T buffer
  const int pos = tb + t;
  const bool valid = pos >= lo && pos < hi;
  // d = s * scale - mb (log2 domain, relative to the per-column running reference mb).  On an
  // item's first tile (had == false) no column has a reference yet: d = s * scale, and the growth
  // path below always runs (every tile has a valid token), so no vote is needed.  Afterwards every
  // column has one, and the vote is "does any valid d exceed 2^8" -- a max, not per-element tests.
  bool grow = true;
  if (!had) {
#pragma unroll
    for (int c = 0; c < NH; ++c) s[c] = __float_as_uint(valid ? __uint_as_float(s[c]) * scale_log2 : -INFINITY);
  } else {
    float dmax = -INFINITY;
    if (valid) {
#pragma unroll
      for (int c4 = 0; c4 < NH; c4 += 4) {
        const float4 m4 = *reinterpret_cast<const float4*>(mrow + c4);
        const float mm[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) s[c4 + e] = __float_as_uint(fmaf(__uint_as_float(s[c4 + e]), scale_log2, -mm[e]));
      }
      dmax = tc::max_tree(s);
    } else {
#pragma unroll
      for (int c = 0; c < NH; ++c) s[c] = __float_as_uint(-INFINITY);
    }
    SLOT_END(3);
    grow = wg_any(dmax > 8.f, 2 + p);
    SLOT_END(8);
  }
  if (grow) {
    // column max of d over the 128 tokens: warp redux, then across the 4 warps via smem
    const int wq = t >> 5, ln = t & 31;
#pragma unroll
    for (int c = 0; c < NH; ++c) {
      const float wm = warp_max(__uint_as_float(s[c]));
      if (ln == (c & 31)) red[wq * 32 + c] = wm;
    }
    wg_sync(2 + p, 128);
    if (t < NH) {                                    // column owner: new reference and shift
      const int col = t;
      const float cm = fmaxf(fmaxf(red[col], red[32 + col]), fmaxf(red[64 + col], red[96 + col]));
      const float mo = mrow[col];
      const bool gc = cm > -INFINITY && (mo == -INFINITY || cm > 8.f);
      const float mb = mo == -INFINITY ? 0.f : mo;
      shs[col] = gc ? cm : 0.f;
      if (gc) mrow[col] = mb + cm;
    }
    wg_sync(2 + p, 128);
#pragma unroll
    for (int c = 0; c < NH; ++c) s[c] = __float_as_uint(__uint_as_float(s[c]) - shs[c]);   // d relative to the new reference
    if (had) {   // this item's O^T columns and row sums follow the new reference: * 2^-shift
#pragma unroll
      for (int c = 0; c < NH; ++c) ls[c] *= ex2(-shs[c]);
      mbar_wait(pv_prev, pv_prev_par);             // O^T has absorbed PV(j-1)
      tc_fence_after();
#pragma unroll
      for (int cb = 0; cb < NH; cb += 8) {
        uint32_t o[8];
        tmem_ld32x8(tmem + lane_base + ocol + cb, o);
        tc_wait_ld();
#pragma unroll
        for (int c = 0; c < 8; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * ex2(-shs[cb + c]));
        tmem_st32x8(tmem + lane_base + ocol + cb, o);
      }
      tc_wait_st();
    }
  }
  // P^T row t, columns [c0, c0 + NH) (MN-major, 128B swizzle): p = 2^(d - shift) rounded to bf16.
  // The exponentials are formed before the wait for PV(j-2), which frees this P^T buffer.
  SLOT_END(10);
  uint32_t pk[NH / 2];
#pragma unroll
  for (int c = 0; c < NH; c += 2) pk[c / 2] = pack_bf16(ex2(__uint_as_float(s[c])), ex2(__uint_as_float(s[c + 1])));
#pragma unroll
  for (int c = 0; c < NH; c += 2)                    // row sums of exactly the bf16 P fed to PV
    add_bf16x2_f32x2(pk[c / 2], ls[c], ls[c + 1]);
  SLOT_END(9);
  if (need_pv) STW(6, mbar_wait(pv_free, pv_free_par));
#pragma unroll
  for (int cc = 0; cc < NH / 8; ++cc) {
    const int chunk = (c0 >> 3) + cc;
    *reinterpret_cast<uint4*>(pbuf + t * 128 + ((chunk ^ (t & 7)) << 4)) =
        make_uint4(pk[cc * 4 + 0], pk[cc * 4 + 1], pk[cc * 4 + 2], pk[cc * 4 + 3]);
  }
}

// Per-CTA item schedule entry, produced by the scheduler warp (warp 1) and consumed in order by
// the TMA, MMA and both softmax warpgroups (removes the dependent global loads of the item
// descriptors from every role's critical path).
// One entry per token range: an item is one range, or (kItemRanges) a list of ranges streamed as
// one accumulation.  `item` numbers the CTA's non-empty items (Q / O^T double-buffer parity);
// `first` / `last` mark an item's first and last non-empty range.
// K1 inside the split launch (FusedAppend), before the CTA's roles start: warp w appends the
// new-token K/V rows of branches blockIdx.x + (w + 12 i) gridDim.x exactly as kv_append_kernel
// does (ADVANCE: slot own_len, then own_len + 1; REWRITE: slot own_len - 1; no write ever leaves
// the caches) and releases the branch's flag.  One warp per branch keeps the dependent
// own_len -> page -> copy chains of a CTA's branches in parallel; no grid-wide barrier follows
// (a count of CTAs done, polled by every item with a growing range, measured 4 % slower on c4's
// 8-query share than the separate append kernel).
constexpr int kAppendWarps = kThreads / 32;
__device__ __forceinline__ void fused_append(const TcArgs& a, int sw, int lane) {
  constexpr int CH = D / 8;
  const FusedAppend& ap = a.app;
  const uint32_t seq = static_cast<uint32_t>(__ldcg(ap.epoch)) + 1u;
  for (int b = blockIdx.x + sw * gridDim.x; b < ap.n_branches; b += kAppendWarps * gridDim.x) {
    const int len = __ldcg(ap.own_len + b);
    const int pos = ap.mode == ORION_APPEND_REWRITE ? len - 1 : len;
    const bool ok = pos >= 0 && pos < __ldg(ap.own_cap + b);
    int page = ok ? __ldg(a.page_table + __ldg(ap.own_pt_off + b) + (pos >> a.page_shift)) : -1;
    if (page >= ap.num_pages || (ok && page < 0)) {
      if (ap.err && lane == 0) atomicCAS(ap.err, 0, b + 1);
      page = -1;
    }
    if (page >= 0) {
      const size_t row = static_cast<size_t>(pos & ((1 << a.page_shift) - 1)) * D;
      for (int i = lane; i < a.hkv * CH; i += 32) {
        const int g = i / CH, c = i % CH;
        const size_t dst = (((static_cast<size_t>(page) * a.hkv + g) * a.kvs) << a.page_shift) * D + row + c * 8;
        const size_t src = (static_cast<size_t>(b) * a.hkv + g) * D + c * 8;
        *reinterpret_cast<uint4*>(ap.k_cache + dst) = *reinterpret_cast<const uint4*>(ap.k_new + src);
        *reinterpret_cast<uint4*>(ap.v_cache + dst) = *reinterpret_cast<const uint4*>(ap.v_new + src);
      }
    }
    // ADVANCE moves own_len only when the slot was written (as kv_append_kernel)
    const int nlen = (page >= 0 && ap.mode == ORION_APPEND_ADVANCE) ? len + 1 : len;
    __syncwarp();                                   // the warp's row copies issued
    if (lane == 0) {
      if (nlen != len) ap.own_len[b] = nlen;
      asm volatile("fence.proxy.async.global;\n" ::: "memory");   // generic K/V writes vs TMA reads
      __threadfence();
      asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(ap.flags + b),
                   "r"(static_cast<int>((seq & 0xfffu) << 20) | (nlen & 0xfffff))
                   : "memory");
    }
  }
}

struct Sched {
  int32_t valid, it, pt_off, t0, end, base, ntiles, npad, kv_head, n_rows, slot0, item, first, last;
  int32_t appended;   // the range may hold rows the fused append wrote in this launch
  int32_t pad;
};
constexpr int kSched = 8;
constexpr uint32_t kSchedConsumers = 1 + 1 + 1 + 128 + 128;   // K-TMA, V-TMA, MMA lanes, WG0, WG1

__device__ __forceinline__ Sched read_sched(const Sched* ring, uint64_t* full, uint64_t* empty, uint32_t k,
                                            bool arrive) {
  mbar_wait(full + (k % kSched), (k / kSched) & 1);
  const Sched e = ring[k % kSched];
  if (arrive) mbar_arrive(empty + (k % kSched));
  return e;
}

// Barrier block layout (shared by the kernel and softmax_item).
struct Bars {
  uint64_t *k_full, *k_empty, *v_full, *v_empty, *s_full, *s_free, *p_full, *pv_done, *q_full, *q_empty,
      *o_free, *acc_full, *sch_full, *sch_empty;
};
__device__ __forceinline__ Bars carve_bars(uint8_t* smem) {
  uint64_t* b = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  Bars r;
  // Every waiter consumes the phases of each barrier in order (both softmax warpgroups take part
  // in every tile), so no phase-parity wait can run two phases ahead and alias.
  r.k_full = b; r.k_empty = b + kSK;
  r.v_full = r.k_empty + kSK; r.v_empty = r.v_full + kSV;
  r.s_full = r.v_empty + kSV;                       // [3]: S^T of tile j in buffer j % 3
  r.s_free = r.s_full + kSB;                        // [3]: S^T buffer read by both warpgroups
  r.p_full = r.s_free + kSB;                        // [2]: P^T[j & 1] written by both warpgroups
  r.pv_done = r.p_full + 2;                         // [2]: PV(j) complete
  r.q_full = r.pv_done + 2; r.q_empty = r.q_full + 2;
  r.o_free = r.q_empty + 2;                         // [2]: epilogue of the item using O^T[i] done
  r.acc_full = r.o_free + 2;                        // [2]: last PV into O^T[i] complete
  r.sch_full = r.acc_full + 2; r.sch_empty = r.sch_full + kSched;
  return r;
}

// A finished item whose O^T readout is deferred: its last PV completes while the next item's first
// tile is processed (O^T is double-buffered by item parity; the MMA reuses this buffer only after
// o_free).  Its lse is already written and its 1 / l per column sits in the warpgroup's `linv`.
struct Pend {
  int32_t valid, slot0, n_rows, nh, kp, item;
};

// The deferred part of an item's epilogue: fp16 o = acc / l from O^T (plan_format.h), then
// o_free.  Runs after the next item's first tile (or at the very end).  linv was written before a
// warpgroup barrier (the next item's start) and is rewritten only after the next item's
// end-of-item barrier, which every thread reaches after this readout: no barrier needed here.
__device__ __forceinline__ void finish_item(const Pend& pd, uint32_t tmem, uint32_t lane_base, int p, int t,
                                            const float* linv, const Bars& B, const TcArgs& a,
                                            unsigned long long* trp) {
  const int c0 = p * pd.nh;
  STW(5, mbar_wait(B.acc_full + pd.kp, (static_cast<uint32_t>(pd.item) >> 1) & 1));
  tc_fence_after();
  __half* dst = a.part_o + static_cast<size_t>(pd.slot0) * D + t;
  const uint64_t pol = l2_policy_evict_last();
  for (int cb = 0; cb < pd.nh; cb += 8) {
    uint32_t o[8];
    tmem_ld32x8(tmem + lane_base + colO(pd.kp) + c0 + cb, o);
    tc_wait_ld();
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c0 + cb + c < pd.n_rows)
        st_global_hint(dst + static_cast<size_t>(c0 + cb + c) * D, __float2half_rn(__uint_as_float(o[c]) * linv[cb + c]), pol);
  }
  tc_fence_before();
  mbar_arrive(B.o_free + pd.kp);
}

// All tiles of one item for one softmax warpgroup (query columns [p*NH, (p+1)*NH)), then its
// share of the item's partial: acc from O^T, m from mrow, l from the per-thread row sums reduced
// over the 128 token rows.
template <int NH>
__device__ __forceinline__ void softmax_item(uint8_t* smem, uint32_t tmem, uint32_t lane_base, int p, int t,
                                             const Sched& e, uint32_t& k, uint32_t& j, float* mrow, float* shs,
                                             float* red, float* linv, const Bars& B, const TcArgs& a,
                                             const Sched* ring, Pend& pend, unsigned long long* trp) {
  // `e` is the item's first ring entry (k); its further ranges are the next entries, read here.
  const int c0 = p * NH;
  const uint32_t kp = static_cast<uint32_t>(e.item) & 1;
  float ls[NH];
#pragma unroll
  for (int c = 0; c < NH; ++c) ls[c] = 0.f;
  if (t < NH) mrow[t] = -INFINITY;
  wg_sync(2 + p, 128);
  Sched cur = e;
  for (int tt = 0, t_in = 0;; ++tt, ++t_in, ++j) {
    if (t_in == cur.ntiles) {                       // next range of the same item
      if (cur.last) break;
      ++k;
      cur = read_sched(ring, B.sch_full, B.sch_empty, k, true);
      t_in = 0;
    }
    const int tb = cur.base + t_in * kTok;
    const int lo = max(tb, cur.t0), hi = min(tb + kTok, cur.end);
    const uint32_t b = j % kSB;
    STW(1, mbar_wait(B.s_full + b, (j / kSB) & 1));
    tc_fence_after();
#ifdef ORION_TC_TRACE
    const unsigned long long ts_ = clock64();
#endif
    uint8_t* pbuf = smem + L::OFF_P + (j & 1) * L::PB;
    const bool need_pv = j >= 2;                    // P^T[j & 1] still feeds PV(j-2)
    softmax_tile<NH>(tmem, lane_base, p, t, colS(b) + c0, pbuf, c0, tb, lo, hi, mrow, shs, red, tt > 0,
                     colO(kp) + c0, ls, a.scale_log2, B.s_free + b, need_pv, B.pv_done + (j & 1),
                     ((j - 2) >> 1) & 1, B.pv_done + ((j - 1) & 1), ((j - 1) >> 1) & 1, trp);
#ifdef ORION_TC_TRACE
    const unsigned long long tf_ = clock64();
#endif
    fence_proxy_async();
    tc_fence_before();
    mbar_arrive(B.p_full + (j & 1));
#ifdef ORION_TC_TRACE
    trp[11] += clock64() - tf_;
    trp[2] += clock64() - ts_;
    trp[0] += 1;
#endif
    if (tt == 0 && pend.valid) {                    // the previous item's deferred readout
      finish_item(pend, tmem, lane_base, p, t, linv, B, a, trp);
      pend.valid = 0;
    }
  }
#ifdef ORION_TC_TRACE
  const unsigned long long te_ = clock64();
#endif
  // ---- epilogue.  l: butterfly over the warp (plain levels while more lanes than columns, then a
  // reduce-scatter leaving column ln % NH in lane ln), then across the 4 warps via red.
  const int ln = t & 31, wq = t >> 5;
#pragma unroll
  for (int off = 16; off >= NH; off >>= 1)
#pragma unroll
    for (int c = 0; c < NH; ++c) ls[c] += __shfl_xor_sync(0xffffffffu, ls[c], off);
#pragma unroll
  for (int off = (NH >= 32 ? 16 : NH / 2), n = (NH >= 32 ? 32 : NH); off >= 1; off >>= 1, n >>= 1) {
    const bool up = (ln & off) != 0;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const float send = up ? ls[i] : ls[i + n / 2];
      const float keep = up ? ls[i + n / 2] : ls[i];
      ls[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  if (ln < NH) red[wq * 32 + ln] = ls[0];
  wg_sync(2 + p, 128);
  // fp16 partial format (plan_format.h): o = acc / l, lse2 = m + log2 l.  l >= 1: the column max
  // that set the reference contributes 2^0 (every item has at least one valid token).  The O^T
  // readout waits for the item's last PV: deferred to the next item's first tile (Pend).
  if (t < NH) {
    const float l = red[t] + red[32 + t] + red[64 + t] + red[96 + t];
    linv[t] = 1.f / l;
    if (c0 + t < e.n_rows) st_global_hint(a.part_lse + e.slot0 + c0 + t, mrow[t] + log2f(l), l2_policy_evict_last());
  }
  pend.valid = 1;
  pend.slot0 = e.slot0; pend.n_rows = e.n_rows; pend.nh = NH; pend.kp = static_cast<int32_t>(kp);
  pend.item = e.item;
#ifdef ORION_TC_TRACE
  trp[4] += clock64() - te_;
#endif
}

__global__ void __launch_bounds__(kThreads, 1)
    split_tct_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                     const __grid_constant__ CUtensorMap tmK16, const __grid_constant__ CUtensorMap tmV16,
                     const TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const Bars bars = carve_bars(smem);
  uint64_t *k_full = bars.k_full, *k_empty = bars.k_empty, *v_full = bars.v_full, *v_empty = bars.v_empty;
  uint64_t *s_full = bars.s_full, *s_free = bars.s_free, *p_full = bars.p_full, *pv_done = bars.pv_done;
  uint64_t *q_full = bars.q_full, *q_empty = bars.q_empty, *o_free = bars.o_free, *acc_full = bars.acc_full;
  uint64_t *sch_full = bars.sch_full, *sch_empty = bars.sch_empty;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sch_empty + kSched);
  Sched* ring = reinterpret_cast<Sched*>(smem + L::OFF_SCHED);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kSK; ++s) { mbar_init(k_full + s, 1); mbar_init(k_empty + s, 1); }
    for (int s = 0; s < kSV; ++s) { mbar_init(v_full + s, 1); mbar_init(v_empty + s, 1); }
    for (int b = 0; b < kSB; ++b) { mbar_init(s_full + b, 1); mbar_init(s_free + b, 256); }
    for (int b = 0; b < 2; ++b) {
      mbar_init(p_full + b, 256); mbar_init(pv_done + b, 1); mbar_init(q_full + b, 1);
      mbar_init(q_empty + b, 1); mbar_init(o_free + b, 256); mbar_init(acc_full + b, 1);
    }
    for (int b = 0; b < kSched; ++b) { mbar_init(sch_full + b, 1); mbar_init(sch_empty + b, kSchedConsumers); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmK)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmV)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmK16)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmV16)) : "memory");
  }
  // V ring starts zeroed: rows a partial tile's boxes never cover must be finite (their P is 0)
  for (int i = tid; i < kSV * L::KVB / 16; i += kThreads)
    reinterpret_cast<uint4*>(smem + L::OFF_V)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  if (warp == kWarpAlloc) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  // KV appended / previous step's reads done.  A hybrid plan's second kernel (pdl_late) was
  // launched only once the first had passed this wait, so it defers its own wait to the end.
  if (!a.pdl_late) pdl_wait();
  if (a.app.enabled) fused_append(a, warp, lane);
  const int n_items = a.n_items;

  TRACE_DECL
  if (warp == kWarpSched) {
    // ------------------------------------------------------------------ scheduler + Q gather
    uint32_t k = 0;                                 // ring entries published (one per range)
    uint32_t iq = 0;                                // non-empty items of this CTA
    // fused append: this launch's flag epoch (every CTA reads the value the previous fused
    // launch's last CTA left)
    const uint32_t seq = a.app.enabled ? static_cast<uint32_t>(__ldcg(a.app.epoch)) + 1u : 0u;
    // Items are handed out by an atomic counter (zeroed by the launcher) in the planner's
    // longest-first order: greedy LPT over the SMs.  A static stride left the busiest SM ~5 %
    // above the mean (ncu sm__cycles_active max / avg on c4).
    for (;;) {
      int it = 0;
      if (lane == 0) it = atomicAdd(a.work_counter, 1);
      it = __shfl_sync(0xffffffffu, it, 0);
      if (it >= n_items) break;
      const WorkItem w = a.items[it];
      const int nr = item_nranges(w);
      int rfirst = -1, rlast = -1;
      RangeT g0 = range_of(a, w, 0, seq);
      if (nr == 1) {                                 // the common single-range item: one lookup
        if (g0.ntiles > 0) rfirst = rlast = 0;
      } else {
        for (int r = 0; r < nr; ++r)
          if (range_of(a, w, r, seq).ntiles > 0) { if (rfirst < 0) rfirst = r; rlast = r; }
      }
      if (rfirst < 0) {                              // every range empty (dyn end <= t0): neutral partial
        for (int i = lane; i < w.n_rows * D / 8; i += 32)
          reinterpret_cast<uint4*>(a.part_o + static_cast<size_t>(w.slot0) * D)[i] = make_uint4(0, 0, 0, 0);
        for (int r = lane; r < w.n_rows; r += 32) a.part_lse[w.slot0 + r] = -INFINITY;
        continue;
      }
      for (int r = rfirst; r <= rlast; ++r) {
        const RangeT g = nr == 1 ? g0 : range_of(a, w, r, seq);
        if (g.ntiles == 0) continue;
        TW(0, mbar_wait(sch_empty + (k % kSched), ((k / kSched) & 1) ^ 1));
        if (lane == 0) {
          Sched e;
          e.valid = 1; e.it = it; e.pt_off = g.pt_off; e.t0 = g.t0; e.end = g.end; e.base = g.base;
          e.ntiles = g.ntiles; e.npad = npad_of(w.n_rows); e.kv_head = w.kv_head; e.n_rows = w.n_rows;
          e.slot0 = w.slot0; e.item = static_cast<int32_t>(iq); e.first = r == rfirst; e.last = r == rlast;
          e.appended = g.dyn >= 0 && a.app.enabled;
          ring[k % kSched] = e;
          mbar_arrive(sch_full + (k % kSched));
        }
        ++k;
        if (r != rfirst) continue;
        // Q rows of item iq -> Q buffer iq & 1, once item iq-2's QKs have completed
        if (iq >= 2) TW(1, mbar_wait(q_empty + (iq & 1), ((iq >> 1) - 1) & 1));
        uint8_t* qb = smem + L::OFF_Q + (iq & 1) * L::QB;
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int rw = lane + rr * 32;
          const bool ok = rw < w.n_rows;
          const __nv_bfloat16* src = a.q;
          if (ok) {
            const int row = w.row_begin + rw;
            const int b = __ldg(a.readers + w.readers_off + row / a.group);
            const int hq = w.kv_head * a.group + row % a.group;
            src = a.q + (static_cast<size_t>(b) * a.hq + hq) * D;
          }
#pragma unroll
          for (int c = 0; c < 16; ++c)
            cp_async16(smem_u32(qb + (c >> 3) * L::HALF_Q + rw * 128 + (((c & 7) ^ (rw & 7)) << 4)),
                       ok ? static_cast<const void*>(src + c * 8) : static_cast<const void*>(a.q), ok);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(q_full + (iq & 1));
      }
      ++iq;
    }
    TW(0, mbar_wait(sch_empty + (k % kSched), ((k / kSched) & 1) ^ 1));
    if (lane == 0) {                                 // terminator
      ring[k % kSched].valid = 0;
      mbar_arrive(sch_full + (k % kSched));
    }
  } else if (warp == kWarpTMA || warp == kWarpTMAV) {
    // ------------------------------------------------------------------ TMA producers
    // warp 2 streams K tiles (released at QK completion), warp 0 streams V tiles (released at PV
    // completion): the two rings never block each other.
    const bool isk = warp == kWarpTMA;
    const int nst = isk ? kSK : kSV;
    uint64_t* full = isk ? k_full : v_full;
    uint64_t* empty = isk ? k_empty : v_empty;
    const CUtensorMap* mbig = isk ? &tmK : &tmV;
    const CUtensorMap* msml = isk ? &tmK16 : &tmV16;
    const uint32_t base_off = isk ? L::OFF_K : L::OFF_V;
    uint32_t j = 0;
    const int pmask = (1 << a.page_shift) - 1;
    const int big = min(64, 1 << a.page_shift);     // rows of a full-tile box (<= one page)
    // A swap-AB item reads its K/V chunk once (a reader block carries all rows of its query that
    // read it), so the stream is marked evict_first: it no longer pushes the partials (evict_last)
    // and the rows-on-lanes kernel's L2-shared prefixes out of L2.  c4 +1.6 %, its 8-query share
    // +8 %, c5 wide +5 % same-box; the rows-on-lanes kernel keeps the default policy (its items
    // share prefixes through L2: evict_first there cost the point prefill 14 %).
    const uint64_t kv_pol = l2_policy_evict_first();
    bool fenced = false;
    for (uint32_t k = 0;; ++k) {
      const Sched e = read_sched(ring, sch_full, sch_empty, k, lane == 0);
      if (e.valid && e.appended && !fenced) {   // rows other CTAs appended (generic writes) -> TMA reads
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        fenced = true;
      }
      if (!e.valid) break;
      for (int tb0 = 0; tb0 < e.ntiles; tb0 += 32) {
        int brow[8];
        int nbox = 0, first_off = 0, full_t = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) brow[b] = 0;
        if (tb0 + lane < e.ntiles) {
          const int a0 = e.base + (tb0 + lane) * kTok;
          const int lo = max(a0, e.t0), hi = min(a0 + kTok, e.end);
          full_t = (lo == a0 && hi == a0 + kTok);
          int pos0, step;
          if (full_t) { nbox = kTok / big; pos0 = a0; step = big; }
          else { pos0 = lo & ~(kBox - 1); nbox = (hi - pos0 + kBox - 1) / kBox; step = kBox; first_off = pos0 - a0; }
#pragma unroll
          for (int b = 0; b < 8; ++b)
            if (b < nbox) {
              const int pos = pos0 + b * step;
              const int page = __ldg(a.page_table + e.pt_off + (pos >> a.page_shift));
              brow[b] = (((page * a.hkv + e.kv_head) * a.kvs) << a.page_shift) + (pos & pmask);
            }
        }
        const int tend = min(e.ntiles, tb0 + 32);
        for (int tt = tb0; tt < tend; ++tt, ++j) {
          const int src = tt - tb0;
          const int tn = __shfl_sync(0xffffffffu, nbox, src);
          const int tf = __shfl_sync(0xffffffffu, full_t, src);
          const int to = __shfl_sync(0xffffffffu, first_off, src);
          int rr[8];
#pragma unroll
          for (int b = 0; b < 8; ++b) rr[b] = __shfl_sync(0xffffffffu, brow[b], src);
          const int st = j % nst;
          const int rpb = tf ? big : kBox;
          const uint32_t bytes = static_cast<uint32_t>(tn * rpb * 128 * 2);
          const CUtensorMap* m = tf ? mbig : msml;
          TW(0, mbar_wait(empty + st, ((j / nst) & 1) ^ 1));
          if (elect_one()) {
            mbar_expect_tx(full + st, bytes);
            const uint32_t dst = smem_u32(smem + base_off + st * L::KVB);
#pragma unroll
            for (int b = 0; b < 8; ++b)
              if (b < tn) {
                const uint32_t roff = static_cast<uint32_t>(to + b * rpb) * 128;
                tma_load_2d(dst + roff, m, 0, rr[b], full + st, kv_pol);
                tma_load_2d(dst + L::HALF_KV + roff, m, 64, rr[b], full + st, kv_pol);
              }
          }
          __syncwarp();
        }
      }
    }
    TRACE_DUMP("producer");
  } else if (warp == kWarpMMA) {
    // ------------------------------------------------------------------ MMA issuer
    // Item k is owned by softmax warpgroup k & 1 (accumulators O^T/L^T[k & 1]).  QK runs up to
    // three tiles ahead of PV (three S^T buffers) and never into item k+2 before every PV of item
    // k is issued (item k+2 reuses item k's Q buffer).  A polling loop issues a PV as soon as its
    // P is published, otherwise a QK whose operands are resident, otherwise sleeps on the oldest
    // dependency.
    const uint64_t dq0 = sw128_desc(smem_u32(smem + L::OFF_Q), 16, 1024);
    const uint64_t dk0 = sw128_desc(smem_u32(smem + L::OFF_K), 16, 1024);
    const uint64_t dv0 = sw128_desc(smem_u32(smem + L::OFF_V), L::HALF_KV, 1024);   // MN-major A
    const uint64_t dp0 = sw128_desc(smem_u32(smem + L::OFF_P), L::HALF_KV, 1024);   // MN-major B
    // geometry of ring entries k % 8: QK is at most four tiles (so four entries) past PV, plus
    // the entry it has read ahead
    int32_t* mi = reinterpret_cast<int32_t*>(smem + L::OFF_MI);   // [8][8]: t0 end base ntiles npad item first last
    auto set_of = [&](uint32_t k, const Sched& e) {
      if (lane == 0) {
        int32_t* r = mi + (k & 7) * 8;
        r[0] = e.t0; r[1] = e.end; r[2] = e.base; r[3] = e.ntiles; r[4] = e.npad;
        r[5] = e.item; r[6] = e.first; r[7] = e.last;
      }
      __syncwarp();
    };
    auto nt_of = [&](uint32_t k) { return mi[(k & 7) * 8 + 3]; };
    auto np_of = [&](uint32_t k) { return mi[(k & 7) * 8 + 4]; };
    auto item_of = [&](uint32_t k) { return static_cast<uint32_t>(mi[(k & 7) * 8 + 5]); };
    uint32_t q_item = 0, v_item = 0;                // item numbers of the QK / PV cursors' entries
    auto first_of = [&](uint32_t k) { return mi[(k & 7) * 8 + 6] != 0; };
    auto last_of = [&](uint32_t k) { return mi[(k & 7) * 8 + 7] != 0; };
    uint32_t kq = 0, tq = 0, jq = 0;                // QK cursor (item, tile in item, global tile)
    uint32_t kv = 0, tv = 0, jv = 0;                // PV cursor
    bool q_live;
    {
      const Sched e = read_sched(ring, sch_full, sch_empty, 0, lane == 0);
      q_live = e.valid;
      set_of(0, e);
      q_item = v_item = static_cast<uint32_t>(e.item);
    }
    auto issue_qk = [&]() {
      const uint32_t j = jq;
      const uint32_t iqq = item_of(kq);
      if (tq == 0 && first_of(kq)) TW(1, mbar_wait(q_full + (iqq & 1), (iqq >> 1) & 1));
      const int s = j % kSK;
      TW(2, mbar_wait(k_full + s, (j / kSK) & 1));
      if (j >= static_cast<uint32_t>(kSB)) TW(3, mbar_wait(s_free + (j % kSB), ((j - kSB) / kSB) & 1));
      tc_fence_after();
      const int ntq = nt_of(kq);
      const uint64_t dq = dq0 + static_cast<uint64_t>(((iqq & 1) * L::QB) >> 4);
      const uint64_t dk = dk0 + static_cast<uint64_t>((s * L::KVB) >> 4);
      const uint32_t id = idesc(np_of(kq), false, false);
#ifdef ORION_TC_TRACE
      const unsigned long long tq0 = clock64();
#endif
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint64_t ok = static_cast<uint64_t>(((ks >> 2) * L::HALF_KV + (ks & 3) * 32) >> 4);
          const uint64_t oq = static_cast<uint64_t>(((ks >> 2) * L::HALF_Q + (ks & 3) * 32) >> 4);
          mma_ss(tmem + colS(j % kSB), dk + ok, dq + oq, id, ks > 0);
        }
        tc_commit(s_full + (j % kSB));
        tc_commit(k_empty + s);
        if (static_cast<int>(tq) + 1 == ntq && last_of(kq)) tc_commit(q_empty + (iqq & 1));   // item's last QK
      }
      __syncwarp();
#ifdef ORION_TC_TRACE
      tr_[8] += clock64() - tq0;
#endif
      ++jq;
      if (static_cast<int>(++tq) == ntq) {
        tq = 0;
        ++kq;
        Sched e;
        TW(7, e = read_sched(ring, sch_full, sch_empty, kq, lane == 0));
        q_live = e.valid;
        set_of(kq, e);
        if (e.valid) q_item = static_cast<uint32_t>(e.item);
      }
    };
    auto issue_pv = [&]() {
      const uint32_t j = jv;
      const int s = j % kSV;
      const uint32_t ivv = item_of(kv);
      const uint32_t wg = ivv & 1;                  // accumulator of item ivv
      TW(6, mbar_wait(v_full + s, (j / kSV) & 1));
#ifdef ORION_TC_TRACE
      const unsigned long long tz0 = clock64();
#endif
      {
        // A partial tile's TMA boxes (16-row granular) may carry rows outside [t0, end) -- e.g.
        // never-written slots past own_len.  Their P is exactly 0, but 0 x NaN is NaN: zero them.
        const int32_t* r = mi + (kv & 7) * 8;
        const int a0 = r[2] + static_cast<int>(tv) * kTok;
        const int lo = max(a0, r[0]) - a0, hi = min(a0 + kTok, r[1]) - a0;
        if (lo > 0 || hi < kTok) {
          const int z0 = lo & ~(kBox - 1), z1 = min(kTok, (hi + kBox - 1) & ~(kBox - 1));
          uint8_t* vs = smem + L::OFF_V + s * L::KVB;
          const int nz = (lo - z0) + (z1 - hi);
          for (int i = lane; i < nz * 16; i += 32) {
            const int zr = i >> 4, c = i & 15;
            const int row = zr < lo - z0 ? z0 + zr : hi + (zr - (lo - z0));
            *reinterpret_cast<uint4*>(vs + (c >> 3) * L::HALF_KV + row * 128 + (c & 7) * 16) = make_uint4(0, 0, 0, 0);
          }
          fence_proxy_async();
          __syncwarp();
        }
      }
#ifdef ORION_TC_TRACE
      tr_[0] += clock64() - tz0;
#endif
      TW(4, mbar_wait(p_full + (j & 1), (j >> 1) & 1));
      if (tv == 0 && first_of(kv) && ivv >= 2) TW(5, mbar_wait(o_free + wg, ((ivv >> 1) - 1) & 1));   // item ivv-2 read out
      tc_fence_after();
      const uint64_t dv = dv0 + static_cast<uint64_t>((s * L::KVB) >> 4);
      const uint64_t dp = dp0 + static_cast<uint64_t>(((j & 1) * L::PB) >> 4);
      const int npv = np_of(kv);
      const uint32_t id_pv = idesc(npv, true, true);
      const bool first = tv == 0 && first_of(kv);   // the item's first tile: O^T = P V (no accumulate)
#ifdef ORION_TC_TRACE
      const unsigned long long tp0 = clock64();
#endif
      if (elect_one()) {
#pragma unroll
        for (int kt = 0; kt < kTok / 16; ++kt) {
          const uint64_t o = static_cast<uint64_t>((kt * 16 * 128) >> 4);
          const uint32_t acc = (!first || kt > 0) ? 1u : 0u;
          mma_ss(tmem + colO(wg), dv + o, dp + o, id_pv, acc);
        }
        tc_commit(pv_done + (j & 1));
        tc_commit(v_empty + s);
        if (static_cast<int>(tv) + 1 == nt_of(kv) && last_of(kv)) tc_commit(acc_full + wg);   // item complete
      }
      __syncwarp();
#ifdef ORION_TC_TRACE
      tr_[9] += clock64() - tp0;
#endif
      ++jv;
      if (static_cast<int>(++tv) == nt_of(kv)) {
        tv = 0;
        ++kv;
        if (kv < kq || (kv == kq && q_live)) v_item = item_of(kv);
      }
    };
    // in-order: keep QK up to 3 tiles ahead (never into item kv+2), then one PV
    while (true) {
      while (q_live && jq <= jv + 3 && q_item <= v_item + 1) issue_qk();
      const bool v_live = kv < kq || (kv == kq && q_live);
      if (!v_live) break;
      issue_pv();
    }
    TRACE_DUMP("mma");
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ softmax / epilogue
    // Both warpgroups take part in every tile: warpgroup p owns query columns [p*NH, (p+1)*NH) of
    // S^T / P^T / O^T and of the row sums (NH = npad / 2), so the two halves never need merging.
    // Item k accumulates into O^T[k & 1]: its epilogue overlaps the next item's first PVs.
    const int p = (warp - 4) >> 2;
    const int t = tid - 128 - p * 128;              // token row of S^T / d lane of O^T
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    float* mrow = reinterpret_cast<float*>(smem + L::OFF_M) + p * 32;
    float* shs = reinterpret_cast<float*>(smem + L::OFF_SH) + p * 32;
    float* red = reinterpret_cast<float*>(smem + L::OFF_RED) + p * 128;
    float* linv = reinterpret_cast<float*>(smem + L::OFF_LI) + p * 32;
    uint32_t j = 0;                                 // global tile index
    Pend pend;
    pend.valid = 0;
    for (uint32_t k = 0;; ++k) {
      const Sched e = read_sched(ring, sch_full, sch_empty, k, true);
      if (!e.valid) break;
      if (e.npad == 16) softmax_item<8>(smem, tmem, lane_base, p, t, e, k, j, mrow, shs, red, linv, bars, a, ring, pend, TRP);
      else if (e.npad == 32) softmax_item<16>(smem, tmem, lane_base, p, t, e, k, j, mrow, shs, red, linv, bars, a, ring, pend, TRP);
      else softmax_item<32>(smem, tmem, lane_base, p, t, e, k, j, mrow, shs, red, linv, bars, a, ring, pend, TRP);
    }
    if (pend.valid) {
      wg_sync(2 + p, 128);                          // the last item's linv
      finish_item(pend, tmem, lane_base, p, t, linv, bars, a, TRP);
    }
    TRACE_DUMP("softmax");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kWarpAlloc) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
  if (a.app.merge) {
    // K3 in this launch (fused short step): every CTA's partials written -> grid barrier (all CTAs
    // are resident: grid <= SMs, one CTA per SM) -> each warp merges rows of the combine CSR, two
    // rows per warp, exactly as combine16_kernel does (same function, same order: bitwise equal).
    int32_t* bar_count = a.work_counter + kBarCountWord;
    int32_t* bar_gen = a.work_counter + kBarGenWord;
    if (tid == 0) {
      const int gen0 = *reinterpret_cast<volatile int32_t*>(bar_gen);
      __threadfence();                              // this CTA's partials (after the __syncthreads above)
      if (atomicAdd(bar_count, 1) == static_cast<int>(gridDim.x) - 1) {
        *reinterpret_cast<volatile int32_t*>(bar_count) = 0;
        __threadfence();
        atomicAdd(bar_gen, 1);
      } else {
        int g;
        do {
          __nanosleep(64);
          asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(g) : "l"(bar_gen) : "memory");
        } while (g == gen0);
      }
    }
    __syncthreads();
    constexpr int kL = merge_lanes<D>();
    constexpr int kRowsPerWarp = 32 / kL;
    const int nw = kThreads / 32;
    for (int base = (static_cast<int>(blockIdx.x) * nw + warp) * kRowsPerWarp; base < a.app.n_rows;
         base += static_cast<int>(gridDim.x) * nw * kRowsPerWarp) {
      const int row = base + lane / kL;
      const bool valid = row < a.app.n_rows;
      merge_row16<D>(a.app.comb_off, a.app.comb_slot, a.part_o, a.part_lse, a.app.out, a.app.lse, valid ? row : 0,
                     valid, lane & (kL - 1));
    }
  }
  if (tid == 0) release_work_counter(a.work_counter, a.app.enabled != 0);
  if (a.pdl_late) pdl_wait();                        // complete only after the first kernel (combine reads both)
}

}  // namespace tct

namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn get_encode_t() {
  // C++11 function-local static: initialised exactly once, thread-safe.
  static const EncodeTiledFn fn = []() -> EncodeTiledFn {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiledFn>(p);
    return nullptr;
  }();
  return fn;
}
bool make_map_t(CUtensorMap* m, const void* base, int64_t rows, int box_rows) {
  EncodeTiledFn enc = get_encode_t();
  if (!enc) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(tct::D), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(tct::D) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

orion_status launch_split_tct(const PlanHeader* h, const TcArgs& a, const void* k, const void* v,
                              int32_t num_pages, cudaStream_t st) {
  const int num_sms = current_device_sms();
  const cudaError_t attr_err =
      ensure_dynamic_smem(reinterpret_cast<const void*>(tct::split_tct_kernel), tct::L::BYTES);
  if (attr_err != cudaSuccess)
    return fail(ORION_ERR_CUDA, "cudaFuncSetAttribute(split_tct): %s", cudaGetErrorString(attr_err));
  CUtensorMap mk, mv, mk16, mv16;
  const int64_t rows = static_cast<int64_t>(num_pages) * h->num_kv_heads * a.kvs * h->page_size;
  const int big = std::min(64, h->page_size);
  if (!make_map_t(&mk, k, rows, big) || !make_map_t(&mv, v, rows, big) || !make_map_t(&mk16, k, rows, tct::kBox) ||
      !make_map_t(&mv16, v, rows, tct::kBox))
    return fail(ORION_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  int grid = std::min<int>(h->n_items, num_sms > 0 ? num_sms : 148);
  if (h->max_ctas > 0) grid = std::min(grid, h->max_ctas);
#ifdef ORION_CHECK
  if (const char* g = getenv("ORION_DEBUG_GRID")) grid = std::max(1, std::min(grid, atoi(g)));   // debug build only
#endif
  if (!a.work_counter) return fail(ORION_ERR_INVALID_ARG, "split_tct without a work counter");
  cudaError_t e = launch_pdl(tct::split_tct_kernel, dim3(grid), dim3(tct::kThreads), tct::L::BYTES, st, mk, mv,
                             mk16, mv16, a);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ORION_ERR_CUDA, "split_tct_kernel: %s", cudaGetErrorString(e));
  return ORION_OK;
}

}  // namespace orion
