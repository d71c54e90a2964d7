// split_pair.cu — point-prefill attention (the Pre stage, PAPER.md:329,
// 387) with every shared K/V tile streamed once for two readers.
//
// A point-prefill plan is reader-stationary: one work item per (branch, kv head, <= 128-row block)
// streams the branch's whole range list (its dependency spans in list order, then its own content
// causally), so Q is loaded once and each row has one partial, written directly as bf16 out / lse.
// Every branch of a query starts its list with the query's shared prefix (and siblings share
// their common dependencies), so item-per-CTA streams those tiles once per reader: on the c4
// workload 24.5 GB of K/V per layer through L2 for 3 GB of unique KV, and the TMA / barrier
// skeleton alone took two thirds of the kernel.  Here a CTA runs a PAIR of items
// (2u, 2u+1; the planner puts two readers of one kv head, or two row blocks of one reader, next to
// each other and records in items[2u].t1 how many leading ranges their lists share):
//   shared ranges   one K/V tile, two S = Q_A.K^T / Q_B.K^T and two O += P.V MMAs (mask AB);
//   unique tails    A's and B's remaining tiles interleaved one by one (mask A / mask B), so both
//                   softmax warpgroups stay busy.
// Roles (384 threads, one persistent CTA per SM, pair units strided over CTAs):
//   warp 0           TMEM allocator (512 columns: S_A, S_B | P_A, P_B | O_A | O_B).
//   warp 1           QK issuer (S_p = Q_p.K^T, M = 128 rows x N = 64 tokens, once S_p was read).
//   warp 2           TMA producer (K ring, V ring of 64-token stages; one box per page run of a
//                    full tile, 16-row boxes on a ragged edge, 128B swizzle).
//   warp 3           PV issuer (O_p += P_p.V with P from TMEM, as soon as P_p is published).
//   warps 4-7 / 8-11 softmax warpgroup A / B: the rows of item 2u / 2u+1 (thread = row = TMEM
//                    lane), the same masking, lazy rescale and bf16-P row sums as split_tc.cu, and
//                    each its own epilogue (out = acc / l in bf16, lse) -- no merge between them.
//                    A warpgroup gathers its next item's Q rows as soon as its last QK completed.
// All waits are mbarrier phase waits in one global tile order j (the unit walk below, identical
// in every role) plus per-warpgroup tile / unit counters.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>

#include "../../include/orion.h"
#include "plan_format.h"
#include "split_tc.h"
#include "tc_ptx.h"
#include "tmem_ops.h"

namespace orion {
namespace tcp {
using namespace tc;

template <int D> struct PRings;
template <> struct PRings<128> { static constexpr int K = 3, V = 6; };
template <> struct PRings<64> { static constexpr int K = 4, V = 8; };
constexpr int kRows = 128;

template <int D>
struct Smem {
  static constexpr int QB = kRows * D * 2;      // one Q buffer (per warpgroup)
  static constexpr int KVB = kTok * D * 2;      // one K (or V) stage
  static constexpr int HALF_Q = kRows * 128;    // 64-dim half of Q
  static constexpr int HALF_KV = kTok * 128;    // 64-dim half of a K/V stage
  static constexpr int SK = PRings<D>::K, SV = PRings<D>::V;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = 2 * QB;
  static constexpr int OFF_V = OFF_K + SK * KVB;
  static constexpr int OFF_RING = OFF_V + SV * KVB;      // scheduled pair units
  static constexpr int OFF_BAR = OFF_RING + 64;
  static constexpr int N_BAR = 2 * SK + 2 * SV + 6 * 2 + 2 * 8;
  static constexpr int BYTES = OFF_BAR + N_BAR * 8 + 16;
};

__device__ __forceinline__ uint32_t colS(uint32_t p) { return p * 64; }
__device__ __forceinline__ uint32_t colP(uint32_t p) { return 128 + p * 32; }
__device__ __forceinline__ uint32_t colO(uint32_t p) { return 256 + p * 128; }
constexpr int kThreads = 384;
constexpr int kWarpAlloc = 0, kWarpQK = 1, kWarpTMA = 2, kWarpPV = 3;
constexpr int kRing = 8;          // scheduler ring entries
constexpr int kRingReaders = 11;  // producer, QK and PV warps + the 8 softmax warps

struct Unit {
  WorkItem w[2];
  int has_b, n_sh;
};
__device__ __forceinline__ Unit load_unit(const TcArgs& a, int u) {
  Unit U;
  U.w[0] = a.items[2 * u];
  U.has_b = 2 * u + 1 < a.n_items;
  if (U.has_b) U.w[1] = a.items[2 * u + 1];
  U.n_sh = U.has_b ? U.w[0].t1 : 0;
  return U;
}

// Tile cursor over ranges [r, n) of one item.
struct Cur {
  int r, t, n;
  RangeG g;
  bool ok;
};
__device__ __forceinline__ void cur_seek(const TcArgs& a, const WorkItem& w, Cur& c) {
  c.ok = false;
  for (; c.r < c.n; ++c.r) {
    c.g = range_geom(a, w, c.r);
    if (c.g.ntiles > 0) { c.ok = true; return; }
  }
}
__device__ __forceinline__ void cur_next(const TcArgs& a, const WorkItem& w, Cur& c) {
  if (++c.t < c.g.ntiles) return;
  c.t = 0;
  ++c.r;
  cur_seek(a, w, c);
}

// The unit's tile order, identical in every role: the shared leading ranges (mask 3 = both
// warpgroups), then the two unique tails alternating tile by tile (mask 1 = A, mask 2 = B).  An
// iterator rather than a callback walk, so each role's per-tile body is instantiated once (the
// softmax body is large; three inlined copies measurably cost instruction fetch).
struct UnitIter {
  int rs, ts, n_sh;
  RangeG gs;
  Cur ca, cb;
  bool turn_b;
  __device__ __forceinline__ UnitIter(const TcArgs& a, const Unit& U) {
    n_sh = U.n_sh; rs = 0; ts = 0; turn_b = false;
    if (n_sh > 0) gs = range_geom(a, U.w[0], 0);
    ca = Cur{U.n_sh, 0, item_nranges(U.w[0]), {}, false};
    cb = Cur{U.n_sh, 0, U.has_b ? item_nranges(U.w[1]) : 0, {}, false};
    cur_seek(a, U.w[0], ca);
    if (U.has_b) cur_seek(a, U.w[1], cb);
  }
  __device__ __forceinline__ bool next(const TcArgs& a, const Unit& U, int& mask, RangeG& g, int& t) {
    while (rs < n_sh) {
      if (ts < gs.ntiles) { mask = 3; g = gs; t = ts++; return true; }
      if (++rs < n_sh) { gs = range_geom(a, U.w[0], rs); ts = 0; }
    }
    if (cb.ok && (turn_b || !ca.ok)) {
      mask = 2; g = cb.g; t = cb.t; cur_next(a, U.w[1], cb); turn_b = false;
      return true;
    }
    if (ca.ok) {
      mask = 1; g = ca.g; t = ca.t; cur_next(a, U.w[0], ca); turn_b = true;
      return true;
    }
    return false;
  }
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    split_pair_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                      const __grid_constant__ CUtensorMap tmK16, const __grid_constant__ CUtensorMap tmV16,
                      const TcArgs a) {
  using L = Smem<D>;
  constexpr int NH = D / 64;
  constexpr int SK = L::SK, SV = L::SV;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* k_full = bars;
  uint64_t* k_empty = k_full + SK;
  uint64_t* v_full = k_empty + SK;
  uint64_t* v_empty = v_full + SV;
  uint64_t* s_full = v_empty + SV;    // [2] per warpgroup: QK done
  uint64_t* s_free = s_full + 2;      // [2] warpgroup read S_p out
  uint64_t* p_full = s_free + 2;      // [2] warpgroup published P_p
  uint64_t* pv_done = p_full + 2;     // [2] PV into O_p done
  uint64_t* q_full = pv_done + 2;     // [2] Q_p of the warpgroup's next item gathered
  uint64_t* o_free = q_full + 2;      // [2] O_p read out by the epilogue
  uint64_t* u_full = o_free + 2;      // [kRing] scheduler published a unit index
  uint64_t* u_empty = u_full + kRing; // [kRing] every reader warp took it
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(u_empty + kRing);
  volatile int32_t* ring = reinterpret_cast<volatile int32_t*>(smem + L::OFF_RING);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_units = (a.n_items + 1) >> 1;
  if (tid == 0) {
    for (int s = 0; s < SK; ++s) { mbar_init(k_full + s, 1); mbar_init(k_empty + s, 1); }
    for (int s = 0; s < SV; ++s) { mbar_init(v_full + s, 1); mbar_init(v_empty + s, 1); }
    for (int p = 0; p < 2; ++p) {
      mbar_init(s_full + p, 1); mbar_init(s_free + p, 128); mbar_init(p_full + p, 128);
      mbar_init(pv_done + p, 1); mbar_init(q_full + p, 128); mbar_init(o_free + p, 128);
    }
    for (int s = 0; s < kRing; ++s) { mbar_init(u_full + s, 1); mbar_init(u_empty + s, kRingReaders); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmK)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmV)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmK16)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmV16)) : "memory");
  }
  for (int i = tid; i < SV * L::KVB / 16; i += blockDim.x)          // V ring starts finite
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
  TRACE_DECL
  // Pair units are handed out dynamically (atomicAdd on a counter the launcher zeroed) in plan
  // order: units cost up to ~3x each other (a DAG's late points read many dependencies), and a
  // static stride of the grid over a periodic cost pattern leaves whole CTAs with the heavy ones.
  // Entry k of the ring holds the k-th unit this CTA runs (-1 = done); every reader warp takes
  // every entry in order.
  auto take = [&](uint32_t k) -> int {
    const int s = k % kRing;
    mbar_wait(u_full + s, (k / kRing) & 1);
    const int u = ring[s];
    __syncwarp();
    if (lane == 0) mbar_arrive(u_empty + s);
    return u;
  };

  if (warp == kWarpAlloc) {
    // ------------------------------------------------------------------ scheduler
    for (uint32_t k = 0;; ++k) {
      const int s = k % kRing;
      mbar_wait(u_empty + s, ((k / kRing) & 1) ^ 1);
      int u = 0;
      if (lane == 0) {
        u = atomicAdd(a.work_counter, 1);
        if (u >= n_units) u = -1;
        ring[s] = u;
        mbar_arrive(u_full + s);
      }
      u = __shfl_sync(0xffffffffu, u, 0);
      if (u < 0) break;
    }
  } else if (warp == kWarpTMA) {
    // ------------------------------------------------------------------ TMA producer
    // Lane b resolves box b of the tile (<= 4 boxes: one per page run of a full tile, or 16-row
    // boxes on a ragged edge); one elected lane waits for the ring slots and issues the copies.
    uint32_t j = 0;
    const int pmask = (1 << a.page_shift) - 1;
    const int big = min(kTok, 1 << a.page_shift);
    for (uint32_t k = 0;; ++k) {
      const int u = take(k);
      if (u < 0) break;
      const Unit U = load_unit(a, u);
      UnitIter ui(a, U);
      int mask, t;
      RangeG g;
      while (ui.next(a, U, mask, g, t)) {
        const int kvh = (mask & 1) ? U.w[0].kv_head : U.w[1].kv_head;
        const int a0 = g.base + t * kTok;
        const int lo = max(a0, g.t0), hi = min(a0 + kTok, g.end);
        const bool full = (lo == a0 && hi == a0 + kTok);
        int nbox, pos0, step, first_off;
        if (full) { nbox = kTok / big; pos0 = a0; step = big; first_off = 0; }
        else { pos0 = lo & ~(kBox - 1); nbox = (hi - pos0 + kBox - 1) / kBox; step = kBox; first_off = pos0 - a0; }
        int brow = 0;
        if (lane < nbox) {
          const int pos = pos0 + lane * step;
          const int page = __ldg(a.page_table + g.pt_off + (pos >> a.page_shift));
          brow = (((page * a.hkv + kvh) * a.kvs) << a.page_shift) + (pos & pmask);
        }
        int rr[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) rr[b] = __shfl_sync(0xffffffffu, brow, b);
        const int sk = j % SK, sv = j % SV;
        const uint32_t bytes = static_cast<uint32_t>(nbox * step * 128 * NH);
        const CUtensorMap* mk = full ? &tmK : &tmK16;
        const CUtensorMap* mv = full ? &tmV : &tmV16;
        TW(0, mbar_wait(k_empty + sk, ((j / SK) & 1) ^ 1));
        if (elect_one()) {
          mbar_expect_tx(k_full + sk, bytes);
          const uint32_t dk = smem_u32(smem + L::OFF_K + sk * L::KVB);
#pragma unroll
          for (int b = 0; b < 4; ++b)
            if (b < nbox) {
              const uint32_t roff = static_cast<uint32_t>(first_off + b * step) * 128;
#pragma unroll
              for (int h = 0; h < NH; ++h) tma_load_2d(dk + h * L::HALF_KV + roff, mk, h * 64, rr[b], k_full + sk);
            }
        }
        __syncwarp();
        TW(1, mbar_wait(v_empty + sv, ((j / SV) & 1) ^ 1));
        if (elect_one()) {
          mbar_expect_tx(v_full + sv, bytes);
          const uint32_t dv = smem_u32(smem + L::OFF_V + sv * L::KVB);
#pragma unroll
          for (int b = 0; b < 4; ++b)
            if (b < nbox) {
              const uint32_t roff = static_cast<uint32_t>(first_off + b * step) * 128;
#pragma unroll
              for (int h = 0; h < NH; ++h) tma_load_2d(dv + h * L::HALF_KV + roff, mv, h * 64, rr[b], v_full + sv);
            }
        }
        __syncwarp();
        ++j;
      }
    }
    TRACE_DUMP("producer");
  } else if (warp == kWarpQK || warp == kWarpPV) {
    // ------------------------------------------------------------------ MMA issuers
    // n[p]: tiles of warpgroup p so far (its S / P / O barrier phases); uq[p]: its items so far
    // (q_full / o_free phases).  The whole warp runs the control flow; one elected lane issues.
    constexpr uint32_t ID_QK = idesc_bf16(kRows, kTok, false);
    constexpr uint32_t ID_PV = idesc_bf16(kRows, D, true);
    const uint64_t dq0 = sw128_desc(smem_u32(smem + L::OFF_Q), 16, 1024);
    const uint64_t dk0 = sw128_desc(smem_u32(smem + L::OFF_K), 16, 1024);
    const uint64_t dv0 = sw128_desc(smem_u32(smem + L::OFF_V), L::HALF_KV, 1024);
    uint32_t j = 0, n[2] = {0, 0}, uq[2] = {0, 0};
    const bool qk = warp == kWarpQK;
    for (uint32_t k = 0;; ++k) {
      const int u = take(k);
      if (u < 0) break;
      const Unit U = load_unit(a, u);
      bool first[2] = {true, true};
      UnitIter ui(a, U);
      int mask, t;
      RangeG g;
      while (ui.next(a, U, mask, g, t)) {
        if (qk) {
          const int s = j % SK;
          TW(0, mbar_wait(k_full + s, (j / SK) & 1));
          const uint64_t dk = dk0 + static_cast<uint64_t>((s * L::KVB) >> 4);
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            if (!((mask >> p) & 1)) continue;
            if (first[p]) { TW(1, mbar_wait(q_full + p, uq[p] & 1)); first[p] = false; }
            if (n[p] > 0) TW(2 + p, mbar_wait(s_free + p, (n[p] - 1) & 1));     // S_p read out
            tc_fence_after();
            const uint64_t dq = dq0 + static_cast<uint64_t>((p * L::QB) >> 4);
            if (elect_one()) {
#pragma unroll
              for (int ks = 0; ks < D / 16; ++ks) {
                const uint64_t off = static_cast<uint64_t>(((ks >> 2) * L::HALF_KV + (ks & 3) * 32) >> 4);
                const uint64_t offq = static_cast<uint64_t>(((ks >> 2) * L::HALF_Q + (ks & 3) * 32) >> 4);
                mma_ss(tmem + colS(p), dq + offq, dk + off, ID_QK, ks > 0);
              }
              tc_commit(s_full + p);
            }
            __syncwarp();
            ++n[p];
          }
          if (elect_one()) tc_commit(k_empty + s);
          __syncwarp();
        } else {
          const int s = j % SV;
          TW(4, mbar_wait(v_full + s, (j / SV) & 1));
          const uint64_t dv = dv0 + static_cast<uint64_t>((s * L::KVB) >> 4);
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            if (!((mask >> p) & 1)) continue;
            TW(5 + p, mbar_wait(p_full + p, n[p] & 1));
            const bool fst = first[p];
            if (fst && uq[p] > 0) TW(7, mbar_wait(o_free + p, (uq[p] - 1) & 1));   // previous O_p read
            first[p] = false;
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
              for (int kt = 0; kt < kTok / 16; ++kt)
                mma_ts(tmem + colO(p), tmem + colP(p) + kt * 8, dv + static_cast<uint64_t>((kt * 16 * 128) >> 4),
                       ID_PV, (!fst || kt > 0) ? 1u : 0u);
              tc_commit(pv_done + p);
            }
            __syncwarp();
            ++n[p];
          }
          if (elect_one()) tc_commit(v_empty + s);
          __syncwarp();
        }
        ++j;
      }
      ++uq[0];
      if (U.has_b) ++uq[1];
    }
    TRACE_DUMP(qk ? "qk" : "pv");
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ softmax / epilogue
    const int p = (warp - 4) >> 2;
    const int r = tid - 128 - p * 128;             // query row == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    auto item_of = [&](int u) -> int { return (u >= 0 && 2 * u + p < a.n_items) ? 2 * u + p : -1; };
    auto load_q = [&](int it) {
      const WorkItem w = a.items[it];
      const bool ok = r < w.n_rows;
      const __nv_bfloat16* src = a.q;
      if (ok) {   // row -> (reader b, content position i, q head h): plan_format.h
        const int rr = w.row_begin + r, rpr = a.lc * a.group;
        const int b = __ldg(a.readers + w.readers_off + rr / rpr);
        const int i = (rr % rpr) / a.group;
        const int h = w.kv_head * a.group + rr % a.group;
        src = a.q + ((static_cast<size_t>(b) * a.lc + i) * a.hq + h) * D;
      }
      uint8_t* qb = smem + L::OFF_Q + p * L::QB;
#pragma unroll
      for (int c = 0; c < D / 8; ++c) {
        const uint32_t dst = smem_u32(qb + (c >> 3) * L::HALF_Q + r * 128 + (((c & 7) ^ (r & 7)) << 4));
        cp_async16(dst, ok ? static_cast<const void*>(src + c * 8) : static_cast<const void*>(a.q), ok);
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    auto publish_q = [&]() {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      fence_proxy_async();
      mbar_arrive(q_full + p);
    };
    uint32_t k = 0;
    int u = take(0);
    if (item_of(u) >= 0) { load_q(item_of(u)); publish_q(); }
    uint32_t j = 0, np = 0;
    while (u >= 0) {
      const Unit U = load_unit(a, u);
      const bool mine_unit = p == 0 || U.has_b;
      const WorkItem w = p ? U.w[1] : U.w[0];
      const int nt_mine = mine_unit ? item_tiles(a, w) : 0;
      bool peeked = false;
      int u_next = -1, next_it = -1;
      const bool active = mine_unit && (warp & 3) * 32 < w.n_rows;   // warp-uniform
      const int rpos = mine_unit ? ((w.row_begin + r) % (a.lc * a.group)) / a.group : 0;
      float m_used = -INFINITY;
      float2 l2 = make_float2(0.f, 0.f);            // row sum of the bf16 P (even / odd columns)
      int cnt = 0;
      UnitIter ui(a, U);
      int mask, t;
      RangeG g;
      while (ui.next(a, U, mask, g, t)) {
        if ((mask >> p) & 1) {
          const int tb = g.base + t * kTok;
          const int row_end = g.causal ? min(g.end, g.t0 + rpos + 1) : g.end;
          TW(0, mbar_wait(s_full + p, np & 1));
          tc_fence_after();
          uint32_t sr[64];
          TW(1, tmem_ld32x64(tmem + lane_base + colS(p), sr); tc_wait_ld());
          tc_fence_before();
          mbar_arrive(s_free + p);                 // QK of this warpgroup's next tile may overwrite S_p
          if (++cnt == nt_mine) {                  // every QK of this item done: next item's Q
            u_next = take(k + 1);
            peeked = true;
            next_it = item_of(u_next);
            if (next_it >= 0) load_q(next_it);
          }
          bool pv_ok = np == 0;
          const bool edge = g.causal || (tb < g.t0) || (tb + kTok > g.end);
          uint32_t pk[32];
          if (active) {
            float mx = -INFINITY;
            if (!edge) {
#pragma unroll
              for (int c = 0; c < 64; ++c) mx = fmaxf(mx, __uint_as_float(sr[c]));
            } else {
              const int lo_c = g.t0 - tb, hi_c = row_end - tb;
#pragma unroll
              for (int c = 0; c < 64; ++c) {
                const float v = (c >= lo_c && c < hi_c) ? __uint_as_float(sr[c]) : -INFINITY;
                sr[c] = __float_as_uint(v);
                mx = fmaxf(mx, v);
              }
            }
            mx *= a.scale_log2;
            const bool grow = mx > m_used + 8.f;     // lazy rescale (exact: O_p and l refer to m_used)
            if (__any_sync(0xffffffffu, grow)) {
              const float alpha = grow ? ex2(m_used - mx) : 1.f;
              if (np > 0 && cnt > 1) {
                if (!pv_ok) { mbar_wait(pv_done + p, (np - 1) & 1); pv_ok = true; }
                tc_fence_after();
#pragma unroll 1
                for (int cb = 0; cb < D; cb += 16) {
                  uint32_t o[16];
                  tmem_ld32x16(tmem + lane_base + colO(p) + cb, o);
                  tc_wait_ld();
#pragma unroll
                  for (int c = 0; c < 16; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
                  tmem_st32x16(tmem + lane_base + colO(p) + cb, o);
                }
                tc_wait_st();
              }
              if (grow) m_used = mx;
              l2 = __fmul2_rn(l2, make_float2(alpha, alpha));
            }
            const float mb = m_used == -INFINITY ? 0.f : m_used;
            const float2 sc2 = make_float2(a.scale_log2, a.scale_log2), nmb2 = make_float2(-mb, -mb);
#pragma unroll
            for (int c = 0; c < 32; ++c) {   // packed fp32x2 FMA / add: half the FP32 instructions
              const float2 e = __ffma2_rn(make_float2(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])),
                                          sc2, nmb2);
              pk[c] = pack_bf16(ex2(e.x), ex2(e.y));
              l2 = __fadd2_rn(l2, make_float2(__uint_as_float(pk[c] << 16),          // reading S17
                                              __uint_as_float(pk[c] & 0xFFFF0000u)));
            }
          } else {
#pragma unroll
            for (int c = 0; c < 32; ++c) pk[c] = 0u;
          }
          if (!pv_ok) TW(2, mbar_wait(pv_done + p, (np - 1) & 1));   // PV of the previous tile read P_p
          tc_fence_after();
          TW(3, tmem_st32x32(tmem + lane_base + colP(p), pk); tc_wait_st());
          // Zero V rows outside [t0, end) of an edge tile once it landed (0 x NaN = NaN).  A shared
          // tile is zeroed by warpgroup A only: the PV issuer issues PV_A (after A published)
          // before PV_B.
          const bool zeroer = mask != 3 || p == 0;
          if (edge && zeroer) {
            mbar_wait(v_full + (j % SV), (j / SV) & 1);
            if (r < kTok) {
              const int pos = tb + r;
              if (pos < g.t0 || pos >= g.end) {
                uint8_t* vrow = smem + L::OFF_V + (j % SV) * L::KVB + r * 128;
#pragma unroll
                for (int h = 0; h < NH; ++h) {
                  uint4* p4 = reinterpret_cast<uint4*>(vrow + h * L::HALF_KV);
#pragma unroll
                  for (int c = 0; c < 8; ++c) p4[c] = make_uint4(0, 0, 0, 0);
                }
              }
            }
          }
          fence_proxy_async();
          tc_fence_before();
          mbar_arrive(p_full + p);
          ++np;
        }
        ++j;
      }
      if (!peeked) { u_next = take(k + 1); next_it = item_of(u_next); }
      if (!mine_unit) { u = u_next; ++k; continue; }
      // ---- epilogue: out = O_p / l in bf16 and lse (the row's only partial)
      if (cnt > 0) TW(4, mbar_wait(pv_done + p, (np - 1) & 1));   // last PV of this item
      tc_fence_after();
      const float l_run = l2.x + l2.y;
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      size_t orow = 0;
      if (a.out && r < w.n_rows) {
        const int rr = w.row_begin + r, rpr = a.lc * a.group;
        const int b = __ldg(a.readers + w.readers_off + rr / rpr);
        orow = (static_cast<size_t>(b) * a.lc + (rr % rpr) / a.group) * a.hq + w.kv_head * a.group + rr % a.group;
      }
      if (active) {
#pragma unroll 1
        for (int cb = 0; cb < D; cb += 16) {
          uint32_t o[16];
          tmem_ld32x16(tmem + lane_base + colO(p) + cb, o);
          tc_wait_ld();
          if (r < w.n_rows) {
            if (cnt == 0) {
#pragma unroll
              for (int c = 0; c < 16; ++c) o[c] = 0u;
            }
            if (a.out) {
#pragma unroll
              for (int c = 0; c < 16; c += 4) {
                uint2 pk2;
                pk2.x = pack_bf16(__uint_as_float(o[c]) * inv, __uint_as_float(o[c + 1]) * inv);
                pk2.y = pack_bf16(__uint_as_float(o[c + 2]) * inv, __uint_as_float(o[c + 3]) * inv);
                *reinterpret_cast<uint2*>(a.out + orow * D + cb + c) = pk2;
              }
            } else {   // fp32 partial (acc, m, l): the single partial of the row, K3 reproduces out
              float* dst = a.part_acc + static_cast<size_t>(w.slot0 + r) * D + cb;
#pragma unroll
              for (int c = 0; c < 16; c += 4)
                *reinterpret_cast<float4*>(dst + c) = make_float4(__uint_as_float(o[c]), __uint_as_float(o[c + 1]),
                                                                  __uint_as_float(o[c + 2]), __uint_as_float(o[c + 3]));
            }
          }
        }
      }
      if (r < w.n_rows) {
        if (!a.out) a.part_ml[w.slot0 + r] = make_float2(cnt > 0 ? m_used : -INFINITY, l_run);
        else if (a.lse) a.lse[orow] = l_run > 0.f ? (m_used + log2f(l_run)) * 0.69314718055994531f : -INFINITY;
      }
      tc_fence_before();
      mbar_arrive(o_free + p);
      if (next_it >= 0) publish_q();
      u = u_next;
      ++k;
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    if ((warp & 3) == 0) TRACE_DUMP(p ? "smB" : "smA");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kWarpAlloc) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
  if (threadIdx.x == 0) release_work_counter(a.work_counter);
}

}  // namespace tcp

template <int D>
orion_status launch_split_pair(const PlanHeader* h, const TcArgs& a, const CUtensorMap maps[4], cudaStream_t st) {
  const int num_sms = current_device_sms();
  const cudaError_t attr_err = ensure_dynamic_smem(reinterpret_cast<const void*>(tcp::split_pair_kernel<D>),
                                                   tcp::Smem<D>::BYTES + 1024);
  if (attr_err != cudaSuccess)
    return fail(ORION_ERR_CUDA, "cudaFuncSetAttribute(split_pair): %s", cudaGetErrorString(attr_err));
  const int n_units = (h->n_items + 1) / 2;
  if (!a.work_counter) return fail(ORION_ERR_INVALID_ARG, "paired plan without a work counter");
  int grid = std::min<int>(n_units, num_sms > 0 ? num_sms : 148);
  if (h->max_ctas > 0) grid = std::min(grid, h->max_ctas);
  tcp::split_pair_kernel<D><<<grid, tcp::kThreads, tcp::Smem<D>::BYTES + 1024, st>>>(maps[0], maps[1], maps[2],
                                                                                     maps[3], a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ORION_ERR_CUDA, "split_pair_kernel: %s", cudaGetErrorString(e));
  return ORION_OK;
}

template orion_status launch_split_pair<64>(const PlanHeader*, const TcArgs&, const CUtensorMap[4], cudaStream_t);
template orion_status launch_split_pair<128>(const PlanHeader*, const TcArgs&, const CUtensorMap[4], cudaStream_t);

}  // namespace orion
