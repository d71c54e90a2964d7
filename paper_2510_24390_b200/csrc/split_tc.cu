// split_tc.cu — K2 split attention on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Rows-on-lanes orientation (query rows on the MMA M dimension, one TMEM lane / softmax thread
// per row): used for head_dim 64 decode, ORION_PLAN_ROWS_ON_LANES, and point prefill, whose Lc*G
// rows per branch fill the 128-row M tile.  One persistent CTA
// per SM walks the plan's work items (a shared piece x kv head x chunk x <= 128 rows, or for a
// prefill plan one branch's whole range list).  Roles:
//   warp 0           TMEM allocator (512 columns), then the item scheduler (atomic counter -> ring).
//   warp 1           QK issuer: S(j) = Q.K(j)^T (tcgen05.mma kind::f16, A = Q smem, B = K smem,
//                    M = 128 rows x N = 64 tokens) into S[t & 1] (t: tile index in its item) once K landed and the
//                    softmax warpgroup has read S(j-2) out.
//   warp 2 (1 lane)  TMA producer: K and V rings of 64-token stages (one box per page run of a
//                    full tile, 16-row boxes on a ragged edge, 128B swizzle), page-table lookups
//                    resolved 32 tiles at a time.
//   warp 3           PV issuer: O[t & 1] += P.V (A = P from TMEM, B = V smem MN-major,
//                    M = 128 x N = d) as soon as P(j) is published.  Two issuers, so one
//                    warpgroup's next S never waits behind the other's P (tcgen05.commit tracks
//                    the issuing thread's own MMAs).
//   warps 4-7 / 8-11 softmax warpgroups owning the even / odd tiles of an item: tcgen05.ld of the
//                    S row, masking (ragged edges; per-row causal limits in a prefill's own
//                    range), lazy-rescaled online max in the log2 domain (O and l rescaled only
//                    when the running max grows by > 2^8), P = exp2 rounded to bf16 into TMEM,
//                    l summed per thread from the same rounded P, V rows outside the range
//                    zeroed once the tile has landed.  At item end warpgroup 1 hands (m, l) to
//                    warpgroup 0, which merges the two accumulators into the fp32 partial
//                    (m, l, acc) -- or, for a prefill plan, straight into bf16 out and lse.
//                    Warpgroup 0 also gathers the next items' Q rows.
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
namespace tc {

// Separate K and V rings: a K stage is released as soon as its QK completes, a V stage only after
// its PV, so the producer can run ~3 tiles ahead of the QK cursor (enough bytes in flight to cover
// HBM latency at the per-SM share of the bandwidth).
template <int D> struct Rings;
template <> struct Rings<128> { static constexpr int K = 3, V = 6; };
template <> struct Rings<64> { static constexpr int K = 4, V = 8; };
constexpr int kRows = 128;     // MMA M (query rows per item)

constexpr int kRing = 6;          // item ring entries (warp 0 schedules after TMEM allocation)
constexpr int kAhead = 3;         // items fetched ahead of the oldest unfinished one
constexpr int kMaxRanges = 64;    // ranges whose geometry an entry carries (more: read from the plan)
// A scheduled item with the geometry of its ranges, resolved once by the scheduler warp (one lane
// per range: the plan's Range and the dynamic end's own_len loads overlap) and read from shared
// memory by every role.  Walking an item's range list through dependent global loads at every
// item and range boundary had cost each role ~1 us per range on the critical path (point-prefill
// lists carry up to ~20 ranges, c5 chain-64 masked items ~50).
struct ItemG {
  int32_t it, n_ranges, ntiles, pad_;
  WorkItem w;
  RangeG r[kMaxRanges];
};
static_assert(sizeof(RangeG) == 32, "RangeG is 32 bytes");

template <int D>
struct Smem {
  static constexpr int QB = kRows * D * 2;      // one Q buffer
  static constexpr int KVB = kTok * D * 2;      // one K (or V) stage
  static constexpr int HALF_Q = kRows * 128;    // 64-dim half of Q
  static constexpr int HALF_KV = kTok * 128;    // 64-dim half of a K/V stage
  static constexpr int OFF_Q = 0;
  static constexpr int SK = Rings<D>::K, SV = Rings<D>::V;
  static constexpr int OFF_K = 2 * QB;
  static constexpr int OFF_V = OFF_K + SK * KVB;
  static constexpr int OFF_XCH = OFF_V + SV * KVB;   // both WGs' (m, l) per row, x2 (item parity)
  static constexpr int OFF_RING = OFF_XCH + 4 * kRows * 8;   // scheduled items with their geometry
  static constexpr int OFF_BAR = OFF_RING + kRing * static_cast<int>(sizeof(ItemG));
  // k/v full+empty; s_full, p_full, pv_done, q_full; o_free; s_free; u_full + u_empty
  static constexpr int N_BAR = 2 * SK + 2 * SV + 2 + 2 + 2 + 2 + 1 + 2 + 2 * kRing;
  static constexpr int BYTES = OFF_BAR + N_BAR * 8 + 16;
};

static_assert(Smem<128>::BYTES + 1024 <= 232448 && Smem<64>::BYTES + 1024 <= 232448, "shared memory budget");

// TMEM columns: S and P double-buffered by tile parity; one O accumulator per softmax warpgroup.
__device__ __forceinline__ uint32_t colS(uint32_t p) { return p * 64; }
__device__ __forceinline__ uint32_t colP(uint32_t p) { return 128 + p * 32; }
__device__ __forceinline__ uint32_t colO(uint32_t p) { return 256 + p * 128; }
// Q of the current item as the QK MMAs' A operand in TMEM (D / 2 columns): copied from its smem
// staging buffer once per item (tcgen05.cp, in the QK issuer's pipeline order) instead of being
// re-read from shared memory by every tile's QK -- a third of a tile's smem operand traffic.
constexpr uint32_t kColQ = 192;
constexpr int kThreadsTC = 384;   // warps 0-3: TMEM alloc / idle / TMA / MMA; 4-7: WG0; 8-11: WG1
// The TMA and MMA warps sit on SM sub-partitions 2 and 3 so that their barrier polling does not
// steal issue slots from the softmax warps of items with <= 64 rows (TMEM lanes 0-63 are only
// reachable from warps 4k and 4k+1, i.e. sub-partitions 0 and 1).
constexpr int kWarpAlloc = 0, kWarpQK = 1, kWarpTMA = 2, kWarpMMA = 3;
constexpr int kRingReaders = 11;  // producer, QK and PV warps + the 8 softmax warps

__device__ __forceinline__ RangeG geo_range(const TcArgs& a, const ItemG& e, int r) {
  return r < kMaxRanges ? e.r[r] : range_geom(a, e.w, r);
}

template <int D>
__global__ void __launch_bounds__(kThreadsTC, 1)
    split_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                    const __grid_constant__ CUtensorMap tmK16, const __grid_constant__ CUtensorMap tmV16,
                    const TcArgs a) {
  using L = Smem<D>;
  constexpr int NH = D / 64;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps the smem space
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  constexpr int SK = L::SK, SV = L::SV;
  uint64_t* k_full = bars;
  uint64_t* k_empty = k_full + SK;
  uint64_t* v_full = k_empty + SK;
  uint64_t* v_empty = v_full + SV;
  uint64_t* s_full = v_empty + SV;
  uint64_t* p_full = s_full + 2;
  uint64_t* pv_done = p_full + 2;
  uint64_t* q_full = pv_done + 2;
  uint64_t* o_free = q_full + 2;
  uint64_t* s_free = o_free + 1;                  // softmax WG has read S[b] into registers
  uint64_t* u_full = s_free + 2;                  // [kRing] scheduler published an item index
  uint64_t* u_empty = u_full + kRing;             // [kRing] every reader warp took it
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(u_empty + kRing);
  ItemG* geo = reinterpret_cast<ItemG*>(smem + L::OFF_RING);
  float2* xch = reinterpret_cast<float2*>(smem + L::OFF_XCH);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < SK; ++s) { mbar_init(k_full + s, 1); mbar_init(k_empty + s, 1); }
    for (int s = 0; s < SV; ++s) { mbar_init(v_full + s, 1); mbar_init(v_empty + s, 1); }
    for (int b = 0; b < 2; ++b) {
      mbar_init(s_full + b, 1); mbar_init(p_full + b, 128); mbar_init(pv_done + b, 1);
      mbar_init(q_full + b, 128);
    }
    mbar_init(o_free, 256);                         // both warpgroups read both O accumulators
    mbar_init(s_free + 0, 128);
    mbar_init(s_free + 1, 128);
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
  const int n_items = a.n_items;
  // Programmatic dependent launch: wait for the previous kernel (the KV append) first, then let
  // the next one launch -- a hybrid plan's second split kernel relies on this order (it starts
  // without its own wait once this kernel has triggered; split_tc.h TcArgs::pdl_late).
  pdl_wait();
  pdl_trigger();

  TRACE_DECL
  // Items are handed out by an atomic counter in plan order: greedy list scheduling over the SMs
  // (a static grid stride left the busiest SM 19 % above the mean on the c4 point prefill).  Warp 0
  // publishes the k-th item this CTA runs, with its range geometry, in ring entry k % kRing (it =
  // -1: done); every other role takes every entry in order and releases it when done with it.
  auto take = [&](uint32_t k) -> const ItemG& {
    mbar_wait(u_full + (k % kRing), (k / kRing) & 1);
    return geo[k % kRing];
  };
  auto release = [&](uint32_t k) {
    __syncwarp();
    if (lane == 0) mbar_arrive(u_empty + (k % kRing));
  };
  if (warp == kWarpAlloc) {
    // ------------------------------------------------------------------ scheduler
    for (uint32_t k = 0;; ++k) {
      const int s = k % kRing;
      mbar_wait(u_empty + s, ((k / kRing) & 1) ^ 1);
      // Take item k from the global counter only once item k - kAhead is done: a CTA holding
      // several fetched but unstarted items at the end of the plan leaves other SMs idle (with the
      // ring's full depth of look-ahead the busiest SM ran 1.4x the mean on c5 chain-64).
      if (k >= static_cast<uint32_t>(kAhead))
        mbar_wait(u_empty + ((k - kAhead) % kRing), ((k - kAhead) / kRing) & 1);
      ItemG& e = geo[s];
      int it;
      for (;;) {
        it = 0;
        if (lane == 0) {
          it = atomicAdd(a.work_counter, 1);
          if (it >= n_items) it = -1;
        }
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it < 0) break;
        const WorkItem w = a.items[it];
        const int nr = item_nranges(w);
        int tiles = 0;
        for (int r = lane; r < nr; r += 32) {
          const RangeG g = range_geom(a, w, r);
          if (r < kMaxRanges) e.r[r] = g;
          tiles += g.ntiles;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) tiles += __shfl_xor_sync(0xffffffffu, tiles, o);
        if (tiles > 0 || a.out) {
          if (lane == 0) { e.w = w; e.n_ranges = nr; e.ntiles = tiles; }
          break;
        }
        // An empty item (its dynamic ranges end at or before t0 at the current lengths) never
        // enters the ring: this warp writes its neutral partials and takes the next item.  (In the
        // ring it could deadlock the look-ahead: a warpgroup holding item k while it skips empty
        // entries towards its prefetch would wait for entry k + kAhead, which waits for item k.)
        for (int i = lane; i < w.n_rows * (D / 8); i += 32) {
          const int row = i / (D / 8), c = i % (D / 8);
          if (a.part16) {
            reinterpret_cast<uint4*>(a.part_o + static_cast<size_t>(w.slot0 + row) * D)[c] = make_uint4(0, 0, 0, 0);
          } else {
            float4* dst = reinterpret_cast<float4*>(a.part_acc + static_cast<size_t>(w.slot0 + row) * D) + 2 * c;
            dst[0] = make_float4(0.f, 0.f, 0.f, 0.f);
            dst[1] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
          if (c == 0) {
            if (a.part16) a.part_lse[w.slot0 + row] = -INFINITY;
            else a.part_ml[w.slot0 + row] = make_float2(-INFINITY, 0.f);
          }
        }
      }
      if (lane == 0) e.it = it;
      __syncwarp();
      if (lane == 0) mbar_arrive(u_full + s);
      if (it < 0) break;
    }
  } else if (warp == kWarpTMA) {
    // ------------------------------------------------------------------ TMA producer
    // Tiles sit on the 64-token grid.  A tile fully inside [t0, end) is fetched with one box of
    // min(64, P) token rows per page (map *_big); an item's first/last partial tile with 16-row
    // boxes (map *_16).  The warp resolves the boxes of 32 tiles at once (one lane per tile, so the
    // page-table loads overlap); lane 0 waits for ring slots and issues the copies.
    uint32_t j = 0;
    const int pmask = (1 << a.page_shift) - 1;
    const int big = min(kTok, 1 << a.page_shift);          // rows of a full-tile box
    for (uint32_t ke = 0;; ++ke) {
      const ItemG& e = take(ke);
      if (e.it < 0) { release(ke); break; }
      const int kv_head = e.w.kv_head;
      for (int rg_i = 0; rg_i < e.n_ranges; ++rg_i) {
      const RangeG g = geo_range(a, e, rg_i);
      for (int tb0 = 0; tb0 < g.ntiles; tb0 += 32) {
        // lane l describes tile tb0 + l: up to 4 boxes (row coordinate each), kind, offsets
        int brow[4] = {0, 0, 0, 0};
        int nbox = 0, first_off = 0, full = 0;
        if (tb0 + lane < g.ntiles) {
          const int a0 = g.base + (tb0 + lane) * kTok;
          const int lo = max(a0, g.t0), hi = min(a0 + kTok, g.end);
          full = (lo == a0 && hi == a0 + kTok);
          int pos0, step;
          if (full) { nbox = kTok / big; pos0 = a0; step = big; first_off = 0; }
          else { pos0 = lo & ~(kBox - 1); nbox = (hi - pos0 + kBox - 1) / kBox; step = kBox; first_off = pos0 - a0; }
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            if (b < nbox) {
              const int pos = pos0 + b * step;
              const int page = __ldg(a.page_table + g.pt_off + (pos >> a.page_shift));
              brow[b] = (((page * a.hkv + kv_head) * a.kvs) << a.page_shift) + (pos & pmask);
            }
          }
        }
        const int tend = min(g.ntiles, tb0 + 32);
        for (int t = tb0; t < tend; ++t, ++j) {
          const int src = t - tb0;
          const int tn = __shfl_sync(0xffffffffu, nbox, src);
          const int tf = __shfl_sync(0xffffffffu, full, src);
          const int to = __shfl_sync(0xffffffffu, first_off, src);
          int rr[4];
#pragma unroll
          for (int b = 0; b < 4; ++b) rr[b] = __shfl_sync(0xffffffffu, brow[b], src);
          const int sk = j % SK, sv = j % SV;
          const int rows_per_box = tf ? big : kBox;
          const uint32_t bytes = static_cast<uint32_t>(tn * rows_per_box * 128 * NH);
          const CUtensorMap* mk = tf ? &tmK : &tmK16;
          const CUtensorMap* mv = tf ? &tmV : &tmV16;
          TW(0, mbar_wait(k_empty + sk, ((j / SK) & 1) ^ 1));
          if (elect_one()) {
            mbar_expect_tx(k_full + sk, bytes);
            const uint32_t dk = smem_u32(smem + L::OFF_K + sk * L::KVB);
#pragma unroll
            for (int b = 0; b < 4; ++b)
              if (b < tn) {
                const uint32_t roff = static_cast<uint32_t>(to + b * rows_per_box) * 128;
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
              if (b < tn) {
                const uint32_t roff = static_cast<uint32_t>(to + b * rows_per_box) * 128;
#pragma unroll
                for (int h = 0; h < NH; ++h) tma_load_2d(dv + h * L::HALF_KV + roff, mv, h * 64, rr[b], v_full + sv);
              }
          }
          __syncwarp();
        }
      }
      }
      release(ke);
    }
    TRACE_DUMP("producer");
  } else if (warp == kWarpMMA || warp == kWarpQK) {
    // ------------------------------------------------------------------ MMA issuer
    // Two cursors walk the flattened (item, tile) sequence: QK runs two tiles ahead of PV, so
    // S(j+2) = Q K(j+2)^T is issued as soon as softmax warpgroup j&1 has read S(j) into registers
    // (s_free), and O[j&1] += P(j) V(j) (plus l += P(j).1) as soon as it has published P(j).
    // The whole warp runs the control flow (warp-uniform descriptors); one elected lane issues.
    constexpr uint32_t ID_QK = idesc_bf16(kRows, kTok, false);
    constexpr uint32_t ID_PV = idesc_bf16(kRows, D, true);
    const uint64_t dq0 = sw128_desc(smem_u32(smem + L::OFF_Q), 16, 1024);
    const uint64_t dk0 = sw128_desc(smem_u32(smem + L::OFF_K), 16, 1024);
    const uint64_t dv0 = sw128_desc(smem_u32(smem + L::OFF_V), L::HALF_KV, 1024);
    struct Cur {
      int live, t, nt;
      uint32_t k, j, e, ent;                        // e: ring entries taken; ent: the current one
    };
    auto next_ne = [&](Cur& c) {                    // next non-empty item of the ring, or the end
      for (;;) {
        const uint32_t ke = c.e++;
        const ItemG& g = take(ke);
        if (g.it < 0) { release(ke); c.live = 0; c.nt = 0; return; }
        if (g.ntiles > 0) { c.live = 1; c.nt = g.ntiles; c.ent = ke; return; }
        release(ke);
      }
    };
    auto start = [&](Cur& c) {
      c.t = 0; c.k = 0; c.j = 0; c.e = 0;
      next_ne(c);
    };
    auto advance = [&](Cur& c) {
      ++c.j;
      if (++c.t == c.nt) {
        release(c.ent);
        next_ne(c);
        c.t = 0; ++c.k;
      }
    };
    // Tile t of an item goes to softmax warpgroup t & 1 (item-relative, so an item's arithmetic does
    // not depend on which CTA runs it or what ran before: results are deterministic under the
    // atomic item hand-out); nq_p / nv_p count warpgroup p's tiles for its barrier phases
    // (scalars, not arrays indexed by the runtime parity: those would live in local memory)
    uint32_t nq0 = 0, nq1 = 0, nv0 = 0, nv1 = 0;
    auto issue_qk = [&](const Cur& c) {
      const uint32_t j = c.j;
      const uint32_t p = c.t & 1;
      if (c.t == 0) {
        TW(1, mbar_wait(q_full + (c.k & 1), (c.k >> 1) & 1));
      }
      const int s = j % SK;
      TW(2, mbar_wait(k_full + s, (j / SK) & 1));
      const uint32_t nqp = p ? nq1 : nq0;
      if (nqp > 0) TW(3, mbar_wait(s_free + p, (nqp - 1) & 1));   // S[p] read out
      // QK(j) is issued as soon as S(j-2) is read out, ahead of PV(j-2): S(j) is then ready when
      // the warpgroup finishes tile j-2, and PV(j-2) still completes long before the warpgroup
      // stores P(j) (after tile j's exponentials).
      tc_fence_after();
      const uint64_t dq = dq0 + static_cast<uint64_t>(((c.k & 1) * L::QB) >> 4);
      const uint64_t dk = dk0 + static_cast<uint64_t>((s * L::KVB) >> 4);
      const uint32_t dS = tmem + colS(p);
      if (elect_one()) {
        if (c.t == 0) {                             // the item's Q: smem staging buffer -> TMEM
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks)
            tc_cp_128x256b(tmem + kColQ + ks * 8,
                           dq + static_cast<uint64_t>(((ks >> 2) * L::HALF_Q + (ks & 3) * 32) >> 4));
        }
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint64_t off = static_cast<uint64_t>(((ks >> 2) * L::HALF_KV + (ks & 3) * 32) >> 4);
          mma_ts(dS, tmem + kColQ + ks * 8, dk + off, ID_QK, ks > 0);
        }
        tc_commit(s_full + p);
        tc_commit(k_empty + s);
      }
      __syncwarp();
      if (p) ++nq1; else ++nq0;
    };
    auto issue_pv = [&](const Cur& c) {
      const uint32_t j = c.j;
      const uint32_t p = c.t & 1;
      const int s = j % SV;
      TW(6, mbar_wait(v_full + s, (j / SV) & 1));
      TW(4, mbar_wait(p_full + p, (p ? nv1 : nv0) & 1));
      if (c.t == 0 && c.k > 0) TW(5, mbar_wait(o_free, (c.k - 1) & 1));   // previous item's O read
      tc_fence_after();
      const uint64_t dv = dv0 + static_cast<uint64_t>((s * L::KVB) >> 4);
      const uint32_t aP = tmem + colP(p);
      const uint32_t dO = tmem + colO(p);
      const bool first = c.t < 2;        // first tile of this parity in the item
      if (elect_one()) {
#pragma unroll
        for (int kt = 0; kt < kTok / 16; ++kt) {
          mma_ts(dO, aP + kt * 8, dv + static_cast<uint64_t>((kt * 16 * 128) >> 4), ID_PV,
                 (!first || kt > 0) ? 1u : 0u);

        }
        tc_commit(pv_done + p);
        tc_commit(v_empty + s);
      }
      __syncwarp();
      if (p) ++nv1; else ++nv0;
    };
    // Two issuers (tcgen05.commit tracks the issuing thread's own MMAs): warp 1 issues every
    // S(j) = Q K(j)^T as soon as K(j) landed and softmax warpgroup j&1 has read S(j-2) out
    // (s_free), warp 3 every O += P(j) V(j) as soon as P(j) is published.  Neither waits behind
    // the other's dependencies, so one warpgroup's next S never queues behind the other
    // warpgroup's P.  Q buffer reuse needs no extra guard: warpgroup 0 publishes item k+2's Q
    // only after item k's epilogue, i.e. after every MMA of item k.
    Cur c;
    start(c);
    if (warp == kWarpQK) {
      while (c.live) { issue_qk(c); advance(c); }
    } else {
      while (c.live) { issue_pv(c); advance(c); }
    }
    TRACE_DUMP("mma");
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ softmax / epilogue
    // Warpgroup p (p = 0: warps 4-7, p = 1: warps 8-11) owns the tiles j with j&1 == p: its own
    // running max m_p, sum l_p and accumulator O_p.  Thread = query row = TMEM lane.  At item end
    // WG1 hands (m_1, l_1) to WG0, which merges O_0 and O_1 and writes the partial.
    const int p = (warp - 4) >> 2;
    const int r = tid - 128 - p * 128;             // query row == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    auto load_q = [&](int k_item, int ent) {       // WG0 only; ent: the item's ring entry or -1
      if (ent >= 0) {
        const WorkItem& w = geo[ent % kRing].w;
        const bool ok = r < w.n_rows;
        const __nv_bfloat16* src = a.q;
        if (ok) {   // row -> (reader b, content position i, q head h): plan_format.h
          const int rr = w.row_begin + r, rpr = a.lc * a.group;
          const int b = __ldg(a.readers + w.readers_off + rr / rpr);
          const int i = (rr % rpr) / a.group;
          const int h = w.kv_head * a.group + rr % a.group;
          src = a.q + ((static_cast<size_t>(b) * a.lc + i) * a.hq + h) * D;
        }
        uint8_t* qb = smem + L::OFF_Q + (k_item & 1) * L::QB;
#pragma unroll
        for (int c = 0; c < D / 8; ++c) {
          const uint32_t dst = smem_u32(qb + (c >> 3) * L::HALF_Q + r * 128 + (((c & 7) ^ (r & 7)) << 4));
          cp_async16(dst, ok ? static_cast<const void*>(src + c * 8) : static_cast<const void*>(a.q), ok);
        }
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    uint32_t ke = 0;                                // ring entries taken by this warp
    auto next_item = [&]() -> int {                 // the next item's ring entry (held), or -1
      for (;;) {
        const uint32_t kk = ke++;
        const ItemG& g = take(kk);
        if (g.it < 0) { release(kk); return -1; }
        if (g.ntiles > 0) return static_cast<int>(kk);
        // ntiles == 0 reaches the ring only in a direct-output (prefill) plan, whose items are
        // never empty (the own causal range has Lc >= 1 tokens); decode plans' empty items are
        // resolved by the scheduler warp
        release(kk);
      }
    };
    int cur = next_item(), pf = -1;
    if (p == 0) {                                   // Q of item 0 now, item 1 ahead
      load_q(0, cur);
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      fence_proxy_async();
      mbar_arrive(q_full + 0);
      if (cur >= 0) pf = next_item();
      load_q(1, pf);
    }
    uint32_t j = 0, k = 0, np = 0;                  // np: this warpgroup's tiles so far
#ifdef ORION_TC_TIMELINE
    // dev only (-DORION_TC_TIMELINE): CTA 0's first 48 turns per warpgroup, printed at the end
    long long tl_r[48], tl_e[48];
#endif
    // The two warpgroups take turns at the exponentials (named barriers 2: WG0's turn, 3: WG1's):
    // one warpgroup's ex2 phase saturates the SM's MUFU on its own, so running them one after the
    // other overlaps each warpgroup's S read-out, P store and barrier waits with the other's
    // exponentials instead of both doing them at once.  Turns follow the item's tile order
    // (tile t: warpgroup t & 1); an item with an odd tile count ends with a pass by WG1, so every
    // item hands the turn back to WG0.  WG1 gives WG0 the first turn; WG0 takes the last token.
    if (p == 1) asm volatile("bar.arrive 2, 256;\n" ::: "memory");
    while (cur >= 0) {
      const ItemG& cg = geo[cur % kRing];
      const WorkItem w = cg.w;
      const bool active = (warp & 3) * 32 < w.n_rows;   // warp-uniform
      // point prefill: this row's content position i; in the causal own range it sees [t0, t0 + i]
      const int rpos = ((w.row_begin + r) % (a.lc * a.group)) / a.group;
      float m_used = -INFINITY;
      float l_run = 0.f;                            // this row's sum of the bf16 P it published
      bool had = false;
      int ti = 0;                                   // tile index within the item (WG ti & 1)
      for (int rg_i = 0; rg_i < cg.n_ranges; ++rg_i) {
      const RangeG g = geo_range(a, cg, rg_i);
      // a masked range (hybrid big items): rows of readers outside its mask see none of it
      const bool rmask = g.masked && !((g.mask >> ((w.row_begin + r) / (a.lc * a.group))) & 1u);
      const int row_end = rmask ? g.t0 : (g.causal ? min(g.end, g.t0 + rpos + 1) : g.end);
      for (int t = 0; t < g.ntiles; ++t, ++j, ++ti) {
        if ((ti & 1) != p) continue;
        const int tb = g.base + t * kTok;
        TW(6, mbar_wait(s_full + p, np & 1));
        tc_fence_after();
        uint32_t sr[64];
#ifdef ORION_TC_TRACE
        unsigned long long ts0 = clock64();
#endif
        tmem_ld32x64(tmem + lane_base + colS(p), sr);
        tc_wait_ld();
#ifdef ORION_TC_TRACE
        tr_[0] += clock64() - ts0; ts0 = clock64();
#endif
        tc_fence_before();
        mbar_arrive(s_free + p);                  // QK(j+2) may overwrite S[p] now
        // PV(j-2) must be complete before O_p is rescaled or P[p] rewritten; the wait is taken as
        // late as possible so that its latency overlaps this tile's exponentials.
        bool pv_ok = np == 0;
        const bool edge = g.causal || (tb < g.t0) || (tb + kTok > g.end);
        const bool cmask = edge || rmask;            // this row's scores need the column mask
        uint32_t pk[32];
#ifdef ORION_TC_TRACE
        unsigned long long tm0 = clock64();
#endif
        if (active) {
          float mx = -INFINITY;                     // raw scores; scale > 0 commutes with max
          if (cmask) {
            const int lo_c = g.t0 - tb, hi_c = row_end - tb;   // valid columns [lo_c, hi_c)
#pragma unroll
            for (int c = 0; c < 64; ++c)
              sr[c] = (c >= lo_c && c < hi_c) ? sr[c] : __float_as_uint(-INFINITY);
          }
          mx = max_tree(sr);
          mx *= a.scale_log2;
          // Lazy rescale (exact: O_p and l_p refer to m_used).  Warp-uniform so the aligned TMEM
          // accesses are executed by the whole warp.
          const bool mine = mx > m_used + 8.f;
#ifdef ORION_TC_TRACE
          tr_[5] += clock64() - tm0; tm0 = clock64();
#endif
          if (__any_sync(0xffffffffu, mine)) {
            const float alpha = mine ? ex2(m_used - mx) : 1.f;   // 0 when m_used == -inf
            if (had) {
              if (!pv_ok) { TW(7, mbar_wait(pv_done + p, (np - 1) & 1)); pv_ok = true; }
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
            if (mine) m_used = mx;
            l_run *= alpha;
          }
        }
#ifdef ORION_TC_TIMELINE
        const long long tl_ready = clock64();
#endif
        TW(10, asm volatile("bar.sync %0, 256;\n" ::"r"(2 + p) : "memory"));   // my turn at the exponentials
#ifdef ORION_TC_TRACE
        tr_[8] += clock64() - tm0;
        const unsigned long long tx0 = clock64();
#endif
        if (active) {
          const float mb = m_used == -INFINITY ? 0.f : m_used;
          float la[4] = {0.f, 0.f, 0.f, 0.f};   // 4 chains: the mixed adds are dependent
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            pk[c] = pack_bf16(ex2(fmaf(__uint_as_float(sr[2 * c]), a.scale_log2, -mb)),
                              ex2(fmaf(__uint_as_float(sr[2 * c + 1]), a.scale_log2, -mb)));
            // l: the row sum of exactly the bf16 P that enters P.V (reading S17)
            la[c & 3] = add_bf16x2_f32(pk[c], la[c & 3]);
          }
          l_run += (la[0] + la[1]) + (la[2] + la[3]);
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) pk[c] = 0u;
        }
#ifdef ORION_TC_TRACE
        tr_[11] += clock64() - tx0;
#endif
#ifdef ORION_TC_TIMELINE
        if (np < 48) { tl_r[np] = tl_ready; tl_e[np] = clock64(); }   // ready for / end of the turn
#endif
        asm volatile("bar.arrive %0, 256;\n" ::"r"(3 - p) : "memory");   // the other warpgroup's turn
#ifdef ORION_TC_TRACE
        tr_[1] += clock64() - ts0; ts0 = clock64();
#endif
        if (!pv_ok) TW(7, mbar_wait(pv_done + p, (np - 1) & 1));
        tc_fence_after();
        tmem_st32x32(tmem + lane_base + colP(p), pk);
        tc_wait_st();
#ifdef ORION_TC_TRACE
        tr_[2] += clock64() - ts0; ts0 = clock64();
#endif
        if (edge) {   // zero V rows outside [t0, end) once the tile has landed (0 x NaN = NaN);
                      // alias-free: S(j) landed, so K(j) and every earlier V stage, V(j - SV) included, did
          mbar_wait(v_full + (j % SV), (j / SV) & 1);
        }
        if (edge && r < kTok) {
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
        if (edge) fence_proxy_async();   // the zeroed V rows (generic writes) before the PV reads them
        tc_fence_before();
        mbar_arrive(p_full + p);
#ifdef ORION_TC_TRACE
        tr_[3] += clock64() - ts0;
#endif
        had = true;
        ++np;
      }
      }
      if (p == 1 && (cg.ntiles & 1)) {   // odd tile count: WG1 passes its turn
        asm volatile("bar.sync 3, 256;\n" ::: "memory");
        asm volatile("bar.arrive 2, 256;\n" ::: "memory");
      }
#ifdef ORION_TC_TRACE
      const unsigned long long tep0 = clock64();
#endif
      if (p == 0) {                  // next item's Q was gathered one item ahead: publish it
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        fence_proxy_async();
        mbar_arrive(q_full + ((k + 1) & 1));
      }
      // ---- epilogue
      if (had) {
        mbar_wait(pv_done + p, (np - 1) & 1);      // last PV of this WG complete
        tc_fence_after();
      }
      // Both warpgroups publish their (m, l), then each merges O_0 and O_1 over its half of the
      // head dimension (warpgroup p: columns [p D/2, (p + 1) D/2)), so the readout and its
      // scattered row stores take half as long and run on both warpgroups at once.
      xch[((k & 1) * 2 + p) * kRows + r] = make_float2(had ? m_used : -INFINITY, l_run);
      TW(9, asm volatile("bar.sync 1, 256;\n" ::: "memory"));
      {
        const float2 o0 = xch[((k & 1) * 2 + 0) * kRows + r];
        const float2 o1 = xch[((k & 1) * 2 + 1) * kRows + r];
        const bool had0 = __any_sync(0xffffffffu, o0.x > -INFINITY);   // WG0 owned a tile
        const bool had1 = __any_sync(0xffffffffu, o1.x > -INFINITY);   // WG1 owned a tile
        const float M = fmaxf(o0.x, o1.x);
        const float Mb = M == -INFINITY ? 0.f : M;
        const float a0 = had0 ? ex2(o0.x - Mb) : 0.f;
        const float a1 = had1 ? ex2(o1.x - Mb) : 0.f;
        const float l0 = had0 ? o0.y : 0.f, l1 = had1 ? o1.y : 0.f;
        // Direct output (point-prefill plans: the item holds every token of its rows, so this is
        // the row's only partial): out = acc / l in bf16 and lse, no combine pass.
        const float Lr = a0 * l0 + a1 * l1;
        const float inv = Lr > 0.f ? 1.f / Lr : 0.f;
        size_t orow = 0;
        if (a.out && r < w.n_rows) {
          const int rr = w.row_begin + r, rpr = a.lc * a.group;
          const int b = __ldg(a.readers + w.readers_off + rr / rpr);
          orow = (static_cast<size_t>(b) * a.lc + (rr % rpr) / a.group) * a.hq + w.kv_head * a.group + rr % a.group;
        }
        float* dst = a.part_acc + static_cast<size_t>(w.slot0 + r) * D;
        // 16-bit results (bf16 out, fp16 partials) are staged in item k's Q buffer -- free since
        // its Q went to TMEM -- as 128 rows x D/8 16-byte chunks (chunk c of row r at c ^ (r % (D/8)):
        // conflict-free row writes and chunk reads), then copied out with 16-byte row-contiguous
        // stores instead of one scattered 8-byte store per thread and 4 columns.
        const bool staged = a.out || a.part16;
        uint8_t* const ob = smem + L::OFF_Q + (k & 1) * L::QB;
        if (active) {
#pragma unroll 1
          for (int cb = p * (D / 2); cb < (p + 1) * (D / 2); cb += 16) {
            uint32_t o[16], q1[16];
            if (had0) { tmem_ld32x16(tmem + lane_base + colO(0) + cb, o); }
            if (had1) { tmem_ld32x16(tmem + lane_base + colO(1) + cb, q1); }
            tc_wait_ld();
            if (r < w.n_rows) {
#pragma unroll
              for (int c = 0; c < 16; c += 4) {
                float4 v;
                v.x = (had0 ? a0 * __uint_as_float(o[c]) : 0.f) + (had1 ? a1 * __uint_as_float(q1[c]) : 0.f);
                v.y = (had0 ? a0 * __uint_as_float(o[c + 1]) : 0.f) + (had1 ? a1 * __uint_as_float(q1[c + 1]) : 0.f);
                v.z = (had0 ? a0 * __uint_as_float(o[c + 2]) : 0.f) + (had1 ? a1 * __uint_as_float(q1[c + 2]) : 0.f);
                v.w = (had0 ? a0 * __uint_as_float(o[c + 3]) : 0.f) + (had1 ? a1 * __uint_as_float(q1[c + 3]) : 0.f);
                if (staged) {
                  uint2 pk2;
                  if (a.out) {
                    pk2.x = pack_bf16(v.x * inv, v.y * inv);
                    pk2.y = pack_bf16(v.z * inv, v.w * inv);
                  } else {                 // fp16 partial format (plan_format.h): o = acc / l
                    __half2 h0 = __floats2half2_rn(v.x * inv, v.y * inv);
                    __half2 h1 = __floats2half2_rn(v.z * inv, v.w * inv);
                    pk2.x = *reinterpret_cast<uint32_t*>(&h0);
                    pk2.y = *reinterpret_cast<uint32_t*>(&h1);
                  }
                  const int col = cb + c, ch = col >> 3;
                  *reinterpret_cast<uint2*>(ob + r * (D * 2) + ((ch ^ (r & (D / 8 - 1))) << 4) + ((col & 4) << 1)) = pk2;
                } else {
                  *reinterpret_cast<float4*>(dst + cb + c) = v;
                }
              }
            }
          }
        }
        if (p == 0 && r < w.n_rows) {
          if (a.part16) a.part_lse[w.slot0 + r] = Lr > 0.f ? M + log2f(Lr) : -INFINITY;
          else if (!a.out) a.part_ml[w.slot0 + r] = make_float2(M, Lr);
          else if (a.lse) a.lse[orow] = Lr > 0.f ? (M + log2f(Lr)) * 0.69314718055994531f : -INFINITY;
        }
        tc_fence_before();
        mbar_arrive(o_free);
        if (staged) {
          asm volatile("bar.sync 1, 256;\n" ::: "memory");   // the item's rows are staged
          constexpr int CPR = D / 8;                            // 16-byte chunks per row
          const int t = tid - 128;
          for (int idx = t; idx < w.n_rows * CPR; idx += 256) {
            const int row = idx / CPR, ch = idx % CPR;
            const uint4 val = *reinterpret_cast<const uint4*>(ob + row * (D * 2) + ((ch ^ (row & (CPR - 1))) << 4));
            if (a.out) {
              const int rr = w.row_begin + row, rpr = a.lc * a.group;
              const int b = __ldg(a.readers + w.readers_off + rr / rpr);
              __nv_bfloat16* gdst = a.out + ((static_cast<size_t>(b) * a.lc + (rr % rpr) / a.group) * a.hq +
                                             w.kv_head * a.group + rr % a.group) * D;
              reinterpret_cast<uint4*>(gdst)[ch] = val;
            } else {   // (no evict_last hint here: it cost c5 chain 3 %, its L2-shared history)
              reinterpret_cast<uint4*>(a.part_o + static_cast<size_t>(w.slot0 + row) * D)[ch] = val;
            }
          }
          asm volatile("bar.sync 1, 256;\n" ::: "memory");   // buffer read out: WG0 refills it with Q
        }
      }
      release(static_cast<uint32_t>(cur));
      if (p == 1) {
        cur = next_item();
      } else {
        const int nx = pf;
        pf = pf >= 0 ? next_item() : -1;
        load_q(k, pf);               // Q buffer (k & 1) is free: every QK of item k completed
        cur = nx;
      }
#ifdef ORION_TC_TRACE
      tr_[4] += clock64() - tep0;
#endif
      ++k;
    }
    if (p == 0) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    if (p == 0) asm volatile("bar.sync 2, 256;\n" ::: "memory");   // the token WG1 passed last
    if ((warp & 3) < 2) TRACE_DUMP("softmax");
#ifdef ORION_TC_TIMELINE
    if (blockIdx.x == 0 && (warp & 3) == 0 && lane == 0)
      for (uint32_t i = 0; i < min(np, 48u); ++i) printf("TL p=%d np=%u ready=%lld end=%lld\n", p, i, tl_r[i], tl_e[i]);
#endif
#ifdef ORION_TC_TRACE
    if (warp == 4 && lane == 0)   // per-CTA balance: total cycles, tiles, items of warpgroup 0
      printf("CTA %d tot %llu tiles %u items %u\n", blockIdx.x, clock64() - tr_t0, np, k);
#endif
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kWarpAlloc) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
  if (threadIdx.x == 0) release_work_counter(a.work_counter);
}

}  // namespace tc

// ------------------------------------------------------------------------------ host launcher
namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
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

bool make_map(CUtensorMap* m, const void* base, int d, int64_t rows, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(d) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

template <int D>
orion_status launch_split_tc(const PlanHeader* h, const TcArgs& a, const void* k, const void* v,
                             int32_t num_pages, cudaStream_t st) {
  const int num_sms = current_device_sms();
  const cudaError_t attr_err = ensure_dynamic_smem(reinterpret_cast<const void*>(tc::split_tc_kernel<D>),
                                                   tc::Smem<D>::BYTES + 1024);
  if (attr_err != cudaSuccess)
    return fail(ORION_ERR_CUDA, "cudaFuncSetAttribute(split_tc): %s", cudaGetErrorString(attr_err));
  CUtensorMap mk, mv, mk16, mv16;
  const int64_t rows = static_cast<int64_t>(num_pages) * h->num_kv_heads * a.kvs * h->page_size;
  const int big = std::min(tc::kTok, h->page_size);
  if (!make_map(&mk, k, D, rows, big) || !make_map(&mv, v, D, rows, big) ||
      !make_map(&mk16, k, D, rows, tc::kBox) || !make_map(&mv16, v, D, rows, tc::kBox))
    return fail(ORION_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  if (h->paired) {
    const CUtensorMap maps[4] = {mk, mv, mk16, mv16};
    return launch_split_pair<D>(h, a, maps, st);
  }
  int grid = std::min<int>(h->n_items, num_sms > 0 ? num_sms : 148);
  if (h->max_ctas > 0) grid = std::min(grid, h->max_ctas);
  if (!a.work_counter) return fail(ORION_ERR_INVALID_ARG, "split_tc without a work counter");
  cudaError_t e = launch_pdl(tc::split_tc_kernel<D>, dim3(grid), dim3(tc::kThreadsTC), tc::Smem<D>::BYTES + 1024, st,
                             mk, mv, mk16, mv16, a);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ORION_ERR_CUDA, "split_tc_kernel: %s", cudaGetErrorString(e));
  return ORION_OK;
}

template orion_status launch_split_tc<64>(const PlanHeader*, const TcArgs&, const void*, const void*, int32_t,
                                          cudaStream_t);
template orion_status launch_split_tc<128>(const PlanHeader*, const TcArgs&, const void*, const void*, int32_t,
                                           cudaStream_t);

}  // namespace orion
