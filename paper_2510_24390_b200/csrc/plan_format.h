// plan_format.h — device plan layout shared by the host planner (host.cpp) and the kernels
// (kernels.cu).  Product-side only; the oracle never sees it.
//
// A plan is one contiguous byte buffer:
//   PlanHeader | WorkItem[n_items] | readers[n_reader_entries] (int32 branch ids)
//              | comb_off[n_rows + 1] (int32) | comb_slot[n_partials] (int32) | Range[n_ranges]
// Workspace (caller-allocated, device), one partial (softmax state of one query row over one
// work item's tokens) per slot, in one of two formats fixed by the plan's variant:
//   fp32 (kVariantTC, kVariantMmaSync):
//     part_acc fp32 [n_partials][head_dim] | part_ml fp32 [n_partials][2]  (m in log2 units, l)
//     the row's partial output is acc / l, its log2-sum-exp m + log2(l)
//   fp16 (kVariantTCT):
//     part_o fp16 [n_partials][head_dim] (= acc / l) | part_lse fp32 [n_partials] (m + log2 l)
//     half the bytes; fp16's 2^-11 relative rounding is 4x below the bf16 rounding of out.  o is
//     a convex combination of V rows, so |o| <= max |V|: V entries must stay within fp16 range
//     (|v| <= 65504; include/orion.h).
// acc_bytes = byte offset of the second array.  tcgen05 plans end the workspace with 16 bytes at
// counter_off: the split kernel's atomic item counter, zeroed by the launcher before each launch.
#pragma once
#include <stdint.h>

namespace orion {

constexpr int32_t kPlanMagic = 0x314e524f;  // "ORN1"
constexpr int32_t kPlanVersion = 1;
constexpr int kRowsPerItemTC = 128;  // query rows per work item, tcgen05 kernel (MMA M = 128)
constexpr int kRowsPerItemMMA = 64;  // query rows per work item, mma.sync kernel (4 warps x m16)
constexpr int kRowsPerItem = kRowsPerItemMMA;  // smem sizing of the mma.sync kernel
constexpr int kRowsPerItemTCT = 64;  // query rows per work item, transposed tcgen05 kernel (MMA N)
constexpr int kRowsPerItemBig = 128; // hybrid decode plans: rows of a big item (rows-on-lanes kernel, MMA M)
enum : int32_t { kVariantTC = 0, kVariantMmaSync = 1, kVariantTCT = 2 };
inline bool partials_fp16(int32_t variant) { return variant == kVariantTCT; }
constexpr int32_t kItemCausal = 1;
constexpr int32_t kItemRanges = 2;
constexpr int32_t kRangeMasked = 4;   // Range only: readers_mask (pad_[0]) selects the item's readers
                                      // (bit i: the item's i-th reader) that read this range
constexpr int64_t kMergeTokens = 8192;   // token cap of a merged multi-range decode item
// Workspace tail of the tcgen05 kernels' counters: words 0-1 (item counter, done count) of the
// first split kernel, words 4-5 of a hybrid plan's second; the fused append's launch epoch at word
// kAppendEpochWord (its own cache line), then one append flag per branch (kCounterBytes on).
constexpr int64_t kCounterBytes = 256;
constexpr int kAppendEpochWord = 32;
constexpr int kBarCountWord = 40, kBarGenWord = 48;   // the fused merge's grid barrier
constexpr int64_t kSmallStepTokens = 1024;   // small-step split: below this many tokens per item at 2 items per SM
constexpr int kTileTokens = 64;    // tokens per pipeline stage in the split kernel

struct PlanHeader {
  int32_t magic, version;
  int32_t n_branches, num_q_heads, num_kv_heads, head_dim, page_size, group;
  int32_t n_items, n_partials, n_rows, n_reader_entries;
  int64_t items_off, readers_off, comb_off_off, comb_slot_off;  // byte offsets from plan start
  int64_t plan_bytes, workspace_bytes, acc_bytes;                // acc_bytes = part_ml offset
  int64_t n_pieces, unique_tokens, logical_tokens;
  float sm_scale;
  int32_t variant;  // kVariantTCT (default, d = 128), kVariantTC (d = 64 or ORION_PLAN_ROWS_ON_LANES),
                    // kVariantMmaSync (ORION_PLAN_MMA_SYNC)
  int32_t max_ctas; // persistent split kernels: grid cap (opts->num_sms; 0 = all SMs)
  int32_t prefill_rows;  // 0: decode plan; Lc: point-prefill plan (rows = branch x Lc x Hq)
  int64_t ranges_off;    // byte offset of Range[n_ranges] (multi-range items)
  int32_t n_ranges;
  int32_t paired;
  int64_t streamed_tokens;  // orion_plan_stats::streamed_tokens
  int64_t counter_off;      // tcgen05 plans: workspace byte offset of the split kernels' work counters
                            // (16 bytes each: the first kernel's, then a hybrid plan's second one)
  int32_t n_big;            // kVariantTCT hybrid plans: items [0, n_big) have 65..128 rows and run on the
                            // rows-on-lanes kernel (fp16 partials); [n_big, n_items) on the swap-AB kernel
  int32_t pad0;
  uint64_t plan_id;         // FNV-1a of the serialised plan body: the host and device copies must match
};        // prefill plans: items 2u, 2u+1 run as one pair unit (split_pair.cu);
                         // items[2u].t1 = number of leading ranges the two lists share
static_assert(sizeof(PlanHeader) % 16 == 0, "header must keep 16-byte alignment");

// One split-kernel work item: tokens [t0, min(t1, own_len[dyn])) of the page run at pt_off,
// kv head `kv_head`, query rows [row_begin, row_begin + n_rows) of the piece's row space.  With
// R = Lc * group rows per reader (Lc = 1 for decode, prefill_rows for a prefill plan), row r ->
// reader branch b = readers[readers_off + r / R], content position i = (r % R) / group, q head
// h = kv_head*group + r % group; its output row is (b * Lc + i) * Hq + h.
// Row r writes partial slot slot0 + (r - row_begin).
struct WorkItem {
  int32_t pt_off, t0, t1, dyn;
  int32_t kv_head, readers_off, row_begin, n_rows;
  int32_t slot0, piece, flags, n_ranges;   // flags: kItemCausal, kItemRanges
};

// A token range of a multi-range item (kItemRanges: the item streams ranges[pt_off ..
// pt_off + n_ranges) of the plan in order, as one accumulation): tokens [t0, min(t1,
// own_len[dyn])) of the page run at pt_off; flags & kItemCausal: row i sees tokens < t0 + i + 1;
// flags & kRangeMasked: only rows of the readers whose bit is set in pad_[0] see the range (hybrid
// plans' big items, rows-on-lanes kernel only: a reader block's ranges with different reader
// subsets streamed as one accumulation; at most 32 readers per such item).
struct Range {
  int32_t pt_off, t0, t1, dyn, flags, pad_[3];
};
static_assert(sizeof(Range) == 32, "Range is 2 x 16 bytes");
static_assert(sizeof(WorkItem) == 48, "WorkItem is 3 x 16 bytes");

}  // namespace orion
