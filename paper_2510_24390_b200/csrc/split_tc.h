// split_tc.h — internal interface between the launchers (kernels.cu) and the tcgen05 split
// kernel (split_tc.cu).  Product-side only.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/orion.h"
#include "plan_format.h"

namespace orion {

orion_status fail(orion_status code, const char* fmt, ...);
// Debug-build (ORION_CHECK) report of an append whose own-run page id is outside [0, num_pages):
// begin returns the device record to pass to the kernel (nullptr in release builds), end reads it.
int* append_check_begin(cudaStream_t st);
orion_status append_check_end(cudaStream_t st, const char* what);
orion_status check_shape_public(const orion_attn_shape* s);

// Per-device launch setup, thread-safe: the SM count of the current device, and the opt-in
// dynamic shared-memory size of `func` on it (set once per (device, function); the attribute is
// per device, so a process driving several GPUs needs it on each).
int current_device_sms();
cudaError_t ensure_dynamic_smem(const void* func, int bytes);

// Programmatic dependent launch (PDL).  Kernels of one expansion step (append -> split ->
// combine -> next layer's append) are launched with programmatic stream serialization: the next
// kernel may be scheduled while the previous one drains, runs its data-independent prologue
// (barrier init, TMEM allocation, smem zeroing), and blocks in pdl_wait() -- which returns only
// once the previous grid has completed and its memory is visible -- before it touches global
// memory.  pdl_trigger() lets the next grid be scheduled early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// Work counter of the persistent split kernels: counter[0] hands out items (atomicAdd), counter[1]
// counts finished CTAs.  The last CTA to finish zeroes both, so the next launch on the same
// workspace starts from zero with no memset between the previous kernel and this one (a memset
// node would break the programmatic-dependent-launch chain append -> split).  The workspace's
// counter words must be zero before its first launch (include/orion.h).  Called by one thread per
// CTA after the CTA's last access to the counter.
__device__ __forceinline__ void release_work_counter(int32_t* counter) {
  __threadfence();
  if (atomicAdd(counter + 1, 1) == static_cast<int>(gridDim.x) - 1) {
    atomicExch(counter, 0);
    atomicExch(counter + 1, 0);
  }
}
// The fused append's launch epoch (FusedAppend): advanced by the last CTA of a fused launch, so
// the next fused launch's CTAs all read epoch + 1 as their flag value.
__device__ __forceinline__ void release_work_counter(int32_t* counter, bool advance_epoch) {
  __threadfence();
  if (atomicAdd(counter + 1, 1) == static_cast<int>(gridDim.x) - 1) {
    atomicExch(counter, 0);
    atomicExch(counter + 1, 0);
    if (advance_epoch) atomicAdd(counter + kAppendEpochWord, 1);
  }
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// K1 fused into the swap-AB split kernel (orion_expand_step on a plan without big items): every
// CTA first appends the new K/V rows of its share of the branches and releases each branch's flag
// (flags[b] = this launch's epoch + 1); a range growing with branch b reads own_len[b] only once
// flags[b] carries that value (acquire; the appended rows reach its TMA loads through proxy
// fences).  No grid-wide barrier: an item waits only for the branches it reads.  The epoch sits in
// work counter word kAppendEpochWord, the flags after the counters (plan_format.h).
// enabled = 0: no append in the kernel.
struct FusedAppend {
  const __nv_bfloat16* k_new;
  const __nv_bfloat16* v_new;
  __nv_bfloat16* k_cache;
  __nv_bfloat16* v_cache;
  const int32_t* own_pt_off;
  const int32_t* own_cap;
  int32_t* own_len;       // the array TcArgs::own_len points to
  int32_t* epoch;         // work counter word kAppendEpochWord
  int32_t* flags;         // [n_branches]
  int32_t* err;           // debug build: first branch whose target page is out of range
  int32_t n_branches, mode, num_pages, enabled;
  // K3 as the same launch's last phase (merge = 1): after a grid barrier (sense reversal on work
  // counter words kBarCountWord / kBarGenWord) every CTA merges a share of the rows' fp16
  // partials (merge16.h) into out / lse, so a short step is one launch.
  int32_t merge, n_rows;
  const int32_t* comb_off;
  const int32_t* comb_slot;
  __nv_bfloat16* out;
  float* lse;
};

struct TcArgs {
  const WorkItem* items;
  const Range* ranges;    // multi-range items (kItemRanges)
  const int32_t* readers;
  const __nv_bfloat16* q;
  const int32_t* page_table;
  const int32_t* own_len;
  float* part_acc;        // fp32 partial format (split_tc)
  float2* part_ml;
  __half* part_o;         // fp16 partial format (split_tct)
  float* part_lse;
  int32_t n_items, hq, hkv, group, page_shift;
  int32_t kvs;            // (page, kv head) block stride in blocks: 1 separate K/V, 2 interleaved
  int32_t lc;             // query rows per reader and q head: 1 (decode) or Lc (point prefill)
  __nv_bfloat16* out;     // non-null: every row has exactly one partial (a point-prefill plan) and
  float* lse;             // the epilogue writes out = acc / l (bf16) and lse directly: no combine
  float scale_log2;
  int32_t* work_counter;  // items (split_tct) / pair units (split_pair) handed out by atomicAdd
  int32_t part16;         // rows-on-lanes kernel on a hybrid plan's big items: write the fp16 partial
                          // format (part_o = acc / l, part_lse = m + log2 l) instead of fp32
  FusedAppend app;
  int32_t pdl_late;       // second kernel of a hybrid step: it may start once the first kernel has
                          // passed its own dependency wait (the step's inputs are complete) and waits
                          // for the first kernel's completion only before it exits
};

template <int D>
orion_status launch_split_tc(const PlanHeader* h, const TcArgs& a, const void* k, const void* v,
                             int32_t num_pages, cudaStream_t st);

// Point-prefill plans with paired items (PlanHeader::paired): split_pair.cu.  maps = K, V tensor
// maps with full-tile boxes, then K, V with 16-row boxes.
template <int D>
orion_status launch_split_pair(const PlanHeader* h, const TcArgs& a, const CUtensorMap maps[4], cudaStream_t st);

orion_status launch_split_tct(const PlanHeader* h, const TcArgs& a, const void* k, const void* v,
                              int32_t num_pages, cudaStream_t st);

}  // namespace orion
