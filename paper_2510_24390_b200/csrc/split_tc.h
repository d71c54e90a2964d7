// split_tc.h — internal interface between the launchers (kernels.cu) and the tcgen05 split
// kernel (split_tc.cu).  Product-side only.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/orion.h"
#include "plan_format.h"

namespace orion {

orion_status fail(orion_status code, const char* fmt, ...);

struct TcArgs {
  const WorkItem* items;
  const int32_t* readers;
  const __nv_bfloat16* q;
  const int32_t* page_table;
  const int32_t* own_len;
  float* part_acc;        // fp32 partial format (split_tc)
  float2* part_ml;
  __half* part_o;         // fp16 partial format (split_tct)
  float* part_lse;
  int32_t n_items, hq, hkv, group, page_shift;
  float scale_log2;
};

template <int D>
orion_status launch_split_tc(const PlanHeader* h, const TcArgs& a, const void* k, const void* v,
                             int32_t num_pages, cudaStream_t st);

orion_status launch_split_tct(const PlanHeader* h, const TcArgs& a, const void* k, const void* v,
                              int32_t num_pages, cudaStream_t st);

}  // namespace orion
