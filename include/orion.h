/*
 * orion.h — C ABI of the B200-native hot path of Orion's content parallel expansion
 * (Gao et al., arXiv 2510.24390, "Improving LLM Reasoning via Dependency-Aware Query
 * Decomposition and Logic-Parallel Content Expansion").
 *
 * The library implements ONE expansion decode step (Alg. 1 l.16 "LLM processes
 * the running node set R"; §3.3 PAPER.md:387 yellow "LLM Decoding" bars) for every point
 * ("branch") of every in-flight query at once, plus the host-side DAG work that feeds it:
 *
 *   orion_dag_waves      Alg. 1 l.1-8 + Eq. (1)-(3): validate a point DAG, split points into
 *                        Prefill/Decode stages, compute expansion levels and per-branch
 *                        segment lists (which KV spans each branch attends to).
 *   orion_bind_segments  map symbolic segment lists to token ranges of a paged KV cache.
 *   orion_expand_plan    cut the bound segments into shared pieces (maximal token ranges with
 *                        a fixed reader set) and emit the device work plan.
 *   orion_kv_append      write each branch's new-token K/V into its own pages (device).
 *   orion_expand_step    orion_kv_append + orion_expand_attn in one call (device; on short
 *                        steps one launch: append, split and combine in the split kernel).
 *   orion_expand_attn    dependency-masked batched GQA decode attention over the paged bf16
 *                        cache; each shared piece is read from HBM once per (query, kv head)
 *                        group (device; split kernel + combine kernel).
 *
 * Conventions (all functions):
 *  - Every buffer is caller-owned.  The library keeps no pointer after a call returns, has no
 *    global state (except a thread-local error string), never allocates device memory and never
 *    synchronises a stream.  Device functions only enqueue work on `stream`.
 *  - Errors are returned as orion_status codes; nothing is thrown, aborted or exited.  On a
 *    non-OK status, orion_last_error() returns a thread-local human-readable message.
 *  - Two-call sizing: when an output buffer is too small the function returns
 *    ORION_ERR_CAPACITY and writes the required size to the *_needed argument.
 *  - Host functions are pure and thread-safe; a plan is immutable once built and may be used by
 *    any number of launches.  Host functions run without a GPU.
 *  - Point ids are 1..n_points within a query.  Branch indices are global
 *    0..n_branches-1 over all queries of one call.
 *  - KV cache layout, per layer: K and V each bf16 [num_pages][num_kv_heads][page_size][head_dim].
 *    q and out: bf16 [n_branches][num_q_heads][head_dim]; lse: fp32 [n_branches][num_q_heads].
 *    GQA mapping: q head h reads kv head h / (num_q_heads / num_kv_heads) (reading S16).
 */
#ifndef ORION_H_
#define ORION_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t orion_status;
enum {
  ORION_OK = 0,
  ORION_ERR_INVALID_ARG = 1,   /* bad pointer, size, kind, policy, overlap, empty context */
  ORION_ERR_CYCLE = 2,         /* the point DAG has a cycle (SPEC.md:67 CycleDetected) */
  ORION_ERR_UNKNOWN_POINT = 3, /* an edge names a point outside 1..n */
  ORION_ERR_CAPACITY = 4,      /* output buffer too small; see *_needed */
  ORION_ERR_UNSUPPORTED = 5,   /* shape not compiled in / segment pattern not supported */
  ORION_ERR_CUDA = 6           /* a CUDA launch failed; message from cudaGetErrorString */
};

/* Edge kinds (§3.3 "Null, Contextual, and Dependent"). */
enum { ORION_EDGE_NULL = 0, ORION_EDGE_CONTEXTUAL = 1, ORION_EDGE_DEPENDENT = 2 };

/* Dependency-set policies (readings S6-S8).
 * ANCESTORS: a branch attends to every transitive ancestor; FULL span if the ancestor's decode
 *            happens-before the branch's prefill in the stage graph, else CONTENT span.
 * PARENTS_EQ3: Eq. (2)/(3) literally: direct parents only, OUTPUT span for a
 *            Dependent edge, CONTENT span for a Contextual edge. */
enum { ORION_POLICY_ANCESTORS = 0, ORION_POLICY_PARENTS_EQ3 = 1 };

/* Symbolic segment kinds.  A point k's KV segment S_k = [P_k content (Lc_k tokens) | Output_k]. */
enum {
  ORION_SEG_PREFIX = 0,  /* the query's shared prefix, Prompt_Pre of Eq. (2) (reading S13) */
  ORION_SEG_CONTENT = 1, /* S_k[0, Lc_k)          f(k,j) = P_k (Eq. 3, Contextual)          */
  ORION_SEG_FULL = 2,    /* S_k[0, T_k)           ANCESTORS span of a Dependent ancestor    */
  ORION_SEG_OUTPUT = 3,  /* S_k[Lc_k, T_k)        f(k,j) = Output_k (Eq. 3, Dependent)      */
  ORION_SEG_OWN = 4      /* S_j[0, T_j)           the branch's own tokens incl. the new one */
};

/* Stage phases in the wave listing (Alg. 1 l.8 "split each node into prefilling and decoding"). */
enum { ORION_PHASE_PREFILL = 0, ORION_PHASE_DECODE = 1 };

/* kv_append modes.  ADVANCE: write at own_len[b], then own_len[b] += 1 (a real decode step).
 * REWRITE: write at own_len[b]-1, lengths unchanged (stationary steady-state benchmarking). */
enum { ORION_APPEND_ADVANCE = 0, ORION_APPEND_REWRITE = 1 };

/* from = prerequisite point k, to = dependent point j. */
typedef struct { int32_t from, to, kind; } orion_edge;

/* One symbolic list entry.  point = 0 for PREFIX, else the query-local point id. */
typedef struct { int32_t kind, point; } orion_segref;

/* One bound segment: tokens [start, start + len_eff) of the page run that starts at
 * page_table[pt_off]; token position t lives on page page_table[pt_off + t / page_size],
 * row t % page_size.  dyn = -1: len_eff = len (static).  dyn = b >= 0: the segment grows with
 * branch b's decode: len_eff = clamp(own_len[b] - start, 0, len), i.e. len is a capacity bound. */
typedef struct { int32_t pt_off, start, len, dyn; } orion_seg;

typedef struct {
  int32_t num_q_heads;   /* Hq */
  int32_t num_kv_heads;  /* Hkv; Hq % Hkv == 0 */
  int32_t head_dim;      /* 64 or 128 */
  int32_t page_size;     /* power of two in [16, 256] */
  float sm_scale;        /* softmax scale; <= 0 selects 1/sqrt(head_dim) (reading S16) */
  int32_t kv_interleaved; /* 0: K and V caches are separate [num_pages][Hkv][P][d] arrays.
                             1: one [num_pages][Hkv][2][P][d] array (K and V of a (page, kv head)
                             adjacent: a decode tile's K and V are one 32 KB run); pass
                             k_cache = base and v_cache = base + P*d elements */
} orion_attn_shape;

/* Per query: its points are global branches [branch0, branch0 + n_points). */
typedef struct { int32_t n_points, branch0, prefix_pt_off, prefix_len; } orion_query_desc;

/* Per global branch (= point): its page run, content length Lc and capacity in tokens. */
typedef struct { int32_t pt_off, content_len, capacity; } orion_point_desc;

/* Plan flags (split-kernel variant).  Default: the transposed tcgen05/TMEM/TMA kernel (tokens on
 * the MMA M dimension, <= 64 query rows per work item; head_dim 128) — head_dim 64 uses the
 * rows-on-lanes tcgen05 kernel.  ORION_PLAN_ROWS_ON_LANES forces the rows-on-lanes tcgen05 kernel
 * (<= 128 rows per item); ORION_PLAN_MMA_SYNC the legacy mma.sync m16n8k16 + cp.async kernel
 * (<= 64 rows per item).  All variants compute the same result (same plan semantics). */
enum { ORION_PLAN_MMA_SYNC = 1, ORION_PLAN_ROWS_ON_LANES = 2, ORION_PLAN_NO_MERGE = 4, ORION_PLAN_PAIR = 8,
       ORION_PLAN_NO_HYBRID = 16 };
/* Hybrid decode plans (default for head_dim 128): readers are grouped into blocks of up to 128 query
 * rows; a block's items with 65..128 rows run on the rows-on-lanes kernel (one 128-row MMA tile
 * reads each K/V tile once for all of them), items with <= 64 rows on the swap-AB kernel -- two
 * launches, both writing the fp16 partial format the combine reads.  ORION_PLAN_NO_HYBRID keeps
 * every item on the swap-AB kernel (<= 64 rows per item). */
/* ORION_PLAN_NO_MERGE: one work item per (piece, kv head, chunk, row block) -- without it, the
 * tcgen05 decode plans group rows into fixed reader blocks and merge every chunk one block reads
 * with the same reader subset into a multi-range item (one partial per row for the lot).
 * ORION_PLAN_PAIR (point-prefill plans, opt-in): consecutive items (two readers of one kv head)
 * run as a pair on one CTA, and every K/V tile of the ranges their lists share (the query's
 * prefix, common dependencies) is streamed once for both -- 38 % fewer K/V bytes through L2 on
 * c4, but measured slower than one item per pass, so not the default. */

typedef struct {
  int32_t num_sms;        /* SMs the persistent split kernel may occupy (grid cap, e.g. to leave
                             SMs to a co-scheduled prefill stream); <= 0 = all SMs */
  int32_t chunk_tokens;   /* max tokens per work item along a piece; <= 0 selects the default */
  int32_t flags;          /* ORION_PLAN_* bits, 0 = defaults */
  int32_t prefill_rows;   /* 0: decode plan (one query row per branch and q head).  Lc > 0: point-
                             prefill plan (orion_point_prefill_attn): every branch contributes the
                             Lc content tokens of its point as query rows; its OWN segment (the one
                             whose dyn == the branch) is read causally over [start, start + Lc) and
                             must have len >= Lc; all points must have content length Lc. */
} orion_plan_opts;

typedef struct {
  int64_t n_items;          /* split-kernel work items */
  int64_t n_pieces;         /* shared pieces (token range x reader set), per kv head counted once */
  int64_t n_partials;       /* fp32 partial rows written by the split kernel */
  int64_t n_rows;           /* n_branches * num_q_heads */
  int64_t unique_tokens;    /* sum of piece capacities (upper bound of unique KV tokens per kv head) */
  int64_t logical_tokens;   /* sum over branches of their context capacity (per kv head) */
  int64_t plan_bytes;
  int64_t workspace_bytes;
  int64_t streamed_tokens;  /* K/V token rows the split kernel streams, all kv heads (capacity
                               bound): a paired prefill plan streams its pairs' shared ranges once */
  int64_t paired;           /* 1: point-prefill plan run as item pairs (ORION_PLAN_PAIR) */
  int64_t n_big;            /* hybrid decode plan: items run on the rows-on-lanes kernel (65..128 rows) */
} orion_plan_stats;

/*
 * orion_dag_waves — Alg. 1 l.1-8, Eq. (1) generalised to
 * longest-path expansion levels (reading S10), and Eq. (2)/(3) read as KV
 * segment lists (readings S6-S9).  Host only, no CUDA.
 *
 *  n_points            N >= 1; points are 1..N.
 *  edges[n_edges]      typed edges; Null edges are dropped, duplicates merged, Dependent
 *                      dominates Contextual on the same pair (reading S5).
 *  policy              ORION_POLICY_*.
 *  pre_level[N], dec_level[N]  out: level of Prefill(i) / Decode(i) (index i-1).
 *  n_levels[1]         out: 1 + max level.
 *  wave_offsets[2N+1]  out, nullable: CSR over levels (only n_levels+1 entries are written).
 *  wave_stages[2N]     out, nullable: stages in wave order, each wave sorted by (point, Pre<Dec),
 *                      encoded as point * 2 + phase.
 *  seg_offsets[N+1]    out: CSR over points of the segment lists.
 *  segs[segs_cap]      out: [PREFIX] + dependencies ascending by point id + [OWN(j)].
 *  segs_needed[1]      out: total list entries (always written when validation passed).
 *  err_info[err_cap]   out, nullable: on CYCLE the point ids of one cycle in order; on
 *                      UNKNOWN_POINT / bad kind the offending edge index.  err_info is written up
 *                      to err_cap entries; the first entry not written is left untouched.
 * Errors: INVALID_ARG (N < 1, null pointer, kind outside 0..2 — checked per edge in input order
 * before the point-range check of the same edge), UNKNOWN_POINT, CYCLE (a non-Null self-loop is a
 * 1-cycle), CAPACITY (segs_cap < *segs_needed; levels are still written).
 */
orion_status orion_dag_waves(int32_t n_points, const orion_edge* edges, int32_t n_edges,
                             int32_t policy, int32_t* pre_level, int32_t* dec_level,
                             int32_t* n_levels, int32_t* wave_offsets, int32_t* wave_stages,
                             int32_t* seg_offsets, orion_segref* segs, int32_t segs_cap,
                             int32_t* segs_needed, int32_t* err_info, int32_t err_cap);

/*
 * orion_bind_segments — physical binding of symbolic lists (reading S7/S19; SURVEY.md
 * §8(c) O2).  Host only.
 *   PREFIX     -> {prefix_pt_off, 0, prefix_len, -1}
 *   CONTENT(k) -> {pt_off_k, 0, Lc_k, -1}
 *   FULL(k)    -> {pt_off_k, 0, cap_k, dyn = branch of k}
 *   OUTPUT(k)  -> {pt_off_k, Lc_k, cap_k - Lc_k, dyn = branch of k}
 *   OWN(j)     -> {pt_off_j, 0, cap_j, dyn = branch of j}
 *  queries[n_queries]       query descriptors; branches of different queries must not overlap.
 *  points[n_branches]       per-branch page runs (n_branches = max(branch0 + n_points)).
 *  seg_offsets[n_branches+1], refs[]  global CSR: branch b's list is refs[seg_offsets[b] ..
 *                           seg_offsets[b+1]), with query-local point ids (as produced by
 *                           orion_dag_waves for that query).
 *  segs_out[seg_offsets[n_branches]]  out.
 * Errors: INVALID_ARG (null pointers, bad kind, point outside its query, Lc > capacity,
 * negative sizes).
 */
orion_status orion_bind_segments(int32_t n_queries, const orion_query_desc* queries,
                                 int32_t n_branches, const orion_point_desc* points,
                                 const int32_t* seg_offsets, const orion_segref* refs,
                                 orion_seg* segs_out);

/*
 * orion_expand_plan — host planner for orion_expand_attn.  Groups segments by page run (pt_off),
 * cuts every run at all segment boundaries into pieces, attaches to each piece its reader set
 * (the branches whose lists cover it), merges neighbours with equal reader sets, splits pieces
 * into work items of at most opts->chunk_tokens tokens and 64 query rows, orders work items
 * longest-first, and lays out the combine lists.  Host only; the caller uploads plan_buf to the
 * device (any 16-byte aligned copy) and keeps the host copy for launches.
 *  h_seg_offsets[n_branches+1], h_segs[]  bound segments (orion_bind_segments).
 *  h_own_len[n_branches]  nullable: current lengths, used to validate that a static segment
 *                         overlapping a growing (dyn) segment never reaches past own_len.
 *  plan_buf[plan_cap]     out (16-byte aligned); plan_needed / workspace_needed out (bytes).
 * Errors: INVALID_ARG (overlapping segments in one branch list; a branch with an empty
 * capacity context; dyn out of range), UNSUPPORTED (two different dyn branches on one page run;
 * shape not supported), CAPACITY.
 */
orion_status orion_expand_plan(const orion_attn_shape* shape, int32_t n_branches,
                               const int32_t* h_seg_offsets, const orion_seg* h_segs,
                               const int32_t* h_own_len, const orion_plan_opts* opts,
                               void* plan_buf, size_t plan_cap, size_t* plan_needed,
                               size_t* workspace_needed);

/* orion_plan_stats — read counters of a built (host) plan. */
orion_status orion_plan_get_stats(const void* h_plan, orion_plan_stats* out);

/*
 * orion_kv_append — KV-cache write of each branch's new token (reading S15).
 * Device; enqueued on `stream`.  One thread block per branch; bit-exact bf16 copy.
 *  k_new, v_new   bf16 [n_branches][Hkv][d] (device).
 *  k_cache, v_cache  bf16 [num_pages][Hkv][P][d] (device, one layer).
 *  own_pt_off[n_branches], own_cap[n_branches]  device int32: branch page runs and capacities.
 *  page_table     device int32;  num_pages  pages in the caches.
 *  own_len[n_branches]  device int32, in/out.  ADVANCE: write slot own_len, then own_len += 1.
 *                 REWRITE: write slot own_len - 1.  A slot outside [0, own_cap), or a page id
 *                 outside [0, num_pages), is skipped and own_len is left unchanged (no write
 *                 outside the caches ever happens); the debug build (ORION_CHECK) reports such a
 *                 page id as INVALID_ARG (it synchronises the stream).
 * Errors: INVALID_ARG (null/unaligned pointers, bad mode, num_pages < 1), UNSUPPORTED (shape), CUDA.
 */
orion_status orion_kv_append(const orion_attn_shape* shape, int32_t n_branches,
                             const void* k_new, const void* v_new, void* k_cache, void* v_cache,
                             const int32_t* own_pt_off, const int32_t* own_cap,
                             const int32_t* page_table, int32_t num_pages, int32_t* own_len,
                             int32_t mode, void* stream);

/*
 * orion_expand_attn — one dependency-masked, batched GQA decode-attention step (PAPER.md:337
 * Alg. 1 l.16; reading S21: every branch of the plan decodes one token).  For each branch b and
 * q head h:  out[b,h] = softmax(sm_scale * q[b,h] . K_ctx(b)^T) . V_ctx(b), where ctx(b) is the
 * concatenation of b's bound segments with their current (dyn) lengths; lse[b,h] = natural-log
 * sum-exp of the scaled scores.  The current token's K/V must already be appended.
 * Device; enqueues the split kernel (partials per work item) and the combine kernel (LSE merge in
 * plan order, RNE to bf16) on `stream`.  The default (swap-AB, head_dim 128) kernel keeps each
 * partial as fp16 o = acc / l, a convex combination of V rows: V entries must lie within fp16
 * range (|v| <= 65504) -- far above LLM value activations; ORION_PLAN_ROWS_ON_LANES keeps fp32
 * partials for inputs that do not.
 *  q, out        bf16 [n_branches][Hq][d] (device).   lse  fp32 [n_branches][Hq], nullable.
 *  k_cache, v_cache, num_pages, page_table  as for orion_kv_append.
 *  own_len       device int32 [n_branches] (dyn segment lengths).
 *  h_plan, d_plan  the host plan and its device copy (same bytes).
 *  workspace     device, >= workspace_needed bytes from orion_expand_plan, 16-byte aligned, and
 *                ZEROED before its first use (e.g. allocated with zeros).  The split kernels keep
 *                their work-distribution counters in its last 256 bytes; every launch leaves them zero
 *                again (the last CTA resets it, so no memset runs between launches), so a
 *                workspace serves one launch at a time, in stream order.
 * Errors: INVALID_ARG (null/unaligned pointers, plan/shape mismatch, workspace too small),
 * UNSUPPORTED (shape), CUDA.  Page-table contents are not checked by the release library (K/V
 * tiles are read by TMA, which zero-fills a box outside the cache instead of faulting): the debug
 * build liborion_check.so (`make check`, select with ORION_LIB) walks every work item's ranges on
 * the device before each split launch and returns INVALID_ARG naming the item for a page id
 * outside [0, num_pages), a negative own_len or a dynamic range past n_branches; it synchronises
 * `stream` (not CUDA-graph capturable).
 */
orion_status orion_expand_attn(const orion_attn_shape* shape, int32_t n_branches, const void* q,
                               void* out, float* lse, const void* k_cache, const void* v_cache,
                               int32_t num_pages, const int32_t* page_table,
                               const int32_t* own_len, const void* h_plan, const void* d_plan,
                               void* workspace, size_t workspace_bytes, void* stream);

/*
 * orion_expand_step — one whole expansion decode step for one layer: orion_kv_append of every
 * branch's new token followed by orion_expand_attn over the same plan (Alg. 1 l.16;
 * SURVEY.md §8(a) a5 + a6 + a7).  Results are those of the two calls in order (outputs bitwise
 * equal; tests/test_gpu_parity.py::test_expand_step_equals_append_then_attn).
 * Device; enqueued on `stream`.  With the release library, a stream of the whole device's context
 * (not a green-context partition: the fused launch's CTAs wait on each other, so all of them must
 * be resident at once), a plan on the default swap-AB kernel without rows-on-lanes items (no
 * `n_big`; every plan whose query groups have <= 64 rows) and a short step (<= 2048 streamed tokens per SM: latency-bound running sets), the whole step is ONE
 * launch of the split kernel: every CTA appends its share of the branches first and releases a
 * per-branch flag (a range growing with branch b waits for b's flag only), and after a grid
 * barrier the CTAs merge the rows' partials themselves (the combine's arithmetic, bitwise).  Otherwise (longer steps, where the separate append overlaps
 * the split's prologue; hybrid plans; head_dim 64; the debug build) it runs the two calls.
 * own_len must stay below 2^20.
 *  q, out, lse, k_cache, v_cache, num_pages, page_table, h_plan, d_plan, workspace,
 *  workspace_bytes   as for orion_expand_attn;
 *  k_new, v_new, own_pt_off, own_cap, own_len, mode   as for orion_kv_append (own_len in/out).
 * Errors: the union of the two calls' errors.
 */
orion_status orion_expand_step(const orion_attn_shape* shape, int32_t n_branches, const void* q,
                               const void* k_new, const void* v_new, void* out, float* lse,
                               void* k_cache, void* v_cache, int32_t num_pages,
                               const int32_t* page_table, const int32_t* own_pt_off,
                               const int32_t* own_cap, int32_t* own_len, int32_t mode,
                               const void* h_plan, const void* d_plan, void* workspace,
                               size_t workspace_bytes, void* stream);

/*
 * orion_step_launches — host: the number of kernels one orion_expand_step (or, for a point-prefill
 * plan, one orion_point_prefill_attn) enqueues with this plan on a stream of the current
 * device's context: 1 when the append and the combine are fused into the split launch, else 3 (4
 * for a hybrid plan with both split kernels).
 * Errors: INVALID_ARG (null pointer, not a plan).
 */
orion_status orion_step_launches(const void* h_plan, int32_t* launches);

/*
 * orion_point_prefill_attn — the attention of the Pre stage (Alg. 1 l.12 / l.19, Eq. (2);
 * SURVEY.md §8(f) rank 1; oracle O5).  Point j's Lc content tokens P_j are the query rows; content
 * token i attends to j's bound segments except OWN, in list order, followed by P_j[0 .. i] (its own
 * run's tokens [0, i], causal):
 *   out[b,i,h] = softmax(sm_scale * q[b,i,h] . K_ctx_i(b)^T) . V_ctx_i(b),  lse likewise.
 * The K/V of P_j must already be in the cache (written by the model's QKV projection); the
 * dependency spans use the current own_len of their points, exactly as in decode.
 * Same arguments as orion_expand_attn, with a plan built with opts->prefill_rows = Lc and
 *  q, out   bf16 [n_branches][Lc][Hq][d] (device);  lse  fp32 [n_branches][Lc][Hq], nullable.
 * Runs the rows-on-lanes tcgen05 split kernel (<= 128 query rows per work item: one MMA M tile)
 * over reader-stationary items (one item streams a branch's whole list for its rows), which
 * writes out / lse itself: no combine pass.  The workspace holds only the kernel's work counter.
 * Errors: as orion_expand_attn; INVALID_ARG if the plan is not a prefill plan (and
 * orion_expand_attn rejects prefill plans).  orion_expand_split / _combine accept both kinds.
 */
orion_status orion_point_prefill_attn(const orion_attn_shape* shape, int32_t n_branches,
                                      const void* q, void* out, float* lse, const void* k_cache,
                                      const void* v_cache, int32_t num_pages,
                                      const int32_t* page_table, const int32_t* own_len,
                                      const void* h_plan, const void* d_plan, void* workspace,
                                      size_t workspace_bytes, void* stream);

/*
 * orion_expand_split / orion_expand_combine — the two kernels of orion_expand_attn as separate
 * launches (same arguments; orion_expand_attn == split then combine on one stream).  split writes
 * only the fp32 partials in `workspace`; combine reads them and writes out / lse.  Exposed so
 * callers can time or overlap the phases; the combine may also be re-run on kept partials.
 */
orion_status orion_expand_split(const orion_attn_shape* shape, int32_t n_branches, const void* q,
                                const void* k_cache, const void* v_cache, int32_t num_pages,
                                const int32_t* page_table, const int32_t* own_len,
                                const void* h_plan, const void* d_plan, void* workspace,
                                size_t workspace_bytes, void* stream);
orion_status orion_expand_combine(const orion_attn_shape* shape, int32_t n_branches, void* out,
                                  float* lse, const void* h_plan, const void* d_plan,
                                  const void* workspace, size_t workspace_bytes, void* stream);

/*
 * orion_expansion_round — one round of the expansion schedule: PAPER.md Alg. 1 l.9-22 with the
 * running set R processed as one batch per round (reading D1; Fig. 4 walkthrough
 * PAPER.md:387; oracle O6).  Host only, reentrant: the schedule state is in caller arrays.
 * Round r prefills every point not yet prefilled whose stage predecessors (Contextual k->j:
 * Pre(k); Dependent k->j: Dec(k)) completed in rounds < r, and decodes one token of
 * every point whose Pre completed in a round < r and whose Dec has not completed.  Pre completes
 * in the round it runs; Dec completes with the point's last token (with its Pre if it has none).
 *  queries[n_queries]          n_points / branch0 used (points of query i are global branches
 *                              branch0 .. branch0 + n_points - 1).
 *  edge_offsets[n_queries+1], edges[]  query i's edges are edges[edge_offsets[i] ..
 *                              edge_offsets[i+1]), query-local point ids 1..n_points.
 *  tokens[n_branches]          decode tokens each point generates (T - Lc).
 *  pre_round, dec_round [n_branches]  in/out: round in which Pre / Dec completed, -1 = not yet
 *                              (initialise to -1).
 *  left[n_branches]            in/out: decode tokens still to generate.
 *  round                       this round's index (0, 1, ... consecutively).
 *  pre_out, dec_out [n_branches], n_pre, n_dec  out: this round's prefill / decode branches,
 *                              ascending.  Both empty: every point has completed.
 * Errors: INVALID_ARG, UNKNOWN_POINT (edge outside its query), CYCLE (nothing can run but stages
 * are pending).
 */
orion_status orion_expansion_round(int32_t n_queries, const orion_query_desc* queries,
                                   const int32_t* edge_offsets, const orion_edge* edges,
                                   int32_t n_branches, const int32_t* tokens, int32_t* pre_round,
                                   int32_t* dec_round, int32_t* left, int32_t round,
                                   int32_t* pre_out, int32_t* n_pre, int32_t* dec_out,
                                   int32_t* n_dec);

/*
 * orion_select_branches — the bound segment lists of a subset of branches (the running set of a
 * round), ready for orion_expand_plan over just that subset.  Host only.  Branch sel[i]'s list
 * becomes list i; a segment growing with a selected branch (dyn = sel[k]) gets dyn = k; one
 * growing with an unselected branch (a finished ancestor) is frozen to the static extent
 * [start, start + clamp(own_len[dyn] - start, 0, len)).
 *  seg_offsets[n_branches+1], segs[]  lists of all branches (orion_bind_segments).
 *  own_len[n_branches]   current lengths.   sel[n_sel]  distinct branch ids.
 *  sel_offsets[n_sel+1], sel_segs[segs_cap]  out; segs_needed out (always written).
 * Errors: INVALID_ARG (bad / repeated ids), CAPACITY (segs_cap < *segs_needed).
 */
orion_status orion_select_branches(int32_t n_branches, const int32_t* seg_offsets,
                                   const orion_seg* segs, const int32_t* own_len, int32_t n_sel,
                                   const int32_t* sel, int32_t* sel_offsets, orion_seg* sel_segs,
                                   int32_t segs_cap, int32_t* segs_needed);

/*
 * orion_context_base — the RoPE position base of every branch's decode token (reading M2,
 * DESIGN.md §2): a token sits at its index in its branch's concatenated context, Eq. (2)'s
 * Concat(Prompt_Pre, (+)_k f(k,j), P_j) order, so branch b's token in slot s of
 * its own run is at position base[b] + s with
 *   base[b] = sum of the effective lengths of b's bound segments that precede its OWN segment
 *             (the first segment whose dyn == b; orion_bind_segments puts it last),
 * effective length = len for a static segment, clamp(own_len[dyn] - start, 0, len) for a growing
 * one (the lengths at the call, i.e. at plan time in the all-points snapshot).  Host only.
 *  seg_offsets[n_branches+1], segs[]  bound lists;  own_len[n_branches]  host int32.
 *  base[n_branches]  out.
 * Errors: INVALID_ARG (null pointers, non-monotone offsets, dyn out of range, a list without its
 * OWN segment, a base above INT32_MAX).
 */
orion_status orion_context_base(int32_t n_branches, const int32_t* seg_offsets, const orion_seg* segs,
                                const int32_t* own_len, int32_t* base);

/*
 * Decoder-layer steps around the attention (oracle O7; reading M1: bf16
 * storage, fp32 arithmetic).  Device; enqueued on `stream`.  The GEMMs between them are plain
 * library calls by the caller.
 *
 * orion_rmsnorm — per row: r = bf16(a + b) (b nullable: r = a); residual_out = r (nullable);
 *   out = bf16(r * rsqrt(mean(r^2) + eps) * weight) (nullable; needs weight).
 *   a, b, out, residual_out  bf16 [n_rows][hidden];  weight bf16 [hidden]; hidden a multiple of 8,
 *   <= 8192; all 16-byte aligned.  Errors: INVALID_ARG, UNSUPPORTED, CUDA.
 */
orion_status orion_rmsnorm(int32_t n_rows, int32_t hidden, const void* a, const void* b,
                           const void* weight, float eps, void* out, void* residual_out, void* stream);

/*
 * orion_rope_append — RoPE fused into the KV append of the decode step.  Per branch b the qkv row
 * [q (Hq*d) | k (Hkv*d) | v (Hkv*d)] (bf16, the QKV GEMM output) is split; q and k are rotated
 * at position pos = pos_base[b] + slot (rotate_half pairs (i, i + d/2), inv_freq_i =
 * rope_theta^(-2i/d); slot = own_len[b] for ADVANCE, own_len[b] - 1 for REWRITE, as in
 * orion_kv_append); q goes to q_out bf16 [n_branches][Hq][d], k and v to the slot of b's own run
 * in the paged caches (skipped when the slot is outside [0, own_cap) or its page id outside
 * [0, num_pages), as in orion_kv_append); ADVANCE then increments own_len.  pos_base[b] = the number of context tokens before b's own run (reading M2: a token's
 * position is its index in its branch's concatenated context).  shape->kv_interleaved as for the
 * attention calls.  Errors: INVALID_ARG, UNSUPPORTED, CUDA.
 */
orion_status orion_rope_append(const orion_attn_shape* shape, int32_t n_branches, const void* qkv,
                               void* q_out, void* k_cache, void* v_cache, const int32_t* own_pt_off,
                               const int32_t* own_cap, const int32_t* page_table, int32_t num_pages,
                               int32_t* own_len, const int32_t* pos_base, float rope_theta,
                               int32_t mode, void* stream);

/*
 * orion_silu_mul — out = bf16(SiLU(g) * u) per row of gate_up = [g (inter) | u (inter)] (the fused
 * gate/up GEMM output), SiLU(g) = g / (1 + e^-g).  bf16, inter a multiple of 8, 16-byte aligned.
 */
orion_status orion_silu_mul(int32_t n_rows, int32_t inter, const void* gate_up, void* out,
                            void* stream);

/* Thread-local message describing the last non-OK status returned on this thread. */
const char* orion_last_error(void);

/* Library version string (also names the compiled-in kernel variants). */
const char* orion_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ORION_H_ */
