// host.cpp — host side of the Orion expansion hot path: DAG -> stage levels -> segment lists
// (orion_dag_waves), symbolic -> physical binding (orion_bind_segments), and the sharing-aware
// work planner (orion_expand_plan).  Pure C++17, no CUDA calls: runs on the GPU-less dev box.
//
// Paper anchors: Alg. 1 l.1-8 (322-329), §3.3 edge kinds (359), Eq. (1) (362-366),
// Eq. (2)/(3) (369-384), Fig. 4 walkthrough (387).  Readings S1-S23 are listed in DESIGN.md.
#include <algorithm>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <iterator>
#include <map>
#include <string>
#include <vector>

#include "../../include/orion.h"
#include "plan_format.h"

namespace orion {

thread_local std::string g_last_error;

orion_status fail(orion_status code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
orion_status fail(orion_status code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

namespace {

constexpr int32_t kMaxPoints = 8192;  // stage-reachability bitsets are (2N)^2 bits

struct Bits {
  std::vector<uint64_t> w;
  explicit Bits(int n = 0) : w((n + 63) / 64, 0) {}
  void set(int i) { w[i >> 6] |= uint64_t(1) << (i & 63); }
  bool get(int i) const { return (w[i >> 6] >> (i & 63)) & 1; }
  void merge(const Bits& o) {
    for (size_t i = 0; i < w.size(); ++i) w[i] |= o.w[i];
  }
};

// Validated point graph: materialised edges with their kind bitmask (bit0 Ctx, bit1 Dep).
struct PointGraph {
  int n = 0;
  std::vector<std::vector<int>> succ;             // point -> successors (0-based)
  std::vector<std::vector<std::pair<int, int>>> par;  // point -> (parent, kindmask), sorted
};

orion_status build_point_graph(int32_t n, const orion_edge* edges, int32_t n_edges,
                               PointGraph& g, int32_t* err_info, int32_t err_cap) {
  if (n < 1 || n > kMaxPoints)
    return fail(ORION_ERR_INVALID_ARG, "n_points=%d outside [1, %d]", n, kMaxPoints);
  if (n_edges < 0 || (n_edges > 0 && !edges))
    return fail(ORION_ERR_INVALID_ARG, "bad edge array");
  std::map<std::pair<int, int>, int> kinds;
  for (int32_t i = 0; i < n_edges; ++i) {
    const orion_edge& e = edges[i];
    if (e.kind < ORION_EDGE_NULL || e.kind > ORION_EDGE_DEPENDENT) {
      if (err_info && err_cap > 0) err_info[0] = i;
      return fail(ORION_ERR_INVALID_ARG, "edge %d: kind %d not in {0,1,2}", i, e.kind);
    }
    if (e.from < 1 || e.from > n || e.to < 1 || e.to > n) {
      if (err_info && err_cap > 0) err_info[0] = i;
      return fail(ORION_ERR_UNKNOWN_POINT, "edge %d: (%d -> %d) names a point outside 1..%d", i,
                  e.from, e.to, n);
    }
    if (e.kind == ORION_EDGE_NULL) continue;  // Null = absence of an edge
    kinds[{e.from - 1, e.to - 1}] |= (e.kind == ORION_EDGE_CONTEXTUAL ? 1 : 2);
  }
  g.n = n;
  g.succ.assign(n, {});
  g.par.assign(n, {});
  for (auto& kv : kinds) {
    g.succ[kv.first.first].push_back(kv.first.second);
    g.par[kv.first.second].push_back({kv.first.first, kv.second});
  }
  // Kahn over the point graph; whatever remains lies on or behind a cycle.
  std::vector<int> indeg(n, 0), order;
  for (int u = 0; u < n; ++u)
    for (int v : g.succ[u]) indeg[v]++;
  for (int u = 0; u < n; ++u)
    if (!indeg[u]) order.push_back(u);
  for (size_t i = 0; i < order.size(); ++i)
    for (int v : g.succ[order[i]])
      if (--indeg[v] == 0) order.push_back(v);
  if ((int)order.size() == n) return ORION_OK;
  // Extract one cycle: walk predecessors inside the remaining set until a node repeats.
  std::vector<char> rem(n, 0);
  for (int u = 0; u < n; ++u) rem[u] = indeg[u] > 0;
  int u = 0;
  while (!rem[u]) ++u;
  std::vector<int> pos(n, -1), walk;
  while (pos[u] < 0) {
    pos[u] = (int)walk.size();
    walk.push_back(u);
    int nxt = -1;
    for (auto& pk : g.par[u])
      if (rem[pk.first]) { nxt = pk.first; break; }
    u = nxt;  // every remaining node has a remaining predecessor
  }
  std::vector<int> cyc(walk.begin() + pos[u], walk.end());
  std::reverse(cyc.begin(), cyc.end());  // predecessor walk -> forward edge order
  if (err_info)
    for (int i = 0; i < (int)cyc.size() && i < err_cap; ++i) err_info[i] = cyc[i] + 1;
  return fail(ORION_ERR_CYCLE, "point DAG has a cycle of length %zu through point %d", cyc.size(),
              cyc[0] + 1);
}

}  // namespace
}  // namespace orion

using namespace orion;

extern "C" const char* orion_last_error(void) { return g_last_error.c_str(); }

extern "C" orion_status orion_dag_waves(int32_t n, const orion_edge* edges, int32_t n_edges,
                                        int32_t policy, int32_t* pre_level, int32_t* dec_level,
                                        int32_t* n_levels, int32_t* wave_offsets,
                                        int32_t* wave_stages, int32_t* seg_offsets,
                                        orion_segref* segs, int32_t segs_cap,
                                        int32_t* segs_needed, int32_t* err_info,
                                        int32_t err_cap) {
  if (!pre_level || !dec_level || !n_levels || !seg_offsets || !segs_needed)
    return fail(ORION_ERR_INVALID_ARG, "null output pointer");
  if (policy != ORION_POLICY_ANCESTORS && policy != ORION_POLICY_PARENTS_EQ3)
    return fail(ORION_ERR_INVALID_ARG, "unknown policy %d", policy);
  PointGraph g;
  orion_status st = build_point_graph(n, edges, n_edges, g, err_info, err_cap);
  if (st != ORION_OK) return st;

  // Stage graph (Alg. 1 l.8): stage s = 2*i + phase.
  //   Pre(i) -> Dec(i);  Ctx k->j: Pre(k) -> Pre(j);  Dep k->j: Dec(k) -> Pre(j).
  const int S = 2 * n;
  std::vector<std::vector<int>> ssucc(S);
  std::vector<int> sindeg(S, 0);
  auto add = [&](int a, int b) { ssucc[a].push_back(b); sindeg[b]++; };
  for (int i = 0; i < n; ++i) add(2 * i, 2 * i + 1);
  for (int j = 0; j < n; ++j)
    for (auto& pk : g.par[j]) {
      if (pk.second & 1) add(2 * pk.first, 2 * j);
      if (pk.second & 2) add(2 * pk.first + 1, 2 * j);
    }
  // Kahn order with longest-path levels (Eq. (1) generalised; reading S10).
  std::vector<int> level(S, 0), order;
  order.reserve(S);
  for (int s = 0; s < S; ++s)
    if (!sindeg[s]) order.push_back(s);
  for (size_t i = 0; i < order.size(); ++i) {
    int s = order[i];
    for (int t : ssucc[s]) {
      level[t] = std::max(level[t], level[s] + 1);
      if (--sindeg[t] == 0) order.push_back(t);
    }
  }
  int nl = 0;
  for (int s = 0; s < S; ++s) nl = std::max(nl, level[s] + 1);
  for (int i = 0; i < n; ++i) {
    pre_level[i] = level[2 * i];
    dec_level[i] = level[2 * i + 1];
  }
  *n_levels = nl;
  if (wave_offsets || wave_stages) {
    std::vector<int> cnt(nl + 1, 0);
    for (int s = 0; s < S; ++s) cnt[level[s] + 1]++;
    for (int w = 0; w < nl; ++w) cnt[w + 1] += cnt[w];
    if (wave_offsets)
      for (int w = 0; w <= nl; ++w) wave_offsets[w] = cnt[w];
    if (wave_stages) {
      std::vector<int> fill(cnt.begin(), cnt.end() - 1);
      for (int s = 0; s < S; ++s)  // ascending s == ascending (point, Pre<Dec)
        wave_stages[fill[level[s]]++] = (s / 2 + 1) * 2 + (s & 1);
    }
  }

  // Segment lists: [PREFIX] + deps ascending by point id + [OWN(j)].
  std::vector<std::vector<orion_segref>> lists(n);
  if (policy == ORION_POLICY_ANCESTORS) {
    // anc[s] = stages with a path to s, propagated in topological order.
    std::vector<Bits> anc(S, Bits(S));
    for (int s : order)
      for (int t : ssucc[s]) {
        anc[t].set(s);
        anc[t].merge(anc[s]);
      }
    for (int j = 0; j < n; ++j) {
      const Bits& a = anc[2 * j];
      for (int k = 0; k < n; ++k) {
        if (k == j || !a.get(2 * k)) continue;  // point ancestor <=> Pre(k) ~> Pre(j)
        lists[j].push_back({a.get(2 * k + 1) ? ORION_SEG_FULL : ORION_SEG_CONTENT, k + 1});
      }
    }
  } else {
    for (int j = 0; j < n; ++j)
      for (auto& pk : g.par[j])
        lists[j].push_back({(pk.second & 2) ? ORION_SEG_OUTPUT : ORION_SEG_CONTENT, pk.first + 1});
  }
  int32_t total = 0;
  for (int j = 0; j < n; ++j) total += 2 + (int32_t)lists[j].size();
  *segs_needed = total;
  if (segs_cap < total || !segs)
    return fail(ORION_ERR_CAPACITY, "segs_cap=%d < needed %d", segs_cap, total);
  int32_t o = 0;
  for (int j = 0; j < n; ++j) {
    seg_offsets[j] = o;
    segs[o++] = {ORION_SEG_PREFIX, 0};
    for (auto& r : lists[j]) segs[o++] = r;
    segs[o++] = {ORION_SEG_OWN, j + 1};
  }
  seg_offsets[n] = o;
  return ORION_OK;
}

extern "C" orion_status orion_bind_segments(int32_t n_queries, const orion_query_desc* queries,
                                            int32_t n_branches, const orion_point_desc* points,
                                            const int32_t* seg_offsets, const orion_segref* refs,
                                            orion_seg* out) {
  if (n_queries < 0 || n_branches < 0 || (n_queries && !queries) || (n_branches && !points) ||
      !seg_offsets || (n_branches && (!refs || !out)))
    return fail(ORION_ERR_INVALID_ARG, "null or negative argument");
  std::vector<int32_t> qof(n_branches, -1);
  for (int32_t q = 0; q < n_queries; ++q) {
    const orion_query_desc& Q = queries[q];
    if (Q.n_points < 1 || Q.branch0 < 0 || Q.branch0 + Q.n_points > n_branches ||
        Q.prefix_len < 0 || Q.prefix_pt_off < 0)
      return fail(ORION_ERR_INVALID_ARG, "query %d: bad descriptor", q);
    for (int32_t b = Q.branch0; b < Q.branch0 + Q.n_points; ++b) {
      if (qof[b] >= 0) return fail(ORION_ERR_INVALID_ARG, "branch %d in two queries", b);
      qof[b] = q;
    }
  }
  for (int32_t b = 0; b < n_branches; ++b) {
    const orion_point_desc& p = points[b];
    if (p.pt_off < 0 || p.content_len < 0 || p.capacity < p.content_len)
      return fail(ORION_ERR_INVALID_ARG, "branch %d: bad point descriptor", b);
    if (qof[b] < 0) return fail(ORION_ERR_INVALID_ARG, "branch %d belongs to no query", b);
    if (seg_offsets[b] > seg_offsets[b + 1] || seg_offsets[b] < 0)
      return fail(ORION_ERR_INVALID_ARG, "seg_offsets not monotone at %d", b);
  }
  for (int32_t b = 0; b < n_branches; ++b) {
    const orion_query_desc& Q = queries[qof[b]];
    for (int32_t i = seg_offsets[b]; i < seg_offsets[b + 1]; ++i) {
      const orion_segref r = refs[i];
      if (r.kind == ORION_SEG_PREFIX) {
        out[i] = {Q.prefix_pt_off, 0, Q.prefix_len, -1};
        continue;
      }
      if (r.point < 1 || r.point > Q.n_points)
        return fail(ORION_ERR_INVALID_ARG, "branch %d entry %d: point %d outside its query", b,
                    i - seg_offsets[b], r.point);
      const int32_t kb = Q.branch0 + r.point - 1;
      const orion_point_desc& P = points[kb];
      switch (r.kind) {
        case ORION_SEG_CONTENT: out[i] = {P.pt_off, 0, P.content_len, -1}; break;
        case ORION_SEG_FULL: out[i] = {P.pt_off, 0, P.capacity, kb}; break;
        case ORION_SEG_OUTPUT: out[i] = {P.pt_off, P.content_len, P.capacity - P.content_len, kb}; break;
        case ORION_SEG_OWN: out[i] = {P.pt_off, 0, P.capacity, kb}; break;
        default: return fail(ORION_ERR_INVALID_ARG, "branch %d: segment kind %d", b, r.kind);
      }
    }
  }
  return ORION_OK;
}

namespace {

struct Interval {
  int32_t start, end, dyn, branch;
};

struct Piece {
  int32_t pt_off, t0, t1, dyn;
  std::vector<int32_t> readers;  // ascending branch ids
};

orion_status check_shape(const orion_attn_shape* s) {
  if (!s) return fail(ORION_ERR_INVALID_ARG, "null shape");
  if (s->num_q_heads < 1 || s->num_kv_heads < 1 || s->num_q_heads % s->num_kv_heads)
    return fail(ORION_ERR_INVALID_ARG, "heads %d/%d", s->num_q_heads, s->num_kv_heads);
  if (s->head_dim != 64 && s->head_dim != 128)
    return fail(ORION_ERR_UNSUPPORTED, "head_dim %d not in {64,128}", s->head_dim);
  if (s->page_size < 16 || s->page_size > 256 || (s->page_size & (s->page_size - 1)))
    return fail(ORION_ERR_UNSUPPORTED, "page_size %d not a power of two in [16,256]", s->page_size);
  if (s->kv_interleaved != 0 && s->kv_interleaved != 1)
    return fail(ORION_ERR_INVALID_ARG, "kv_interleaved must be 0 or 1");
  return ORION_OK;
}

inline int64_t align16(int64_t x) { return (x + 15) & ~int64_t(15); }

}  // namespace

namespace orion {
orion_status check_shape_public(const orion_attn_shape* s) { return check_shape(s); }
}  // namespace orion

extern "C" orion_status orion_expand_plan(const orion_attn_shape* shape, int32_t n_branches,
                                          const int32_t* h_seg_offsets, const orion_seg* h_segs,
                                          const int32_t* h_own_len, const orion_plan_opts* opts,
                                          void* plan_buf, size_t plan_cap, size_t* plan_needed,
                                          size_t* workspace_needed) {
  orion_status st = check_shape(shape);
  if (st != ORION_OK) return st;
  if (n_branches < 1 || !h_seg_offsets || !h_segs || !plan_needed || !workspace_needed)
    return fail(ORION_ERR_INVALID_ARG, "bad plan arguments");
  const int32_t Hq = shape->num_q_heads, Hkv = shape->num_kv_heads, G = Hq / Hkv;
  int32_t chunk = (opts && opts->chunk_tokens > 0) ? opts->chunk_tokens : 512;
  const int32_t flags = opts ? opts->flags : 0;
  const int32_t Lc = (opts && opts->prefill_rows > 0) ? opts->prefill_rows : 0;   // prefill plan
  if (Lc > 0 && (flags & ORION_PLAN_MMA_SYNC))
    return fail(ORION_ERR_UNSUPPORTED, "point-prefill plans run on the tcgen05 rows-on-lanes kernel");
  // Point prefill has Lc*G query rows per branch and kv head: the rows-on-lanes kernel (M = 128).
  const int32_t variant = (flags & ORION_PLAN_MMA_SYNC) ? kVariantMmaSync
                          : (Lc > 0 || (flags & ORION_PLAN_ROWS_ON_LANES) || shape->head_dim != 128) ? kVariantTC
                                                                                                    : kVariantTCT;
  const int32_t R = (Lc > 0 ? Lc : 1) * G;          // query rows per reader branch and kv head
  const int32_t rows_per_item = variant == kVariantTC    ? kRowsPerItemTC
                                : variant == kVariantTCT ? kRowsPerItemTCT
                                                         : kRowsPerItemMMA;
  chunk = std::max(kTileTokens, (chunk + kTileTokens - 1) / kTileTokens * kTileTokens);

  // 1. Group bound segments by page run.  A prefill plan instead keeps every branch's list as a
  //    range list (reader-stationary: one work item streams the whole context of one branch's
  //    Lc*G rows, so Q is loaded once and each row gets one partial); its OWN segment (the one
  //    growing with the branch itself) becomes the last range, read causally over [start, +Lc).
  std::map<int32_t, std::vector<Interval>> groups;
  std::vector<orion_seg> own_causal(Lc > 0 ? n_branches : 0, orion_seg{-1, 0, 0, -1});
  std::vector<std::vector<Range>> branch_ranges(Lc > 0 ? n_branches : 0);
  std::vector<int64_t> logical(n_branches, 0);
  int64_t logical_total = 0;
  for (int32_t b = 0; b < n_branches; ++b) {
    if (h_seg_offsets[b] > h_seg_offsets[b + 1] || h_seg_offsets[b] < 0)
      return fail(ORION_ERR_INVALID_ARG, "seg_offsets not monotone at %d", b);
    for (int32_t i = h_seg_offsets[b]; i < h_seg_offsets[b + 1]; ++i) {
      const orion_seg& s = h_segs[i];
      if (s.pt_off < 0 || s.start < 0 || s.len < 0 || s.dyn < -1 || s.dyn >= n_branches)
        return fail(ORION_ERR_INVALID_ARG, "branch %d segment %d: bad fields", b, i);
      if (Lc > 0 && s.dyn == b) {
        if (own_causal[b].pt_off >= 0)
          return fail(ORION_ERR_INVALID_ARG, "branch %d has two OWN segments", b);
        if (s.len < Lc)
          return fail(ORION_ERR_INVALID_ARG, "branch %d: OWN capacity %d < prefill rows %d", b, s.len, Lc);
        own_causal[b] = s;
        logical[b] += Lc;
        continue;
      }
      if (s.len == 0) continue;  // zero-length segments are skipped (reading S22)
      if (Lc > 0) branch_ranges[b].push_back(Range{s.pt_off, s.start, s.start + s.len, s.dyn, 0, {0, 0, 0}});
      else groups[s.pt_off].push_back({s.start, s.start + s.len, s.dyn, b});
      logical[b] += s.len;
    }
    if (Lc > 0 && own_causal[b].pt_off < 0)
      return fail(ORION_ERR_INVALID_ARG, "branch %d: a prefill plan needs its OWN segment", b);
    if (logical[b] == 0) return fail(ORION_ERR_INVALID_ARG, "branch %d has an empty context", b);
    logical_total += logical[b];
  }

  // 2. Cut each run at every boundary; attach reader sets; merge equal neighbours.
  std::vector<Piece> pieces;
  for (auto& gkv : groups) {
    std::vector<Interval>& iv = gkv.second;
    int32_t dyn = -1;
    for (auto& x : iv)
      if (x.dyn >= 0) {
        if (dyn >= 0 && dyn != x.dyn)
          return fail(ORION_ERR_UNSUPPORTED,
                      "page run %d grows with two branches (%d, %d)", gkv.first, dyn, x.dyn);
        dyn = x.dyn;
      }
    std::vector<int32_t> cuts;
    for (auto& x : iv) { cuts.push_back(x.start); cuts.push_back(x.end); }
    std::sort(cuts.begin(), cuts.end());
    cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
    for (size_t c = 0; c + 1 < cuts.size(); ++c) {
      const int32_t a = cuts[c], z = cuts[c + 1];
      Piece p{gkv.first, a, z, -1, {}};
      bool any_static = false;
      int32_t static_end = 0;
      for (auto& x : iv)
        if (x.start <= a && x.end >= z) {
          p.readers.push_back(x.branch);
          if (x.dyn >= 0) p.dyn = x.dyn;
          else { any_static = true; static_end = std::max(static_end, x.end); }
        }
      if (p.readers.empty()) continue;
      std::sort(p.readers.begin(), p.readers.end());
      for (size_t r = 1; r < p.readers.size(); ++r)
        if (p.readers[r] == p.readers[r - 1])
          return fail(ORION_ERR_INVALID_ARG,
                      "branch %d covers tokens [%d,%d) of run %d twice", p.readers[r], a, z,
                      gkv.first);
      if (p.dyn >= 0 && any_static && h_own_len && static_end > h_own_len[p.dyn])
        return fail(ORION_ERR_INVALID_ARG,
                    "static segment of run %d ends at %d past own_len[%d]=%d", gkv.first,
                    static_end, p.dyn, h_own_len[p.dyn]);
      if (!pieces.empty()) {
        Piece& q = pieces.back();
        if (q.pt_off == p.pt_off && q.t1 == p.t0 && q.dyn == p.dyn && q.readers == p.readers) {
          q.t1 = p.t1;
          continue;
        }
      }
      pieces.push_back(std::move(p));
    }
  }

  // 3. Work items: piece x kv head x chunk x 64-row block.  Chunk length grows with the row
  //    count so the fp32 partial traffic stays a small fraction of the KV bytes.
  std::vector<WorkItem> items;
  std::vector<int32_t> readers;
  std::vector<int64_t> cost;
  int64_t unique_tokens = 0;
  int32_t n_slots = 0;
  const int32_t Lrows = Lc > 0 ? Lc : 1;
  std::vector<std::vector<int32_t>> row_slots((size_t)n_branches * Lrows * Hq);
  auto add_items = [&](int32_t pt_off, int32_t t0, int32_t t1, int32_t dyn, int32_t iflags,
                       const std::vector<int32_t>& rd, int32_t piece_id) {
    const int32_t roff = (int32_t)readers.size();
    readers.insert(readers.end(), rd.begin(), rd.end());
    const int32_t rows = (int32_t)rd.size() * R;
    const int32_t rows_blk = std::min(rows, rows_per_item);
    int32_t ch = std::max(chunk, 32 * rows_blk);
    ch = (ch + kTileTokens - 1) / kTileTokens * kTileTokens;
    for (int32_t g = 0; g < Hkv; ++g)
      for (int32_t t = t0; t < t1; t += ch)
        for (int32_t r0 = 0; r0 < rows; r0 += rows_per_item) {
          WorkItem w{};
          w.pt_off = pt_off; w.t0 = t; w.t1 = std::min(t1, t + ch); w.dyn = dyn;
          w.kv_head = g; w.readers_off = roff; w.row_begin = r0;
          w.n_rows = std::min(rows_per_item, rows - r0); w.slot0 = n_slots; w.piece = piece_id;
          w.flags = iflags;
          for (int32_t r = r0; r < r0 + w.n_rows; ++r) {
            const int32_t b = rd[r / R], i = (r % R) / G, h = g * G + r % G;
            row_slots[((size_t)b * Lrows + i) * Hq + h].push_back(n_slots + (r - r0));
          }
          n_slots += w.n_rows;
          items.push_back(w);
          // ~ cycles: stream the tokens, plus the row tiles' MMA work, plus a fixed start-up.
          cost.push_back((int64_t)(w.t1 - w.t0) * (2 + (w.n_rows + 15) / 16) + 256);
        }
  };
  std::vector<Range> ranges;                         // multi-range items' ranges (plan Range[])
  // Decode plans on the tcgen05 kernels: rows are grouped into fixed reader blocks (R readers =
  // one <= rows_per_item row block; a block never straddles queries, whose branches are
  // consecutive), and every chunk a block's rows read in full with the same reader subset joins
  // one multi-range item.  A Dependent chain's shared history then streams once per block as one
  // accumulation (one partial per row) instead of one short item and one partial per ancestor.
  const bool merge = Lc == 0 && variant != kVariantMmaSync && !(flags & ORION_PLAN_NO_MERGE);
  // Hybrid (swap-AB decode plans): reader blocks of up to 128 rows; a block's items with more than
  // 64 rows run on the rows-on-lanes kernel (MMA M = 128), the others on the swap-AB kernel.
  const bool hybrid = merge && variant == kVariantTCT && !(flags & ORION_PLAN_NO_HYBRID);
  std::vector<char> is_big;
  if (!merge) {
    for (size_t pi = 0; pi < pieces.size(); ++pi) {
      const Piece& p = pieces[pi];
      unique_tokens += p.t1 - p.t0;
      add_items(p.pt_off, p.t0, p.t1, p.dyn, 0, p.readers, (int32_t)pi);
    }
  } else {
    const int32_t RB = std::max(1, (hybrid ? kRowsPerItemBig : rows_per_item) / G);
    // Blocks are counted from each query's first branch, so a query's plan does not depend on
    // what else is in the batch (a strong-scaling shard reproduces the single-GPU plan and its
    // results bitwise).  The planner has no query ids: every list starts with its query's PREFIX
    // segment, whose page run identifies the query; a query is a contiguous run of branches with
    // the same PREFIX run (two queries sharing a prefix page run are told apart unless adjacent).
    std::vector<int32_t> qkey(n_branches), qstart(n_branches);
    for (int32_t b = 0; b < n_branches; ++b) {
      qkey[b] = h_seg_offsets[b] < h_seg_offsets[b + 1] ? h_segs[h_seg_offsets[b]].pt_off : -1 - b;
      qstart[b] = (b > 0 && qkey[b] == qkey[b - 1]) ? qstart[b - 1] : b;
    }
    auto block_of = [&](int32_t b) { return (int64_t)qstart[b] * 1000003 + (b - qstart[b]) / RB; };
    std::map<std::pair<int32_t, std::vector<int32_t>>, int32_t> key_index;
    std::vector<std::pair<int32_t, std::vector<int32_t>>> gkeys;
    std::vector<std::vector<Range>> gchunks;
    std::vector<int32_t> gpiece;
    // Hybrid plans with reader blocks of <= 32 readers: every range a block reads with more than
    // rows_per_item rows joins ONE masked item per (block, kv head) -- its readers the union of
    // the ranges' reader subsets, each range carrying the bitmask of the readers that read it --
    // instead of one item per distinct subset (a Dependent chain's block would otherwise get one
    // short item per ancestor inside the block, each paying an item's start-up and epilogue).
    const bool masked_blocks = hybrid && RB <= 32;
    std::map<std::pair<int32_t, int64_t>, int32_t> bkey_index;
    std::vector<std::pair<int32_t, int64_t>> bkeys;
    std::vector<std::vector<std::pair<Range, std::vector<int32_t>>>> bchunks;
    std::vector<std::vector<int32_t>> bunion;
    std::vector<int32_t> bpiece;
    int64_t big_tokens = 0;                        // tokens of the masked ranges, summed over kv heads
    const int64_t sms = (opts && opts->num_sms > 0) ? opts->num_sms : 148;
    // Small steps (a latency-bound running set: c2's 1-8 branches) would get fewer items than
    // SMs from the chunk and merge lengths tuned for partial traffic; there the chunk and merge
    // caps shrink so the step still spreads over about 2 items per SM (tile granularity), when
    // that needs items shorter than kSmallStepTokens (c4's 8-query share, 2.6K tokens per item at
    // 2 per SM, measured slower with the cap: its partials outweigh the spread).  This
    // makes a small batch's chunking depend on the batch's total work; with an explicit
    // chunk_tokens the planner keeps the fixed chunking (a query's items then never depend on
    // the rest of the batch).
    int64_t work = 0;                              // streamed tokens x reader blocks x kv heads
    for (const Piece& p : pieces) {
      int64_t nblk = 0, last = -1;
      for (int32_t b : p.readers)
        if (block_of(b) != last) last = block_of(b), ++nblk;
      work += (int64_t)(p.t1 - p.t0) * nblk * Hkv;
    }
    const int64_t fill = (work + 2 * sms - 1) / (2 * sms);
    const bool adapt = !(opts && opts->chunk_tokens > 0);   // an explicit chunk length is kept
    const int32_t small_cap = adapt && fill < kSmallStepTokens ? (int32_t)std::max<int64_t>(kTileTokens, (fill + kTileTokens - 1) / kTileTokens * kTileTokens)
                                                  : INT32_MAX;
    const int64_t merge_cap = std::min<int64_t>(kMergeTokens, small_cap);
    static_assert(kSmallStepTokens <= kMergeTokens, "the small-step cap only ever shortens items");
    for (size_t pi = 0; pi < pieces.size(); ++pi) {
      const Piece& p = pieces[pi];
      unique_tokens += p.t1 - p.t0;
      for (size_t i = 0; i < p.readers.size();) {
        const int64_t blk = block_of(p.readers[i]);
        std::vector<int32_t> S;
        while (i < p.readers.size() && block_of(p.readers[i]) == blk) S.push_back(p.readers[i++]);
        const int32_t rows = (int32_t)S.size() * G;
        int32_t ch = std::max(chunk, 32 * std::min(rows, kRowsPerItemBig));
        ch = std::min((ch + kTileTokens - 1) / kTileTokens * kTileTokens, small_cap);
        if (masked_blocks && rows > rows_per_item) {
          for (int32_t g = 0; g < Hkv; ++g) {
            auto key = std::make_pair(g, blk);
            auto f = bkey_index.find(key);
            int32_t idx;
            if (f == bkey_index.end()) {
              idx = (int32_t)bkeys.size();
              bkey_index.emplace(key, idx);
              bkeys.push_back(key);
              bchunks.emplace_back();
              bunion.emplace_back();
              bpiece.push_back((int32_t)pi);
            } else {
              idx = f->second;
            }
            // 1024-token ranges: the granularity at which the block's ranges are grouped into items
            for (int32_t t = p.t0; t < p.t1; t += 1024)
              bchunks[idx].push_back({Range{p.pt_off, t, std::min(p.t1, t + 1024), p.dyn, 0, {0, 0, 0}}, S});
            big_tokens += p.t1 - p.t0;
            std::vector<int32_t> u;
            std::set_union(bunion[idx].begin(), bunion[idx].end(), S.begin(), S.end(), std::back_inserter(u));
            bunion[idx].swap(u);
          }
          continue;
        }
        for (int32_t g = 0; g < Hkv; ++g) {
          auto key = std::make_pair(g, S);
          auto f = key_index.find(key);
          int32_t idx;
          if (f == key_index.end()) {
            idx = (int32_t)gkeys.size();
            key_index.emplace(key, idx);
            gkeys.push_back(key);
            gchunks.emplace_back();
            gpiece.push_back((int32_t)pi);
          } else {
            idx = f->second;
          }
          for (int32_t t = p.t0; t < p.t1; t += ch)
            gchunks[idx].push_back(Range{p.pt_off, t, std::min(p.t1, t + ch), p.dyn, 0, {0, 0, 0}});
        }
      }
    }
    // Masked items are long (whole reader blocks).  When the swap-AB part of the step is small
    // (c5 chain-64: 0.25 of the big part's tokens), cap them to ~4 per SM (4K-8K tokens): 2-3
    // 8K-token items per SM had left the busiest SM 1.4x above the mean.  When it is large (c5
    // wide-64: the points' own runs, as many tokens as the prefix), keep them long: fewer items
    // than SMs leave SMs on which the swap-AB kernel starts at once, beside the first kernel.
    int64_t small_tokens = 0;
    for (const auto& cs : gchunks)
      for (const Range& R : cs) small_tokens += R.t1 - R.t0;
    const int64_t big_cap = 2 * small_tokens >= big_tokens
                                ? kMergeTokens
                                : std::max<int64_t>(4096, std::min<int64_t>(kMergeTokens, big_tokens / (4 * sms)));
    for (size_t bi = 0; bi < bkeys.size(); ++bi) {
      const int32_t g = bkeys[bi].first;
      const std::vector<int32_t>& U = bunion[bi];
      const int32_t rows = (int32_t)U.size() * G;
      if (U.size() > 32 || rows > kRowsPerItemBig)
        return fail(ORION_ERR_INVALID_ARG, "internal: masked block of %zu readers", U.size());
      const int32_t roff = (int32_t)readers.size();
      readers.insert(readers.end(), U.begin(), U.end());
      const auto& cs = bchunks[bi];
      for (size_t c0 = 0; c0 < cs.size();) {
        size_t c1 = c0;
        int64_t tok = 0;
        while (c1 < cs.size() && (c1 == c0 || tok + (cs[c1].first.t1 - cs[c1].first.t0) <= big_cap))
          tok += cs[c1].first.t1 - cs[c1].first.t0, ++c1;
        WorkItem w{};
        w.pt_off = (int32_t)ranges.size(); w.dyn = -1;
        w.flags = kItemRanges; w.n_ranges = (int32_t)(c1 - c0);
        for (size_t c = c0; c < c1; ++c) {
          Range R = cs[c].first;
          if (cs[c].second.size() != U.size()) {
            uint32_t mask = 0;
            for (int32_t b : cs[c].second)
              mask |= 1u << (std::lower_bound(U.begin(), U.end(), b) - U.begin());
            R.flags |= kRangeMasked;
            R.pad_[0] = (int32_t)mask;
          }
          ranges.push_back(R);
        }
        w.kv_head = g; w.readers_off = roff; w.piece = bpiece[bi];
        w.row_begin = 0; w.n_rows = rows; w.slot0 = n_slots;
        for (int32_t r = 0; r < rows; ++r)
          row_slots[(size_t)U[r / G] * Hq + g * G + r % G].push_back(n_slots + r);
        n_slots += rows;
        items.push_back(w);
        is_big.push_back(1);
        cost.push_back(tok * (2 + (rows + 15) / 16) + 256 * (int64_t)(c1 - c0));
        c0 = c1;
      }
    }
    for (size_t gi = 0; gi < gkeys.size(); ++gi) {
      const int32_t g = gkeys[gi].first;
      const std::vector<int32_t>& S = gkeys[gi].second;
      const int32_t rows = (int32_t)S.size() * G;
      // one big item (65..128 rows, hybrid), or row blocks of <= rows_per_item rows (a block of
      // G > rows_per_item rows -- one reader -- is split, never handed to a kernel whole)
      const bool big = hybrid && rows > rows_per_item && rows <= kRowsPerItemBig;
      const int32_t rblk = big ? rows : rows_per_item;
      const int32_t roff = (int32_t)readers.size();
      readers.insert(readers.end(), S.begin(), S.end());
      const std::vector<Range>& cs = gchunks[gi];
      for (size_t c0 = 0; c0 < cs.size();) {
        size_t c1 = c0;
        int64_t tok = 0;
        while (c1 < cs.size() && (c1 == c0 || tok + (cs[c1].t1 - cs[c1].t0) <= merge_cap))
          tok += cs[c1].t1 - cs[c1].t0, ++c1;
        WorkItem w{};
        if (c1 - c0 == 1) {
          w.pt_off = cs[c0].pt_off; w.t0 = cs[c0].t0; w.t1 = cs[c0].t1; w.dyn = cs[c0].dyn;
        } else {
          w.pt_off = (int32_t)ranges.size(); w.dyn = -1;
          w.flags = kItemRanges; w.n_ranges = (int32_t)(c1 - c0);
          ranges.insert(ranges.end(), cs.begin() + c0, cs.begin() + c1);
        }
        w.kv_head = g; w.readers_off = roff; w.piece = gpiece[gi];
        for (int32_t r0 = 0; r0 < rows; r0 += rblk) {
          w.row_begin = r0; w.n_rows = std::min(rblk, rows - r0); w.slot0 = n_slots;
          for (int32_t r = r0; r < r0 + w.n_rows; ++r)
            row_slots[(size_t)S[r / G] * Hq + g * G + r % G].push_back(n_slots + (r - r0));
          n_slots += w.n_rows;
          items.push_back(w);
          is_big.push_back(big ? 1 : 0);
          cost.push_back(tok * (2 + (w.n_rows + 15) / 16) + 256 * (int64_t)(c1 - c0));
        }
        c0 = c1;
      }
    }
  }
  // Prefill: per kv head and branch, one multi-range item per row block: the branch's ranges in
  // list order, then its own content tokens (causal).  Items are then ordered longest context
  // first (stable: equal-length items of a query and kv head stay adjacent) for the kernels' atomic
  // item hand-out; a paired plan keeps generation order (pairs are adjacent items).
  if (Lc > 0) {
    std::vector<int32_t> range_off(n_branches);
    for (int32_t b = 0; b < n_branches; ++b) {
      const orion_seg& s = own_causal[b];
      branch_ranges[b].push_back(Range{s.pt_off, s.start, s.start + Lc, -1, kItemCausal, {0, 0, 0}});
      range_off[b] = (int32_t)ranges.size();
      ranges.insert(ranges.end(), branch_ranges[b].begin(), branch_ranges[b].end());
      unique_tokens += logical[b];
    }
    // Paired plans: a query's branches (same leading range: its prefix) ordered by context length,
    // so the two items of a pair have similar unique tails (a warpgroup whose item ended idles
    // while its partner finishes alone).
    std::vector<int32_t> border(n_branches);
    for (int32_t b = 0; b < n_branches; ++b) border[b] = b;
    if (flags & ORION_PLAN_PAIR)
      std::stable_sort(border.begin(), border.end(), [&](int32_t x, int32_t y) {
        const Range& rx = branch_ranges[x][0];
        const Range& ry = branch_ranges[y][0];
        if (rx.pt_off != ry.pt_off) return rx.pt_off < ry.pt_off;
        if (rx.t0 != ry.t0) return rx.t0 < ry.t0;
        return logical[x] < logical[y];
      });
    for (int32_t g = 0; g < Hkv; ++g)
      for (int32_t bi = 0; bi < n_branches; ++bi) {
        const int32_t b = border[bi];
        const int32_t roff = (int32_t)readers.size();
        readers.push_back(b);
        for (int32_t r0 = 0; r0 < R; r0 += rows_per_item) {
          WorkItem w{};
          w.pt_off = range_off[b]; w.t0 = 0; w.t1 = 0; w.dyn = -1;
          w.kv_head = g; w.readers_off = roff; w.row_begin = r0;
          w.n_rows = std::min(rows_per_item, R - r0); w.slot0 = n_slots; w.piece = -1;
          w.flags = kItemRanges; w.n_ranges = (int32_t)branch_ranges[b].size();
          for (int32_t r = r0; r < r0 + w.n_rows; ++r) {
            const int32_t i = r / G, h = g * G + r % G;
            row_slots[((size_t)b * Lrows + i) * Hq + h].push_back(n_slots + (r - r0));
          }
          n_slots += w.n_rows;
          items.push_back(w);
          cost.push_back(logical[b]);                // context tokens: longest first
        }
      }
  }
  // Prefill pairs: items 2u and 2u+1 (adjacent readers of one kv head, or two row blocks of one
  // reader) run on one CTA; the leading ranges their lists share -- the query's prefix, common
  // dependencies, or everything for two row blocks of a branch -- stream one K/V tile for both.
  const bool paired = Lc > 0 && (flags & ORION_PLAN_PAIR);
  if (paired)
    for (size_t u = 0; u + 1 < items.size(); u += 2) {
      WorkItem& A = items[u];
      const WorkItem& B = items[u + 1];
      int32_t n_sh = 0;
      if (A.kv_head == B.kv_head)
        while (n_sh < A.n_ranges && n_sh < B.n_ranges) {
          const Range& x = ranges[A.pt_off + n_sh];
          const Range& y = ranges[B.pt_off + n_sh];
          if (x.pt_off != y.pt_off || x.t0 != y.t0 || x.t1 != y.t1 || x.dyn != y.dyn || x.flags != y.flags) break;
          ++n_sh;
        }
      A.t1 = n_sh;
    }
  int64_t streamed = 0;
  for (size_t i = 0; i < items.size(); ++i) {
    const WorkItem& w = items[i];
    if (w.flags & kItemRanges) {
      for (int32_t r = 0; r < w.n_ranges; ++r) {
        const Range& x = ranges[w.pt_off + r];
        if (!(paired && (i & 1) && r < items[i - 1].t1)) streamed += x.t1 - x.t0;   // pair: once
      }
    } else {
      streamed += w.t1 - w.t0;
    }
  }
  for (size_t r = 0; r < row_slots.size(); ++r)
    if (row_slots[r].empty())
      return fail(ORION_ERR_INVALID_ARG, "row %zu (branch %zu) has no context", r, r / ((size_t)Lrows * Hq));

  // Longest first; row blocks of one chunk stay adjacent (same cost, stable sort) so they run
  // together and share the chunk through L2.  A hybrid plan lists its big items first.
  is_big.resize(items.size(), 0);
  std::vector<int32_t> perm(items.size());
  for (size_t i = 0; i < perm.size(); ++i) perm[i] = (int32_t)i;
  if (Lc == 0)
    std::stable_sort(perm.begin(), perm.end(), [&](int32_t a, int32_t b) {
      if (is_big[a] != is_big[b]) return is_big[a] > is_big[b];
      return cost[a] > cost[b];
    });
  else if (!paired) {
    // Prefill: the items of one prefix group (kv head x the query's leading range) run together,
    // so the group's prefix streams from DRAM about once and the rest of its readers hit L2;
    // groups in generation order (kv head major), longest first inside a group.
    std::vector<int64_t> gkey(items.size());
    for (size_t i = 0; i < items.size(); ++i) {
      const Range& r0 = ranges[items[i].pt_off];
      gkey[i] = ((int64_t)items[i].kv_head << 40) | ((int64_t)(uint32_t)r0.pt_off << 8);
    }
    std::map<int64_t, int32_t> gorder;
    for (size_t i = 0; i < items.size(); ++i) gorder.emplace(gkey[i], (int32_t)gorder.size());
    std::stable_sort(perm.begin(), perm.end(), [&](int32_t a, int32_t b) {
      const int32_t ga = gorder[gkey[a]], gb = gorder[gkey[b]];
      if (ga != gb) return ga < gb;
      return cost[a] > cost[b];
    });
  }
  int32_t n_big = 0;
  for (size_t i = 0; i < items.size(); ++i) n_big += is_big[i];
  for (size_t i = 0; i < items.size(); ++i)
    if (items[i].n_rows > (is_big[i] ? kRowsPerItemBig : rows_per_item))
      return fail(ORION_ERR_INVALID_ARG, "internal: item %zu has %d rows", i, items[i].n_rows);

  // 4. Serialise.
  const int64_t n_rows = (int64_t)n_branches * Lrows * Hq;
  PlanHeader h{};
  h.magic = kPlanMagic; h.version = kPlanVersion;
  h.n_branches = n_branches; h.num_q_heads = Hq; h.num_kv_heads = Hkv;
  h.head_dim = shape->head_dim; h.page_size = shape->page_size; h.group = G;
  h.n_items = (int32_t)items.size(); h.n_partials = n_slots; h.n_rows = (int32_t)n_rows;
  h.n_reader_entries = (int32_t)readers.size();
  h.items_off = align16(sizeof(PlanHeader));
  h.readers_off = align16(h.items_off + (int64_t)items.size() * sizeof(WorkItem));
  h.comb_off_off = align16(h.readers_off + (int64_t)readers.size() * 4);
  h.comb_slot_off = align16(h.comb_off_off + (n_rows + 1) * 4);
  h.ranges_off = align16(h.comb_slot_off + (int64_t)n_slots * 4);
  h.n_ranges = (int32_t)ranges.size();
  h.plan_bytes = align16(h.ranges_off + (int64_t)ranges.size() * sizeof(Range));
  if (partials_fp16(variant)) {
    h.acc_bytes = align16((int64_t)n_slots * shape->head_dim * 2);
    h.workspace_bytes = h.acc_bytes + align16((int64_t)n_slots * 4);
  } else {
    h.acc_bytes = align16((int64_t)n_slots * shape->head_dim * 4);
    h.workspace_bytes = h.acc_bytes + align16((int64_t)n_slots * 8);
  }
  if (variant != kVariantMmaSync) {   // the tcgen05 kernels' work counters (kept zero between launches)
    h.counter_off = h.workspace_bytes;
    // work counters, the fused append's epoch and one append flag per branch (orion_expand_step)
    h.workspace_bytes += kCounterBytes + align16((int64_t)n_branches * 4);
  }
  h.n_big = n_big;
  h.n_pieces = (int64_t)pieces.size();
  h.unique_tokens = unique_tokens;
  h.logical_tokens = logical_total;
  h.variant = variant;
  h.max_ctas = (opts && opts->num_sms > 0) ? opts->num_sms : 0;
  h.prefill_rows = Lc;
  h.paired = paired ? 1 : 0;
  h.streamed_tokens = streamed;
  h.sm_scale = shape->sm_scale > 0.f ? shape->sm_scale : 1.0f / std::sqrt((float)shape->head_dim);
  *plan_needed = (size_t)h.plan_bytes;
  *workspace_needed = (size_t)h.workspace_bytes;
  if (!plan_buf || plan_cap < (size_t)h.plan_bytes)
    return fail(ORION_ERR_CAPACITY, "plan_cap=%zu < needed %lld", plan_cap, (long long)h.plan_bytes);
  if (reinterpret_cast<uintptr_t>(plan_buf) & 15)
    return fail(ORION_ERR_INVALID_ARG, "plan_buf must be 16-byte aligned");
  char* base = static_cast<char*>(plan_buf);
  std::memset(base, 0, (size_t)h.plan_bytes);
  std::memcpy(base, &h, sizeof h);
  WorkItem* wi = reinterpret_cast<WorkItem*>(base + h.items_off);
  for (size_t i = 0; i < perm.size(); ++i) wi[i] = items[perm[i]];
  std::memcpy(base + h.readers_off, readers.data(), readers.size() * 4);
  int32_t* coff = reinterpret_cast<int32_t*>(base + h.comb_off_off);
  int32_t* cslot = reinterpret_cast<int32_t*>(base + h.comb_slot_off);
  int32_t o = 0;
  for (int64_t r = 0; r < n_rows; ++r) {
    coff[r] = o;
    for (int32_t s : row_slots[r]) cslot[o++] = s;
  }
  coff[n_rows] = o;
  if (!ranges.empty()) std::memcpy(base + h.ranges_off, ranges.data(), ranges.size() * sizeof(Range));
  // plan id: FNV-1a over the body, so a stale or mismatched device copy can be detected
  uint64_t id = 1469598103934665603ull;
  for (int64_t i = h.items_off; i < h.plan_bytes; ++i) id = (id ^ (uint8_t)base[i]) * 1099511628211ull;
  id ^= (uint64_t)h.n_items << 32 ^ (uint64_t)(uint32_t)h.n_partials;
  reinterpret_cast<PlanHeader*>(base)->plan_id = id;
  return ORION_OK;
}

extern "C" orion_status orion_plan_get_stats(const void* h_plan, orion_plan_stats* out) {
  if (!h_plan || !out) return fail(ORION_ERR_INVALID_ARG, "null argument");
  const PlanHeader* h = static_cast<const PlanHeader*>(h_plan);
  if (h->magic != kPlanMagic || h->version != kPlanVersion)
    return fail(ORION_ERR_INVALID_ARG, "not an orion plan");
  out->n_items = h->n_items;
  out->n_pieces = h->n_pieces;
  out->n_partials = h->n_partials;
  out->n_rows = h->n_rows;
  out->unique_tokens = h->unique_tokens;
  out->logical_tokens = h->logical_tokens;
  out->plan_bytes = h->plan_bytes;
  out->workspace_bytes = h->workspace_bytes;
  out->streamed_tokens = h->streamed_tokens;
  out->paired = h->paired;
  out->n_big = h->n_big;
  return ORION_OK;
}

// ------------------------------------------------------------------------------ expansion driver
extern "C" orion_status orion_expansion_round(int32_t n_queries, const orion_query_desc* queries,
                                              const int32_t* edge_offsets, const orion_edge* edges,
                                              int32_t n_branches, const int32_t* tokens,
                                              int32_t* pre_round, int32_t* dec_round, int32_t* left,
                                              int32_t round, int32_t* pre_out, int32_t* n_pre,
                                              int32_t* dec_out, int32_t* n_dec) {
  if (n_queries < 0 || n_branches < 0 || round < 0 || (n_queries > 0 && (!queries || !edge_offsets)) ||
      !tokens || !pre_round || !dec_round || !left || !pre_out || !n_pre || !dec_out || !n_dec)
    return fail(ORION_ERR_INVALID_ARG, "bad expansion_round arguments");
  std::vector<uint8_t> is_pre(n_branches, 0), is_dec(n_branches, 0);
  int32_t pending = 0;
  for (int32_t qi = 0; qi < n_queries; ++qi) {
    const orion_query_desc& q = queries[qi];
    if (q.n_points < 1 || q.branch0 < 0 || q.branch0 + q.n_points > n_branches)
      return fail(ORION_ERR_INVALID_ARG, "query %d: bad point range", qi);
    // stage predecessors of Pre(j): Contextual k->j needs Pre(k), Dependent needs Dec(k)
    std::vector<std::vector<int32_t>> need_pre(q.n_points + 1), need_dec(q.n_points + 1);
    for (int32_t e = edge_offsets[qi]; e < edge_offsets[qi + 1]; ++e) {
      const orion_edge& x = edges[e];
      if (x.kind < ORION_EDGE_NULL || x.kind > ORION_EDGE_DEPENDENT)
        return fail(ORION_ERR_INVALID_ARG, "query %d edge %d: bad kind %d", qi, e, x.kind);
      if (x.from < 1 || x.from > q.n_points || x.to < 1 || x.to > q.n_points)
        return fail(ORION_ERR_UNKNOWN_POINT, "query %d edge %d: point out of range", qi, e);
      if (x.kind == ORION_EDGE_CONTEXTUAL) need_pre[x.to].push_back(x.from);
      if (x.kind == ORION_EDGE_DEPENDENT) need_dec[x.to].push_back(x.from);
    }
    for (int32_t j = 1; j <= q.n_points; ++j) {
      const int32_t b = q.branch0 + j - 1;
      if (dec_round[b] >= 0) continue;
      ++pending;
      if (pre_round[b] >= 0) {
        if (pre_round[b] < round) is_dec[b] = 1;
        continue;
      }
      bool ready = true;
      for (int32_t k : need_pre[j]) {
        const int32_t kb = q.branch0 + k - 1;
        ready = ready && pre_round[kb] >= 0 && pre_round[kb] < round;
      }
      for (int32_t k : need_dec[j]) {
        const int32_t kb = q.branch0 + k - 1;
        ready = ready && dec_round[kb] >= 0 && dec_round[kb] < round;
      }
      if (ready) is_pre[b] = 1;
    }
  }
  int32_t np = 0, nd = 0;
  for (int32_t b = 0; b < n_branches; ++b) {
    if (is_pre[b]) {
      pre_out[np++] = b;
      pre_round[b] = round;
      left[b] = std::max(0, tokens[b]);
      if (left[b] == 0) dec_round[b] = round;
    } else if (is_dec[b]) {
      dec_out[nd++] = b;
      if (--left[b] <= 0) dec_round[b] = round;
    }
  }
  *n_pre = np;
  *n_dec = nd;
  if (pending > 0 && np == 0 && nd == 0)
    return fail(ORION_ERR_CYCLE, "expansion stalled with %d stages pending (cyclic DAG?)", pending);
  return ORION_OK;
}

extern "C" orion_status orion_context_base(int32_t n_branches, const int32_t* seg_offsets,
                                           const orion_seg* segs, const int32_t* own_len,
                                           int32_t* base) {
  if (n_branches < 0 || !seg_offsets || (n_branches > 0 && (!segs || !own_len || !base)))
    return fail(ORION_ERR_INVALID_ARG, "bad context_base arguments");
  for (int32_t b = 0; b < n_branches; ++b) {
    if (seg_offsets[b] < 0 || seg_offsets[b] > seg_offsets[b + 1])
      return fail(ORION_ERR_INVALID_ARG, "seg_offsets not monotone at %d", b);
    int64_t sum = 0;
    bool own = false;
    for (int32_t i = seg_offsets[b]; i < seg_offsets[b + 1] && !own; ++i) {
      const orion_seg& s = segs[i];
      if (s.dyn < -1 || s.dyn >= n_branches || s.len < 0 || s.start < 0)
        return fail(ORION_ERR_INVALID_ARG, "branch %d segment %d: bad fields (dyn %d)", b, i, s.dyn);
      if (s.dyn == b) { own = true; break; }
      sum += s.dyn >= 0 ? std::min(s.len, std::max(0, own_len[s.dyn] - s.start)) : s.len;
    }
    if (!own) return fail(ORION_ERR_INVALID_ARG, "branch %d: list has no OWN segment (dyn == %d)", b, b);
    if (sum > INT32_MAX) return fail(ORION_ERR_INVALID_ARG, "branch %d: position base overflows", b);
    base[b] = (int32_t)sum;
  }
  return ORION_OK;
}

extern "C" orion_status orion_select_branches(int32_t n_branches, const int32_t* seg_offsets,
                                              const orion_seg* segs, const int32_t* own_len,
                                              int32_t n_sel, const int32_t* sel,
                                              int32_t* sel_offsets, orion_seg* sel_segs,
                                              int32_t segs_cap, int32_t* segs_needed) {
  if (n_branches < 0 || n_sel < 0 || !seg_offsets || !segs || !own_len || (n_sel > 0 && !sel) ||
      !sel_offsets || !segs_needed)
    return fail(ORION_ERR_INVALID_ARG, "bad select_branches arguments");
  std::vector<int32_t> pos(n_branches, -1);
  for (int32_t i = 0; i < n_sel; ++i) {
    if (sel[i] < 0 || sel[i] >= n_branches || pos[sel[i]] >= 0)
      return fail(ORION_ERR_INVALID_ARG, "sel[%d] = %d out of range or repeated", i, sel[i]);
    pos[sel[i]] = i;
  }
  int32_t need = 0;
  sel_offsets[0] = 0;
  for (int32_t i = 0; i < n_sel; ++i) {
    need += seg_offsets[sel[i] + 1] - seg_offsets[sel[i]];
    sel_offsets[i + 1] = need;
  }
  *segs_needed = need;
  if (!sel_segs || segs_cap < need)
    return fail(ORION_ERR_CAPACITY, "segs_cap=%d < needed %d", segs_cap, need);
  int32_t o = 0;
  for (int32_t i = 0; i < n_sel; ++i)
    for (int32_t s = seg_offsets[sel[i]]; s < seg_offsets[sel[i] + 1]; ++s) {
      orion_seg x = segs[s];
      if (x.dyn >= n_branches) return fail(ORION_ERR_INVALID_ARG, "segment %d: dyn out of range", s);
      if (x.dyn >= 0) {
        if (pos[x.dyn] >= 0) {
          x.dyn = pos[x.dyn];                        // still growing inside the selection
        } else {                                     // finished (or paused): freeze at own_len
          x.len = std::min(x.len, std::max(0, own_len[x.dyn] - x.start));
          x.dyn = -1;
        }
      }
      sel_segs[o++] = x;
    }
  return ORION_OK;
}
