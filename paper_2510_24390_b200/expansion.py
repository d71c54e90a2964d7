"""Expansion driver: PAPER.md Alg. 1 l.9-22 on one GPU with continuous batching (SURVEY.md §8(f)
rank 2; reading D1 in DESIGN.md; oracle O6).

Every round, `orion_expansion_round` (C, host) returns the points to prefill and the running set
to decode.  The round then
  * prefills its new points -- `orion_point_prefill_attn` over the selection (per layer), their
    own_len set to Lc;
  * decodes one token of the running set -- per layer `orion_kv_append` (layer 0 ADVANCE, the
    other layers REWRITE the same slot) and `orion_expand_attn`.
Plans are built by the native planner over `orion_select_branches`' segment lists, and only when
the running set changes (points join after their Pre, leave after their last token); between
changes the decode state (own_len) lives on the device and is advanced by the append kernel.
With `graph=True` a decode round (every layer's append + split + combine launches, PDL edges
included) is captured once per running set into a CUDA graph and replayed each round: the host
then does one graph launch per round instead of 3-4 launches per layer, so a latency-bound
expansion (few branches, short contexts) is no longer bound by host launch rate.  The release
library's launch path is capture-safe (no synchronising call; the ORION_CHECK build's read-backs
are not, so the debug library must run eagerly).
This module is orchestration only: no arithmetic on the data happens here.
"""
import numpy as np

from . import (APPEND_ADVANCE, APPEND_REWRITE, POLICY_ANCESTORS, ExpansionBatch, bind_segments,
               dag_waves, expansion_round, select_branches)


class Expansion:
    """queries: [{n_points, edges, prefix_pt_off, prefix_len}] (points of query i are the global
    branches branch0_i ..); points: [(pt_off, content_len, capacity)] per branch; every point has
    content length lc and generates tokens[b] decode tokens (T_b - lc)."""

    def __init__(self, hq, hkv, d, page, queries, points, page_table, lc, tokens,
                 policy=POLICY_ANCESTORS, device="cuda", chunk_tokens=0, kv_interleaved=False):
        import torch
        self.hq, self.hkv, self.d, self.page, self.lc = hq, hkv, d, page, lc
        self.device = torch.device(device)
        self.chunk_tokens = chunk_tokens
        self.kv_interleaved = kv_interleaved
        qdesc, offs, refs, eoffs, edges, b0 = [], [0], [], [0], [], 0
        for q in queries:
            w = dag_waves(q["n_points"], q["edges"], policy)
            so = w["seg_offsets"]
            for j in range(q["n_points"]):
                refs.append(w["segs"][so[j]:so[j + 1]])
                offs.append(offs[-1] + int(so[j + 1] - so[j]))
            qdesc.append((q["n_points"], b0, q["prefix_pt_off"], q["prefix_len"]))
            edges += [tuple(e) for e in q["edges"]]
            eoffs.append(len(edges))
            b0 += q["n_points"]
        self.n_branches = b0
        self.qdesc = qdesc
        self.edge_offsets = np.array(eoffs, np.int32)
        self.edges = np.array(edges, np.int32).reshape(-1, 3)
        self.points = np.array(points, np.int32).reshape(-1, 3)
        self.seg_offsets = np.array(offs, np.int32)
        self.segs = bind_segments(qdesc, self.points, self.seg_offsets, np.concatenate(refs))
        self.page_table = torch.from_numpy(np.ascontiguousarray(page_table, np.int32)).to(self.device)
        self.tokens = np.ascontiguousarray(tokens, np.int32)
        self.pre_round = np.full(b0, -1, np.int32)
        self.dec_round = np.full(b0, -1, np.int32)
        self.left = self.tokens.copy()
        self.own_len = np.full(b0, lc, np.int32)     # host mirror of every point's length
        self.rnd = 0
        self.dec_set = None
        self.dec_batch = None
        self.rebuilds = 0
        self.graph = None               # (key, torch.cuda.CUDAGraph) of the current running set
        self.captures = 0

    # -- schedule ------------------------------------------------------------------------------
    def next_round(self):
        """(prefill branches, decode branches) of the next round; both empty when done."""
        pre, dec = expansion_round(self.qdesc, self.edge_offsets, self.edges, self.tokens,
                                   self.pre_round, self.dec_round, self.left, self.rnd)
        self.rnd += 1
        return pre, dec

    def _batch(self, sel, prefill_rows=0):
        so, sg = select_branches(self.seg_offsets, self.segs, self.own_len, sel)
        pts = self.points[sel]
        return ExpansionBatch.from_segments(self.hq, self.hkv, self.d, self.page, so, sg, pts[:, 0],
                                            pts[:, 2], self.page_table, self.own_len[sel],
                                            device=self.device, chunk_tokens=self.chunk_tokens,
                                            prefill_rows=prefill_rows, kv_interleaved=self.kv_interleaved)

    # -- the two kinds of work of a round ------------------------------------------------------
    def prefill(self, pre, q_pre, k_caches, v_caches, out, stream=None):
        """Pre stage of the points `pre`: q_pre / out [layers][len(pre), lc, Hq, d] (rows in the
        order of `pre`), one orion_point_prefill_attn per layer.  Returns the batch used."""
        self.own_len[pre] = self.lc
        batch = self._batch(pre, prefill_rows=self.lc)
        for l in range(len(k_caches)):
            batch.attend(q_pre[l], out[l], k_caches[l], v_caches[l], stream=stream)
        return batch

    def decode(self, dec, q, k_new, v_new, k_caches, v_caches, out, lse=None, stream=None, graph=False):
        """One decode token of the running set `dec` through all layers: q/k_new/v_new/out
        [layers][len(dec), ...] in the order of `dec`.  Rebuilds the plan if the set changed.
        graph=True: replay the round's CUDA graph, captured when the set or a tensor changes."""
        if self.dec_set is None or len(self.dec_set) != len(dec) or not np.array_equal(self.dec_set, dec):
            self.dec_batch = self._batch(dec)
            self.dec_set = np.array(dec, np.int32)
            self.rebuilds += 1
            self.graph = None

        def launches(s):
            for l in range(len(k_caches)):
                mode = APPEND_ADVANCE if l == 0 else APPEND_REWRITE
                self.dec_batch.step(q[l], k_new[l], v_new[l], k_caches[l], v_caches[l], out[l],
                                    None if lse is None else lse[l], mode=mode, stream=s)

        if graph:
            import torch
            ts = [t for ls in (q, k_new, v_new, k_caches, v_caches, out, lse or []) for t in ls]
            key = (self.rebuilds, tuple(t.data_ptr() for t in ts))
            if self.graph is None or self.graph[0] != key:
                # capture_begin/end directly: the torch.cuda.graph context also synchronises,
                # runs the garbage collector and empties the allocator cache (~0.1 s a capture);
                # the launches allocate nothing
                g = torch.cuda.CUDAGraph()
                cs = torch.cuda.Stream(device=self.device)
                cs.wait_stream(torch.cuda.current_stream(self.device) if stream is None else stream)
                with torch.cuda.stream(cs):
                    g.capture_begin(capture_error_mode="thread_local")
                    try:
                        launches(cs)
                    finally:
                        g.capture_end()
                self.graph = (key, g)
                self.captures += 1
            if stream is None:
                self.graph[1].replay()
            else:
                with torch.cuda.stream(stream):
                    self.graph[1].replay()
        else:
            launches(stream)
        self.own_len[dec] += 1
        return self.dec_batch
