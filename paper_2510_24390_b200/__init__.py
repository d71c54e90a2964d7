"""paper_2510_24390_b200 — B200-native hot path of Orion's content parallel expansion.

Python surface of the C ABI in include/orion.h (same names, argument marshalling only):

    dag_waves(n_points, edges, policy)           -> levels, waves, segment lists     (host)
    bind_segments(queries, points, offs, refs)   -> bound segments                   (host)
    expand_plan(shape, offs, segs, own_len)      -> device work plan                 (host)
    kv_append(...)                               -> K1 on the current CUDA stream    (device)
    expand_step(...)                             -> K1 + K2 + K3 (K1 fused into K2 where possible)
    expand_attn(...)                             -> K2 + K3 on the current stream    (device)

`ExpansionBatch` strings them together for a set of in-flight queries: it builds the plan once
per in-flight-set change (Alg. 1 readiness loop) and then runs decode steps
(Alg. 1 l.16) with no host work and no host<->device traffic.
"""
import ctypes

import numpy as np

from . import _lib
from ._lib import (OrionError, POLICY_ANCESTORS, POLICY_PARENTS_EQ3, APPEND_ADVANCE,
                   APPEND_REWRITE, SEG_PREFIX, SEG_CONTENT, SEG_FULL, SEG_OUTPUT, SEG_OWN,
                   EDGE_NULL, EDGE_CONTEXTUAL, EDGE_DEPENDENT, SEG_DTYPE, SEGREF_DTYPE, lib)

__all__ = ["dag_waves", "bind_segments", "expand_plan", "context_base", "plan_stats", "kv_append", "expand_attn", "expand_step",
           "expand_split", "expand_combine",
           "ExpansionBatch", "OrionError", "version", "POLICY_ANCESTORS", "POLICY_PARENTS_EQ3",
           "APPEND_ADVANCE", "APPEND_REWRITE"]


def version():
    return lib().orion_version().decode()


def _shape(hq, hkv, d, page, sm_scale=0.0, kv_interleaved=False):
    return _lib.AttnShape(hq, hkv, d, page, float(sm_scale), int(bool(kv_interleaved)))


def dag_waves(n_points, edges, policy=POLICY_ANCESTORS):
    """orion_dag_waves.  edges: iterable of (from, to, kind).  Returns a dict with
    pre_level, dec_level (np.int32 [n]), n_levels, waves (list of lists of (point, phase)),
    seg_offsets (np.int32 [n+1]) and segs (structured np array of (kind, point))."""
    e = np.array(list(edges), dtype=np.int32).reshape(-1, 3)
    e = np.ascontiguousarray(e)
    n = int(n_points)
    nn = max(n, 1)
    pre = np.zeros(nn, np.int32)
    dec = np.zeros(nn, np.int32)
    nl = np.zeros(1, np.int32)
    woff = np.zeros(2 * nn + 1, np.int32)
    wst = np.zeros(2 * nn, np.int32)
    soff = np.zeros(nn + 1, np.int32)
    need = np.zeros(1, np.int32)
    err = np.full(max(nn, 1), -1, np.int32)
    cap = 4 * nn + 4
    for _ in range(2):
        segs = np.zeros(cap, SEGREF_DTYPE)
        code = lib().orion_dag_waves(n, _lib.ptr(e) if len(e) else None, len(e), int(policy),
                                     _lib.ptr(pre), _lib.ptr(dec), _lib.ptr(nl), _lib.ptr(woff),
                                     _lib.ptr(wst), _lib.ptr(soff), _lib.ptr(segs), cap,
                                     _lib.ptr(need), _lib.ptr(err), len(err))
        if code == _lib.ERR_CAPACITY:
            cap = int(need[0])
            continue
        if code != _lib.OK:
            info = [int(x) for x in err if x >= 0]
            _lib.check(code, info)
        break
    L = int(nl[0])
    waves = [[(int(s) // 2, int(s) % 2) for s in wst[woff[w]:woff[w + 1]]] for w in range(L)]
    return {"pre_level": pre[:n], "dec_level": dec[:n], "n_levels": L, "waves": waves,
            "seg_offsets": soff[:n + 1], "segs": segs[:int(need[0])]}


def bind_segments(queries, points, seg_offsets, refs):
    """orion_bind_segments.  queries: [(n_points, branch0, prefix_pt_off, prefix_len)],
    points: [(pt_off, content_len, capacity)] per global branch; seg_offsets/refs: global CSR."""
    qd = np.ascontiguousarray(np.array(queries, dtype=np.int32).reshape(-1, 4))
    pd = np.ascontiguousarray(np.array(points, dtype=np.int32).reshape(-1, 3))
    so = np.ascontiguousarray(seg_offsets, dtype=np.int32)
    rf = np.ascontiguousarray(refs).astype(SEGREF_DTYPE)
    out = np.zeros(int(so[-1]), SEG_DTYPE)
    _lib.check(lib().orion_bind_segments(len(qd), _lib.ptr(qd), len(pd), _lib.ptr(pd),
                                         _lib.ptr(so), _lib.ptr(rf), _lib.ptr(out)))
    return out


def expansion_round(queries, edge_offsets, edges, tokens, pre_round, dec_round, left, rnd):
    """orion_expansion_round.  queries: [(n_points, branch0, prefix_pt_off, prefix_len)];
    edge_offsets [Q+1] / edges [E, 3] int32; tokens, pre_round, dec_round, left: np.int32 [B],
    the last three updated in place.  Returns (prefill branches, decode branches) of round rnd."""
    qd = np.ascontiguousarray(np.array(queries, dtype=np.int32).reshape(-1, 4))
    eo = np.ascontiguousarray(edge_offsets, dtype=np.int32)
    ed = np.ascontiguousarray(np.array(edges, dtype=np.int32).reshape(-1, 3))
    tk = np.ascontiguousarray(tokens, dtype=np.int32)
    for a in (pre_round, dec_round, left):
        if a.dtype != np.int32 or not a.flags.c_contiguous:
            raise OrionError(_lib.ERR_INVALID_ARG, "state arrays must be contiguous np.int32")
    nb = len(tk)
    po = np.zeros(max(nb, 1), np.int32)
    do = np.zeros(max(nb, 1), np.int32)
    npre = np.zeros(1, np.int32)
    ndec = np.zeros(1, np.int32)
    _lib.check(lib().orion_expansion_round(len(qd), _lib.ptr(qd), _lib.ptr(eo),
                                           _lib.ptr(ed) if len(ed) else None, nb, _lib.ptr(tk),
                                           _lib.ptr(pre_round), _lib.ptr(dec_round), _lib.ptr(left),
                                           int(rnd), _lib.ptr(po), _lib.ptr(npre), _lib.ptr(do),
                                           _lib.ptr(ndec)))
    return po[:int(npre[0])].copy(), do[:int(ndec[0])].copy()


def select_branches(seg_offsets, segs, own_len, sel):
    """orion_select_branches -> (seg_offsets [n_sel+1], segs) of the branches `sel`."""
    so = np.ascontiguousarray(seg_offsets, dtype=np.int32)
    sg = np.ascontiguousarray(segs).astype(SEG_DTYPE)
    ol = np.ascontiguousarray(own_len, dtype=np.int32)
    sl = np.ascontiguousarray(sel, dtype=np.int32)
    off = np.zeros(len(sl) + 1, np.int32)
    need = np.zeros(1, np.int32)
    code = lib().orion_select_branches(len(so) - 1, _lib.ptr(so), _lib.ptr(sg), _lib.ptr(ol), len(sl),
                                       _lib.ptr(sl) if len(sl) else None, _lib.ptr(off), None, 0,
                                       _lib.ptr(need))
    if code != _lib.ERR_CAPACITY and code != _lib.OK:
        _lib.check(code)
    out = np.zeros(max(int(need[0]), 1), SEG_DTYPE)
    _lib.check(lib().orion_select_branches(len(so) - 1, _lib.ptr(so), _lib.ptr(sg), _lib.ptr(ol), len(sl),
                                           _lib.ptr(sl) if len(sl) else None, _lib.ptr(off),
                                           _lib.ptr(out), len(out), _lib.ptr(need)))
    return off, out[:int(need[0])]


def context_base(seg_offsets, segs, own_len):
    """orion_context_base -> np.int32 [n_branches]: per branch, the context tokens before its OWN
    segment at the lengths own_len (reading M2: its token in own slot s sits at base + s)."""
    so = np.ascontiguousarray(seg_offsets, dtype=np.int32)
    sg = np.ascontiguousarray(segs).astype(SEG_DTYPE)
    ol = np.ascontiguousarray(own_len, dtype=np.int32)
    out = np.zeros(max(len(so) - 1, 1), np.int32)
    _lib.check(lib().orion_context_base(len(so) - 1, _lib.ptr(so), _lib.ptr(sg), _lib.ptr(ol), _lib.ptr(out)))
    return out[:len(so) - 1]


PLAN_MMA_SYNC = 1        # ORION_PLAN_MMA_SYNC: legacy mma.sync split kernel
PLAN_ROWS_ON_LANES = 2   # ORION_PLAN_ROWS_ON_LANES: rows-on-lanes tcgen05 split kernel
PLAN_NO_MERGE = 4        # ORION_PLAN_NO_MERGE: one item per piece chunk (no multi-range merging)
PLAN_PAIR = 8            # ORION_PLAN_PAIR: point-prefill items run in pairs sharing K/V tiles (opt-in)
PLAN_NO_HYBRID = 16      # ORION_PLAN_NO_HYBRID: every decode item on the swap-AB kernel (<= 64 rows)


def expand_plan(hq, hkv, d, page, seg_offsets, segs, own_len=None, chunk_tokens=0, num_sms=0,
                sm_scale=0.0, flags=0, prefill_rows=0):
    """orion_expand_plan -> (plan: np.uint8 16-byte aligned host buffer, workspace_bytes).
    prefill_rows = Lc > 0 builds a point-prefill plan (orion_point_prefill_attn)."""
    shape = _shape(hq, hkv, d, page, sm_scale)
    so = np.ascontiguousarray(seg_offsets, dtype=np.int32)
    sg = np.ascontiguousarray(segs).astype(SEG_DTYPE)
    ol = None if own_len is None else np.ascontiguousarray(own_len, dtype=np.int32)
    opts = _lib.PlanOpts(int(num_sms), int(chunk_tokens), int(flags), int(prefill_rows))
    need = ctypes.c_size_t(0)
    ws = ctypes.c_size_t(0)
    nb = len(so) - 1
    code = lib().orion_expand_plan(ctypes.byref(shape), nb, _lib.ptr(so), _lib.ptr(sg), _lib.ptr(ol),
                                   ctypes.byref(opts), None, 0, ctypes.byref(need), ctypes.byref(ws))
    if code != _lib.ERR_CAPACITY:
        _lib.check(code)
    plan = _lib.aligned_empty(need.value)
    _lib.check(lib().orion_expand_plan(ctypes.byref(shape), nb, _lib.ptr(so), _lib.ptr(sg),
                                       _lib.ptr(ol), ctypes.byref(opts), _lib.ptr(plan), need.value,
                                       ctypes.byref(need), ctypes.byref(ws)))
    return plan, int(ws.value)


def plan_stats(plan):
    st = _lib.PlanStats()
    _lib.check(lib().orion_plan_get_stats(_lib.ptr(plan), ctypes.byref(st)))
    return {n: int(getattr(st, n)) for n, _ in _lib.PlanStats._fields_}


def _stream_ptr(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise OrionError(_lib.ERR_INVALID_ARG, "device argument is not a CUDA tensor")


def kv_append(hq, hkv, d, page, k_new, v_new, k_cache, v_cache, own_pt_off, own_cap, page_table,
              own_len, mode=APPEND_ADVANCE, stream=None, kv_interleaved=False):
    """orion_kv_append on `stream` (default: torch's current stream).  All tensors on the GPU."""
    _require_cuda(k_new, v_new, k_cache, v_cache, own_pt_off, own_cap, page_table, own_len)
    shape = _shape(hq, hkv, d, page, 0.0, kv_interleaved)
    _lib.check(lib().orion_kv_append(ctypes.byref(shape), int(own_len.shape[0]), k_new.data_ptr(),
                                     v_new.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(),
                                     own_pt_off.data_ptr(), own_cap.data_ptr(),
                                     page_table.data_ptr(), int(k_cache.shape[0]), own_len.data_ptr(),
                                     int(mode), _stream_ptr(stream)))


def expand_attn(hq, hkv, d, page, q, out, lse, k_cache, v_cache, page_table, own_len, h_plan,
                d_plan, workspace, stream=None, sm_scale=0.0, kv_interleaved=False):
    """orion_expand_attn on `stream` (default: torch's current stream)."""
    _require_cuda(q, out, lse, k_cache, v_cache, page_table, own_len, d_plan, workspace)
    shape = _shape(hq, hkv, d, page, sm_scale, kv_interleaved)
    _lib.check(lib().orion_expand_attn(
        ctypes.byref(shape), int(q.shape[0]), q.data_ptr(), out.data_ptr(),
        None if lse is None else lse.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(),
        int(k_cache.shape[0]), page_table.data_ptr(), own_len.data_ptr(), _lib.ptr(h_plan),
        d_plan.data_ptr(), workspace.data_ptr(), workspace.numel() * workspace.element_size(),
        _stream_ptr(stream)))


def expand_step(hq, hkv, d, page, q, k_new, v_new, out, lse, k_cache, v_cache, page_table, own_pt_off,
                own_cap, own_len, h_plan, d_plan, workspace, mode=APPEND_ADVANCE, stream=None, sm_scale=0.0,
                kv_interleaved=False):
    """orion_expand_step (append + attention of one layer; the append fused into the split launch
    where the plan allows) on `stream` (default: torch's current stream)."""
    _require_cuda(q, k_new, v_new, out, lse, k_cache, v_cache, page_table, own_pt_off, own_cap, own_len,
                  d_plan, workspace)
    shape = _shape(hq, hkv, d, page, sm_scale, kv_interleaved)
    _lib.check(lib().orion_expand_step(
        ctypes.byref(shape), int(q.shape[0]), q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(), out.data_ptr(),
        None if lse is None else lse.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(), int(k_cache.shape[0]),
        page_table.data_ptr(), own_pt_off.data_ptr(), own_cap.data_ptr(), own_len.data_ptr(), int(mode),
        _lib.ptr(h_plan), d_plan.data_ptr(), workspace.data_ptr(), workspace.numel() * workspace.element_size(),
        _stream_ptr(stream)))


def point_prefill_attn(hq, hkv, d, page, q, out, lse, k_cache, v_cache, page_table, own_len, h_plan,
                       d_plan, workspace, stream=None, sm_scale=0.0, kv_interleaved=False):
    """orion_point_prefill_attn: q/out bf16 [B, Lc, Hq, d], lse fp32 [B, Lc, Hq] (nullable)."""
    _require_cuda(q, out, lse, k_cache, v_cache, page_table, own_len, d_plan, workspace)
    shape = _shape(hq, hkv, d, page, sm_scale, kv_interleaved)
    _lib.check(lib().orion_point_prefill_attn(
        ctypes.byref(shape), int(q.shape[0]), q.data_ptr(), out.data_ptr(),
        None if lse is None else lse.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(),
        int(k_cache.shape[0]), page_table.data_ptr(), own_len.data_ptr(), _lib.ptr(h_plan),
        d_plan.data_ptr(), workspace.data_ptr(), workspace.numel() * workspace.element_size(),
        _stream_ptr(stream)))


def expand_split(hq, hkv, d, page, q, k_cache, v_cache, page_table, own_len, h_plan, d_plan,
                 workspace, stream=None, sm_scale=0.0, kv_interleaved=False):
    """orion_expand_split: K2 only (partials into `workspace`)."""
    _require_cuda(q, k_cache, v_cache, page_table, own_len, d_plan, workspace)
    shape = _shape(hq, hkv, d, page, sm_scale, kv_interleaved)
    _lib.check(lib().orion_expand_split(
        ctypes.byref(shape), int(q.shape[0]), q.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(),
        int(k_cache.shape[0]), page_table.data_ptr(), own_len.data_ptr(), _lib.ptr(h_plan),
        d_plan.data_ptr(), workspace.data_ptr(), workspace.numel() * workspace.element_size(),
        _stream_ptr(stream)))


def expand_combine(hq, hkv, d, page, n_branches, out, lse, h_plan, d_plan, workspace, stream=None,
                   sm_scale=0.0, kv_interleaved=False):
    """orion_expand_combine: K3 only (partials in `workspace` -> out / lse)."""
    _require_cuda(out, lse, d_plan, workspace)
    shape = _shape(hq, hkv, d, page, sm_scale, kv_interleaved)
    _lib.check(lib().orion_expand_combine(
        ctypes.byref(shape), int(n_branches), out.data_ptr(), None if lse is None else lse.data_ptr(),
        _lib.ptr(h_plan), d_plan.data_ptr(), workspace.data_ptr(),
        workspace.numel() * workspace.element_size(), _stream_ptr(stream)))


def rmsnorm(a, weight, out=None, b=None, residual_out=None, eps=1e-5, stream=None):
    """orion_rmsnorm: r = a (+ b), residual_out = r, out = r * rsqrt(mean(r^2) + eps) * weight."""
    _require_cuda(a, b, weight, out, residual_out)
    p = lambda t: None if t is None else t.data_ptr()
    _lib.check(lib().orion_rmsnorm(int(a.shape[0]), int(a.shape[-1]), a.data_ptr(), p(b), p(weight),
                                   float(eps), p(out), p(residual_out), _stream_ptr(stream)))


def silu_mul(gate_up, out, stream=None):
    """orion_silu_mul: out = SiLU(gate) * up for gate_up = [gate | up] per row."""
    _require_cuda(gate_up, out)
    _lib.check(lib().orion_silu_mul(int(gate_up.shape[0]), int(out.shape[-1]), gate_up.data_ptr(),
                                    out.data_ptr(), _stream_ptr(stream)))


class ExpansionBatch:
    """The in-flight set of one GPU: several queries, each a point DAG whose points all decode.

    queries: list of dicts {n_points, edges, prefix_pt_off, prefix_len}; points of query i are
             global branches branch0_i .. branch0_i + n_points - 1 in order.
    points:  per global branch (pt_off, content_len, capacity).
    page_table: int32 array of physical page ids; own_len: int32 [n_branches] current lengths.
    """

    def __init__(self, hq, hkv, d, page, queries, points, page_table, own_len,
                 policy=POLICY_ANCESTORS, device="cuda", chunk_tokens=0, sm_scale=0.0, flags=0,
                 num_sms=0, prefill_rows=0, kv_interleaved=False):
        import torch
        self.hq, self.hkv, self.d, self.page = hq, hkv, d, page
        self.sm_scale = sm_scale
        self.kv_interleaved = bool(kv_interleaved)
        qdesc, offs, refs, b0 = [], [0], [], 0
        for q in queries:
            w = dag_waves(q["n_points"], q["edges"], policy)
            so = w["seg_offsets"]
            for j in range(q["n_points"]):
                refs.append(w["segs"][so[j]:so[j + 1]])
                offs.append(offs[-1] + int(so[j + 1] - so[j]))
            qdesc.append((q["n_points"], b0, q["prefix_pt_off"], q["prefix_len"]))
            b0 += q["n_points"]
        self.n_branches = b0
        self.seg_offsets = np.array(offs, np.int32)
        self.refs = np.concatenate(refs) if refs else np.zeros(0, SEGREF_DTYPE)
        pts = np.array(points, np.int32).reshape(-1, 3)
        self.segs = bind_segments(qdesc, pts, self.seg_offsets, self.refs)
        self._setup(self.seg_offsets, self.segs, pts[:, 0], pts[:, 2], page_table, own_len, device,
                    chunk_tokens, flags, num_sms, prefill_rows)

    @classmethod
    def from_segments(cls, hq, hkv, d, page, seg_offsets, segs, own_pt_off, own_cap, page_table,
                      own_len, device="cuda", chunk_tokens=0, sm_scale=0.0, flags=0, num_sms=0,
                      prefill_rows=0, kv_interleaved=False):
        """A batch over already-bound segment lists (e.g. orion_select_branches' running set):
        own_pt_off / own_cap / own_len per branch of the lists."""
        self = cls.__new__(cls)
        self.hq, self.hkv, self.d, self.page = hq, hkv, d, page
        self.sm_scale = sm_scale
        self.kv_interleaved = bool(kv_interleaved)
        self.n_branches = len(seg_offsets) - 1
        self.seg_offsets = np.ascontiguousarray(seg_offsets, np.int32)
        self.segs = segs
        self._setup(self.seg_offsets, segs, own_pt_off, own_cap, page_table, own_len, device,
                    chunk_tokens, flags, num_sms, prefill_rows)
        return self

    def _setup(self, seg_offsets, segs, own_pt_off, own_cap, page_table, own_len, device,
               chunk_tokens, flags, num_sms, prefill_rows):
        import torch
        own = np.ascontiguousarray(own_len, dtype=np.int32)
        self.h_plan, ws = expand_plan(self.hq, self.hkv, self.d, self.page, seg_offsets, segs, own,
                                      chunk_tokens=chunk_tokens, sm_scale=self.sm_scale, flags=flags,
                                      num_sms=num_sms, prefill_rows=prefill_rows)
        self.prefill_rows = prefill_rows
        self.stats = plan_stats(self.h_plan)
        dev = torch.device(device)
        self.d_plan = torch.from_numpy(self.h_plan.copy()).to(dev)
        # zeroed once: the split kernels' work counter must start at zero (include/orion.h)
        self.workspace = torch.zeros((ws + 15) // 16 * 4, dtype=torch.float32, device=dev)
        self.page_table = (page_table if isinstance(page_table, torch.Tensor)
                           else torch.from_numpy(np.ascontiguousarray(page_table, np.int32)).to(dev))
        self.own_pt_off = torch.from_numpy(np.ascontiguousarray(own_pt_off, np.int32)).to(dev)
        self.own_cap = torch.from_numpy(np.ascontiguousarray(own_cap, np.int32)).to(dev)
        self.own_len = torch.from_numpy(own.copy()).to(dev)

    def pos_base(self):
        """orion_context_base at the current lengths: per branch, the context tokens before its
        own run; the RoPE position of its token at own slot s is pos_base + s (reading M2)."""
        return context_base(self.seg_offsets, self.segs, self.own_len.cpu().numpy())

    def rope_append(self, qkv, q_out, k_cache, v_cache, pos_base, rope_theta=500000.0,
                    mode=APPEND_ADVANCE, stream=None):
        """orion_rope_append: rotate q / k of the QKV GEMM output at pos_base + slot, write q,
        append k / v to the branches' own runs.  pos_base: device int32 [n_branches]."""
        _require_cuda(qkv, q_out, k_cache, v_cache, pos_base)
        shape = _shape(self.hq, self.hkv, self.d, self.page, self.sm_scale, self.kv_interleaved)
        _lib.check(lib().orion_rope_append(
            ctypes.byref(shape), self.n_branches, qkv.data_ptr(), q_out.data_ptr(), k_cache.data_ptr(),
            v_cache.data_ptr(), self.own_pt_off.data_ptr(), self.own_cap.data_ptr(),
            self.page_table.data_ptr(), int(k_cache.shape[0]), self.own_len.data_ptr(),
            pos_base.data_ptr(), float(rope_theta), int(mode), _stream_ptr(stream)))

    def step_launches(self):
        """orion_step_launches: kernels one step() enqueues with this plan on the current device."""
        n = np.zeros(1, np.int32)
        _lib.check(lib().orion_step_launches(_lib.ptr(self.h_plan), _lib.ptr(n)))
        return int(n[0])

    def append(self, k_new, v_new, k_cache, v_cache, mode=APPEND_ADVANCE, stream=None):
        kv_append(self.hq, self.hkv, self.d, self.page, k_new, v_new, k_cache, v_cache,
                  self.own_pt_off, self.own_cap, self.page_table, self.own_len, mode, stream,
                  self.kv_interleaved)

    def attend(self, q, out, k_cache, v_cache, lse=None, stream=None):
        """Decode attention (q/out [B, Hq, d]); with a prefill_rows = Lc batch, the point-prefill
        attention of the Pre stage (q/out [B, Lc, Hq, d], lse [B, Lc, Hq])."""
        f = point_prefill_attn if self.prefill_rows else expand_attn
        f(self.hq, self.hkv, self.d, self.page, q, out, lse, k_cache, v_cache, self.page_table,
          self.own_len, self.h_plan, self.d_plan, self.workspace, stream, self.sm_scale,
          self.kv_interleaved)

    def split(self, q, k_cache, v_cache, stream=None):
        expand_split(self.hq, self.hkv, self.d, self.page, q, k_cache, v_cache, self.page_table,
                     self.own_len, self.h_plan, self.d_plan, self.workspace, stream, self.sm_scale,
                     self.kv_interleaved)

    def combine(self, out, lse=None, stream=None):
        expand_combine(self.hq, self.hkv, self.d, self.page, self.n_branches, out, lse,
                       self.h_plan, self.d_plan, self.workspace, stream, self.sm_scale,
                       self.kv_interleaved)

    def step(self, q, k_new, v_new, k_cache, v_cache, out, lse=None, mode=APPEND_ADVANCE,
             stream=None, fused=True):
        """One expansion decode step for one layer: K1 append, then K2 split + K3 combine --
        orion_expand_step (the append inside the split launch where the plan allows), or with
        fused=False the two calls."""
        if fused and not self.prefill_rows:
            expand_step(self.hq, self.hkv, self.d, self.page, q, k_new, v_new, out, lse, k_cache, v_cache,
                        self.page_table, self.own_pt_off, self.own_cap, self.own_len, self.h_plan, self.d_plan,
                        self.workspace, mode, stream, self.sm_scale, self.kv_interleaved)
            return
        self.append(k_new, v_new, k_cache, v_cache, mode, stream)
        self.attend(q, out, k_cache, v_cache, lse, stream)
