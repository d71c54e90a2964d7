"""O5 — point-prefill attention (the Pre stage), by its plain definition (NumPy fp64).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by the product path.

PAPER.md Alg. 1 l.12 / l.19 and Eq. (2): before point j decodes, its
input Input_j = Concat(Prompt_Pre, (+)_{k in Par(j)} f(k,j), P_j) is prefilled.  At KV level
(reading R-A: the prefix's and the dependencies' KV are already cached)
the new rows are the Lc_j content tokens of P_j, the first Lc_j tokens of j's own page run, and

    content token i of point j attends to
        ctx_i(j) = [ j's bound segments except OWN, in list order (O2) ] ‖ P_j[0 .. i]

i.e. the same dependency context as j's decode step (reading S7 / S8: FULL(a) iff Dec(a) happens
before Pre(j), else CONTENT(a); or the EQ3 spans) plus causal attention over P_j itself.
    s = scale * q[j,i,h] . K_ctx^T,  out[j,i,h] = softmax(s) . V_ctx,  lse[j,i,h] = m + ln sum e^(s-m)
with kv head g = h // G (reading S16) and bf16 widened exactly (O3).
"""
import numpy as np

from . import dag
from .attention import attend, bf16_to_f64, context, gather_tokens
from .step import bound_segments


def point_prefill(layout, q_u16, k_u16, v_u16, policy=dag.ANCESTORS, branches=None, scale=None,
                  own_len=None):
    """q_u16 [B, Lc, Hq, d] raw bf16 (row i of branch b = content token i of its point; every
    branch has content_len == Lc); k/v_u16 [pages, Hkv, P, d].  Returns (out [nb, Lc, Hq, d] f64,
    lse [nb, Lc, Hq] f64) for `branches` (default all), one query row at a time."""
    bound = bound_segments(layout, policy, own_len)
    q = bf16_to_f64(q_u16)
    B, Lc, Hq, d = q.shape
    Hkv = k_u16.shape[1]
    G = Hq // Hkv
    P = layout.page_size
    scale = 1.0 / np.sqrt(d) if scale is None else scale
    if branches is None:
        branches = list(range(layout.n_branches))
    out = np.zeros((len(branches), Lc, Hq, d))
    lse = np.zeros((len(branches), Lc, Hq))
    for n, b in enumerate(branches):
        if int(layout.content_len[b]) != Lc:
            raise ValueError(f"branch {b}: content_len {layout.content_len[b]} != Lc {Lc}")
        segs = bound[b]
        own_pages, own_start, _ = segs[-1]          # OWN(j) is the last entry of every list (O1)
        assert own_start == 0
        for g in range(Hkv):
            # raw bf16 rows gathered, then widened exactly (as widening the whole cache first)
            kc = bf16_to_f64(context(k_u16, segs[:-1], g, P)) if len(segs) > 1 else np.zeros((0, d))
            vc = bf16_to_f64(context(v_u16, segs[:-1], g, P)) if len(segs) > 1 else np.zeros((0, d))
            ko = bf16_to_f64(gather_tokens(k_u16, own_pages, 0, Lc, g, P))
            vo = bf16_to_f64(gather_tokens(v_u16, own_pages, 0, Lc, g, P))
            for i in range(Lc):
                kk = np.concatenate([kc, ko[:i + 1]], axis=0)
                vv = np.concatenate([vc, vo[:i + 1]], axis=0)
                o, l = attend(q[b, i, g * G:(g + 1) * G], kk, vv, scale)
                out[n, i, g * G:(g + 1) * G] = o
                lse[n, i, g * G:(g + 1) * G] = l
    return out, lse
