"""One whole expansion decode step on the CPU, composed from O1-O4 for a workloads.Layout.

Per query: segment lists (O1, dag.segment_lists) -> binding (O2, bind.bind_segments)
-> attention (O3, attention.expand_attn).  `branches` restricts the (slow) attention
to a sample of global branch indices (used for full-size sampled parity and timing).
"""
import numpy as np

from . import dag, bind, attention


def bound_segments(layout, policy=dag.ANCESTORS, own_len=None):
    """Global-branch-indexed list of bound segments [(pages, start, len)]."""
    own_len = layout.own_len if own_len is None else own_len
    out = [None] * layout.n_branches
    for qi in range(layout.n_queries):
        n = int(layout.n_points[qi])
        b0 = int(layout.branch0[qi])
        lists = dag.segment_lists(n, layout.edges[qi], policy)
        prefix_pages = layout.pages_of(layout.prefix_pt_off[qi], layout.prefix_len[qi])
        pp, lc, ol = {}, {}, {}
        for k in range(1, n + 1):
            b = b0 + k - 1
            pp[k] = layout.pages_of(layout.point_pt_off[b], layout.point_cap[b])
            lc[k] = int(layout.content_len[b])
            ol[k] = int(own_len[b])
        bound = bind.bind_segments(lists, prefix_pages, int(layout.prefix_len[qi]), pp, lc, ol)
        for k in range(1, n + 1):
            out[b0 + k - 1] = bound[k]
    return out


def expand_step(layout, q_u16, k_u16, v_u16, policy=dag.ANCESTORS, branches=None, scale=None,
                own_len=None):
    """Returns (out [nb,Hq,d] f64, lse [nb,Hq] f64) for `branches` (default: all)."""
    bound = bound_segments(layout, policy, own_len)
    if branches is None:
        branches = list(range(layout.n_branches))
    q = np.asarray(q_u16)[branches]
    sel = [bound[b] for b in branches]
    return attention.expand_attn(q, k_u16, v_u16, sel, layout.page_size, scale)
