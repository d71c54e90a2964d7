"""O2 — physical binding of symbolic segments to token ranges in pages.

Point k owns the pages holding S_k = [P_k (Lc_k tokens) ‖ Output_k] (reading
S7/S19).  Each segment becomes (pages, start, length):

    PREFIX     -> (prefix pages, 0, Lp)            Prompt_Pre of Eq. (2), reading S13
    CONTENT(k) -> (pages_k, 0, Lc_k)               f(k,j) = P_k, Eq. (3) Contextual
    FULL(k)    -> (pages_k, 0, T_k)                ANCESTORS Dependent span, reading S7
    OUTPUT(k)  -> (pages_k, Lc_k, T_k - Lc_k)      f(k,j) = Output_k, Eq. (3) Dependent
    OWN(j)     -> (pages_j, 0, T_j)                P_j plus j's own generated tokens

T_k is point k's current segment length (own_len_k, which includes the token
being decoded — reading S15).  Token t of a bound segment lives on page
pages[(start + t) // P], row (start + t) % P.
"""
from .dag import SEG_PREFIX, SEG_CONTENT, SEG_FULL, SEG_OUTPUT, SEG_OWN


def bind_segments(lists, prefix_pages, lp, point_pages, lc, own_len):
    """lists: {j: [(kind, point)]} for points 1..n.  point_pages/lc/own_len indexed by point id.
    Returns {j: [(pages, start, length)]} in list order."""
    out = {}
    for j, refs in lists.items():
        segs = []
        for kind, k in refs:
            if kind == SEG_PREFIX:
                segs.append((prefix_pages, 0, lp))
            elif kind == SEG_CONTENT:
                segs.append((point_pages[k], 0, lc[k]))
            elif kind == SEG_FULL:
                segs.append((point_pages[k], 0, own_len[k]))
            elif kind == SEG_OUTPUT:
                segs.append((point_pages[k], lc[k], own_len[k] - lc[k]))
            elif kind == SEG_OWN:
                segs.append((point_pages[k], 0, own_len[k]))
            else:
                raise ValueError(kind)
        out[j] = segs
    return out
