"""Seeded bf16 tensors and the paged memory layout.

Layout (DESIGN.md §"HBM layout"): one page pool per layer, K and V each
`[num_pages, Hkv, P, d]` bf16.  Every query owns a run of page-table entries
for its shared prefix, and every point (branch) owns a run for its segment
S_k = [P_k content ‖ Output_k].  Which physical page backs a page-table entry
is a seeded random permutation of a pool 10% larger than needed (SURVEY.md
§8(d) "Concrete synthetic inputs").  No method arithmetic here.
"""
from dataclasses import dataclass, field
import numpy as np
import torch

from .dags import DAGS


def bf16_randn_u16(shape, seed, device="cpu", scale=1.0):
    """i.i.d. N(0,1)*scale rounded to bf16; returned as a torch bf16 tensor on `device`."""
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    x = torch.randn(*shape, generator=g, device=device, dtype=torch.float32)
    if scale != 1.0:
        x = x * scale
    return x.to(torch.bfloat16)


@dataclass
class Layout:
    page_size: int
    n_queries: int
    n_points: np.ndarray      # [Q]
    branch0: np.ndarray       # [Q] global branch index of point 1
    edges: list               # [Q] list of (from, to, kind)
    prefix_pt_off: np.ndarray  # [Q]
    prefix_len: np.ndarray    # [Q]
    point_pt_off: np.ndarray  # [B]
    point_cap: np.ndarray     # [B] capacity in tokens (pages * P)
    content_len: np.ndarray   # [B] Lc
    own_len: np.ndarray       # [B] current |S_b| (includes the token being decoded)
    branch_query: np.ndarray  # [B]
    page_table: np.ndarray    # [n_entries] int32 physical page ids
    num_pages: int            # pool size
    extra: dict = field(default_factory=dict)

    @property
    def n_branches(self):
        return int(self.point_pt_off.shape[0])

    def pages_of(self, pt_off, n_tokens):
        n = -(-int(n_tokens) // self.page_size)
        return [int(p) for p in self.page_table[pt_off:pt_off + n]]


def make_layout(cfg, queries=None, seed=None, contiguous=False, ragged=False,
                extra_tokens=0, dag_override=None, pool_slack=0.10):
    """Allocate page-table runs for `queries` (default: all cfg.n_queries) of config `cfg`."""
    if queries is None:
        queries = list(range(cfg.n_queries))
    seed = cfg.seed if seed is None else seed
    P = cfg.page
    n_points, branch0, edges, pre_off, pre_len = [], [], [], [], []
    pt_off, cap, lc, own, bq = [], [], [], [], []
    entries = 0
    b = 0
    for qi, q in enumerate(queries):
        n, e = (dag_override or DAGS[cfg.dag])()
        n_points.append(n)
        branch0.append(b)
        edges.append(list(e))
        pre_off.append(entries)
        pre_len.append(cfg.lp)
        entries += -(-cfg.lp // P)
        for j in range(1, n + 1):
            c = -(-(cfg.t + extra_tokens) // P) * P
            pt_off.append(entries)
            cap.append(c)
            lc.append(cfg.lc)
            if ragged and cfg.t > cfg.lc + 1:
                own.append(cfg.lc + 1 + ((7919 * (b + 1)) % (cfg.t - cfg.lc)))
            else:
                own.append(cfg.t)
            bq.append(qi)
            entries += c // P
            b += 1
    pool = entries if contiguous else int(np.ceil(entries * (1.0 + pool_slack)))
    if contiguous:
        table = np.arange(entries, dtype=np.int32)
    else:
        rng = np.random.default_rng(seed)
        table = rng.permutation(pool)[:entries].astype(np.int32)
    return Layout(P, len(queries), np.array(n_points, np.int32), np.array(branch0, np.int32), edges,
                  np.array(pre_off, np.int32), np.array(pre_len, np.int32),
                  np.array(pt_off, np.int32), np.array(cap, np.int32), np.array(lc, np.int32),
                  np.array(own, np.int32), np.array(bq, np.int32), table, pool)


def subset_layout(lay, queries):
    """The sub-batch of `lay` holding only `queries` (in that order), with the same page table and
    pool: what one rank of a strong-scaling run owns.  Returns (layout, branch ids in `lay`)."""
    n_points, branch0, edges, pre_off, pre_len, branches = [], [], [], [], [], []
    b = 0
    for qi in queries:
        n = int(lay.n_points[qi])
        n_points.append(n)
        branch0.append(b)
        edges.append(list(lay.edges[qi]))
        pre_off.append(int(lay.prefix_pt_off[qi]))
        pre_len.append(int(lay.prefix_len[qi]))
        branches += range(int(lay.branch0[qi]), int(lay.branch0[qi]) + n)
        b += n
    br = np.array(branches, np.int64)
    bq = np.repeat(np.arange(len(queries), dtype=np.int32), n_points) if queries else np.zeros(0, np.int32)
    sub = Layout(lay.page_size, len(queries), np.array(n_points, np.int32), np.array(branch0, np.int32),
                 edges, np.array(pre_off, np.int32), np.array(pre_len, np.int32),
                 lay.point_pt_off[br].copy(), lay.point_cap[br].copy(), lay.content_len[br].copy(),
                 lay.own_len[br].copy(), bq, lay.page_table, lay.num_pages)
    return sub, br


def make_qkv(cfg, layout, seed=None, device="cpu", q_scale=1.0, sink=False, layers=1):
    """Per-layer caches and per-step inputs.  Returns a dict of torch bf16 tensors:
    k_cache/v_cache [layers, num_pages, Hkv, P, d], q [layers, B, Hq, d], k_new/v_new [layers, B, Hkv, d]."""
    seed = cfg.seed if seed is None else seed
    B = layout.n_branches
    shp_cache = (layers, layout.num_pages, cfg.hkv, cfg.page, cfg.d)
    k = bf16_randn_u16(shp_cache, seed * 16 + 1, device)
    v = bf16_randn_u16(shp_cache, seed * 16 + 2, device)
    q = bf16_randn_u16((layers, B, cfg.hq, cfg.d), seed * 16 + 3, device, scale=q_scale)
    kn = bf16_randn_u16((layers, B, cfg.hkv, cfg.d), seed * 16 + 4, device)
    vn = bf16_randn_u16((layers, B, cfg.hkv, cfg.d), seed * 16 + 5, device)
    if sink:
        for qi in range(layout.n_queries):
            pg = int(layout.page_table[layout.prefix_pt_off[qi]])
            k[:, pg, :, 0, :] = (k[:, pg, :, 0, :].float() * 8.0).to(torch.bfloat16)
    return {"k_cache": k, "v_cache": v, "q": q, "k_new": kn, "v_new": vn}
