"""Host side of the expansion driver: orion_expansion_round against the
oracle schedule O6 (bit-exact, integer work), orion_select_branches against the oracle binding
O2 with the unselected points' lengths frozen."""
import random

import numpy as np
import pytest

import paper_2510_24390_b200 as orion
from paper_2510_24390_b200 import _lib
from oracle import expansion as OE, step as OS
from workloads import configs as C, tensors as T, dags as W


def run_rounds(queries, tokens):
    qd, eo, ed, b0 = [], [0], [], 0
    for n, edges in queries:
        qd.append((n, b0, 0, 0))
        ed += list(edges)
        eo.append(len(ed))
        b0 += n
    tok = np.array(tokens, np.int32)
    pre_r = np.full(b0, -1, np.int32)
    dec_r = np.full(b0, -1, np.int32)
    left = tok.copy()
    out = []
    for r in range(100000):
        p, d = orion.expansion_round(qd, eo, ed, tok, pre_r, dec_r, left, r)
        if len(p) == 0 and len(d) == 0:
            break
        out.append((list(map(int, p)), list(map(int, d))))
    assert (dec_r >= 0).all() and (left == 0).all()
    return out


def test_expansion_round_matches_oracle_schedule():
    rng = random.Random(3)
    for trial in range(60):
        qs, tokens, b0, oq = [], [], 0, []
        for _ in range(rng.randint(1, 4)):
            n = rng.randint(1, 9)
            edges = W.random_dag(random.Random(1000 + trial * 7 + b0), n, p=rng.choice([0.2, 0.5]),
                                 null_frac=0.2)[1]
            qs.append((n, edges))
            oq.append((n, edges, b0))
            tokens += [rng.randint(0, 5) for _ in range(n)]
            b0 += n
        assert run_rounds(qs, tokens) == OE.batch_schedule(oq, tokens)


def test_expansion_round_paper_dags_and_errors():
    for dagf in (W.diamond, W.fig4, W.mixed8, W.mixed16):
        n, edges = dagf()
        assert run_rounds([(n, edges)], [7] * n) == OE.batch_schedule([(n, edges, 0)], [7] * n)
    # a cycle stalls -> CYCLE; an out-of-query edge -> UNKNOWN_POINT
    with pytest.raises(orion.OrionError) as ei:
        run_rounds([(2, [(1, 2, 2), (2, 1, 1)])], [1, 1])
    assert ei.value.code == _lib.ERR_CYCLE
    with pytest.raises(orion.OrionError) as ei:
        run_rounds([(2, [(1, 3, 2)])], [1, 1])
    assert ei.value.code == _lib.ERR_UNKNOWN_POINT


@pytest.mark.parametrize("policy", [0, 1])
def test_select_branches_matches_oracle_binding(policy):
    cfg = C.CONFIGS["c1"].with_(n_queries=2, dag="mixed8", lp=100, t=60, lc=8, page=16)
    lay = T.make_layout(cfg, ragged=True)
    from tests.test_host_lib import _bind_layout
    offs, segs = _bind_layout(cfg, lay, policy)
    rng = np.random.default_rng(4)
    for trial in range(20):
        own = lay.own_len.copy()
        own[:] = rng.integers(cfg.lc, lay.point_cap + 1)
        sel = np.sort(rng.choice(lay.n_branches, rng.integers(1, lay.n_branches + 1), replace=False))
        so, sg = orion.select_branches(offs, segs, own, sel)
        bound = OS.bound_segments(lay, policy, own_len=own)
        for i, br in enumerate(sel):
            mine = sg[so[i]:so[i + 1]]
            assert len(mine) == len(bound[br])
            for k, (s, (pages, start, length)) in enumerate(zip(mine, bound[br])):
                orig = segs[offs[br] + k]
                assert (s["pt_off"], s["start"]) == (orig["pt_off"], orig["start"])
                if s["dyn"] >= 0:                    # still growing: remapped to its selection index
                    assert sel[s["dyn"]] == orig["dyn"]
                    eff = min(max(own[orig["dyn"]] - s["start"], 0), s["len"])
                else:                                # static, or frozen at the current length
                    assert orig["dyn"] < 0 or orig["dyn"] not in set(sel.tolist())
                    eff = s["len"]
                assert (int(s["start"]), int(eff)) == (start, length)
    with pytest.raises(orion.OrionError):
        orion.select_branches(offs, segs, lay.own_len, [0, 0])


def _expansion(cfg, lay, policy=0):
    from paper_2510_24390_b200.expansion import Expansion
    queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i],
                    prefix_pt_off=int(lay.prefix_pt_off[i]), prefix_len=int(lay.prefix_len[i]))
               for i in range(lay.n_queries)]
    points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
    tokens = (np.asarray(lay.own_len) - cfg.lc).astype(np.int32)
    return Expansion(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, lay.page_table, cfg.lc,
                     tokens, policy=policy, device="cpu")


@pytest.mark.parametrize("policy", [0, 1])
def test_expansion_roofline_bytes_brute_force(policy):
    # bench.expansion_decode_bytes (the whole-expansion roofline numerator) against a brute-force
    # count: per decode round, the set of distinct (page run, token) pairs the running branches'
    # oracle-bound contexts (O2, lengths at attention time) touch, x Hkv x d x 2 x 2 B, plus q/out.
    import bench
    cfg = C.CONFIGS["c1"].with_(n_queries=2, lp=40, t=24, lc=8, page=16)
    lay = T.make_layout(cfg, dag_override=W.mixed8)
    ex = _expansion(cfg, lay, policy)
    schedule = []
    while True:
        pre, dec = ex.next_round()
        if len(pre) == 0 and len(dec) == 0:
            break
        if len(pre):
            ex.own_len[pre] = cfg.lc
        if len(dec):
            schedule.append(np.array(dec))
            ex.own_len[dec] += 1
    got = bench.expansion_decode_bytes(cfg, lay, ex, schedule, layers=1)
    own = np.full(lay.n_branches, cfg.lc)
    want = 0
    for dec in schedule:
        cur = own.copy()
        cur[dec] += 1
        bound = OS.bound_segments(lay, policy, own_len=cur)
        toks = set()
        for b in dec:
            for pages, start, ln in bound[b]:
                toks.update((int(pages[(start + t) // cfg.page]), (start + t) % cfg.page) for t in range(ln))
        want += len(toks) * cfg.hkv * cfg.d * 4 + len(dec) * cfg.hq * cfg.d * 4
        own[dec] += 1
    assert got == want
