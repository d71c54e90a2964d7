"""T1 — the native host library (no GPU needed): symbols, orion_dag_waves bit-exact against
the oracle (goldens + fuzz, both policies, error taxonomy), orion_bind_segments against the
oracle's binding, and orion_expand_plan coverage properties (every row's partial items cover
exactly its context, once)."""
import random
import re

import numpy as np
import pytest

import paper_2510_24390_b200 as orion
from paper_2510_24390_b200 import _lib
from oracle import dag as OD, step as OS
from workloads import dags as W, configs as C, tensors as T

HEADER = open(__file__.rsplit("/tests/", 1)[0] + "/include/orion.h").read()


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    decl = set(re.findall(r"^\s*(?:orion_status|const char\*)\s+(orion_\w+)\(", HEADER, re.M))
    assert decl == set(_lib.EXPORTED_SYMBOLS)
    for name in decl:
        assert hasattr(L, name), name
    assert "sm_100a" in orion.version()


def _oracle_or_error(n, edges, policy):
    try:
        return OD.levels(n, edges), OD.waves(n, edges), OD.segment_lists(n, edges, policy), None
    except OD.DagError as e:
        return None, None, None, e


def _compare(n, edges, policy):
    lev, waves, lists, err = _oracle_or_error(n, edges, policy)
    if err is not None:
        with pytest.raises(orion.OrionError) as ei:
            orion.dag_waves(n, edges, policy)
        assert ei.value.code == err.code
        if err.code == OD.CYCLE:
            cyc = ei.value.info
            es = {(a, b) for a, b, k in edges if k}
            assert cyc and all((cyc[i], cyc[(i + 1) % len(cyc)]) in es for i in range(len(cyc)))
        else:
            assert ei.value.info[:1] == err.info
        return
    got = orion.dag_waves(n, edges, policy)
    assert list(got["pre_level"]) == lev[0] and list(got["dec_level"]) == lev[1]
    assert got["n_levels"] == lev[2]
    assert got["waves"] == waves
    so, segs = got["seg_offsets"], got["segs"]
    for j in range(1, n + 1):
        mine = [(int(s["kind"]), int(s["point"])) for s in segs[so[j - 1]:so[j]]]
        assert mine == lists[j], (j, mine, lists[j])


@pytest.mark.parametrize("name", list(W.DAGS))
@pytest.mark.parametrize("policy", [0, 1])
def test_dag_waves_named_families(name, policy):
    _compare(*W.DAGS[name](), policy)


def test_dag_waves_fuzz_bit_exact():
    rng = random.Random(2024)
    for i in range(1200):
        n = rng.randint(1, 64 if i % 10 == 0 else 12)
        n_, edges = W.random_dag(rng, n, p=rng.choice([0.05, 0.2, 0.5]), null_frac=0.15)
        if rng.random() < 0.2 and n > 1:   # inject cycles / bad points / bad kinds
            r = rng.random()
            if r < 0.5:
                a, b = rng.sample(range(1, n + 1), 2)
                edges = edges + [(a, b, 2), (b, a, rng.choice([1, 2]))]
            elif r < 0.75:
                edges = edges + [(rng.randint(1, n), n + rng.randint(1, 3), 1)]
            else:
                edges = edges + [(1, 2, 5)]
        _compare(n, edges, i % 2)


def test_dag_waves_errors_and_degenerate():
    with pytest.raises(orion.OrionError) as ei:
        orion.dag_waves(0, [])
    assert ei.value.code == _lib.ERR_INVALID_ARG
    with pytest.raises(orion.OrionError) as ei:
        orion.dag_waves(3, [], policy=7)
    assert ei.value.code == _lib.ERR_INVALID_ARG
    with pytest.raises(orion.OrionError) as ei:
        orion.dag_waves(2, [(2, 2, 2)])
    assert ei.value.code == _lib.ERR_CYCLE and ei.value.info == [2]
    g = orion.dag_waves(1, [])
    assert g["waves"] == [[(1, 0)], [(1, 1)]]


def _bind_layout(cfg, layout, policy):
    qdesc, offs, refs = [], [0], []
    for qi in range(layout.n_queries):
        n = int(layout.n_points[qi])
        w = orion.dag_waves(n, layout.edges[qi], policy)
        so = w["seg_offsets"]
        for j in range(n):
            refs.append(w["segs"][so[j]:so[j + 1]])
            offs.append(offs[-1] + int(so[j + 1] - so[j]))
        qdesc.append((n, int(layout.branch0[qi]), int(layout.prefix_pt_off[qi]), int(layout.prefix_len[qi])))
    pts = np.stack([layout.point_pt_off, layout.content_len, layout.point_cap], 1)
    segs = orion.bind_segments(qdesc, pts, np.array(offs, np.int32), np.concatenate(refs))
    return np.array(offs, np.int32), segs


@pytest.mark.parametrize("cfgname", ["c1", "c2", "c3"])
@pytest.mark.parametrize("policy", [0, 1])
def test_bind_matches_oracle_binding(cfgname, policy):
    cfg = C.CONFIGS[cfgname].with_(n_queries=min(C.CONFIGS[cfgname].n_queries, 3))
    lay = T.make_layout(cfg, ragged=True, extra_tokens=cfg.page)
    offs, segs = _bind_layout(cfg, lay, policy)
    bound = OS.bound_segments(lay, policy)
    for b in range(lay.n_branches):
        mine = segs[offs[b]:offs[b + 1]]
        assert len(mine) == len(bound[b])
        for s, (pages, start, length) in zip(mine, bound[b]):
            eff = s["len"] if s["dyn"] < 0 else min(max(lay.own_len[s["dyn"]] - s["start"], 0), s["len"])
            assert (int(s["start"]), int(eff)) == (start, length)
            npg = -(-int(s["start"] + s["len"]) // cfg.page)
            assert list(lay.page_table[s["pt_off"]:s["pt_off"] + npg]) == list(pages[:npg])


@pytest.mark.parametrize("cfgname", ["c1", "c2", "c3"])
@pytest.mark.parametrize("policy", [0, 1])
def test_context_base_matches_oracle_positions(cfgname, policy):
    """orion_context_base (the product's RoPE position base, reading M2) against the oracle's own
    derivation from O1/O2 (oracle.decoder.token_positions), at two sets of lengths."""
    from oracle import decoder as DE
    cfg = C.CONFIGS[cfgname].with_(n_queries=min(C.CONFIGS[cfgname].n_queries, 3))
    lay = T.make_layout(cfg, ragged=True, extra_tokens=cfg.page)
    offs, segs = _bind_layout(cfg, lay, policy)
    for own in (lay.own_len, np.maximum(lay.own_len - 7, 0)):
        got = orion.context_base(offs, segs, own)
        want = DE.token_positions(OS.bound_segments(lay, policy, own_len=own), np.zeros_like(own))
        assert np.array_equal(got, want)


def test_context_base_random_dags_and_errors():
    from oracle import decoder as DE
    rng = random.Random(9)
    for trial in range(60):
        cfg = C.CONFIGS["c1"].with_(lp=rng.randint(0, 90), t=rng.randint(9, 70), lc=8, page=16)
        n = rng.randint(1, 9)
        dag = W.random_dag(rng, n, 0.4)
        lay = T.make_layout(cfg, ragged=True, extra_tokens=16, dag_override=lambda: dag)
        policy = trial % 2
        offs, segs = _bind_layout(cfg, lay, policy)
        got = orion.context_base(offs, segs, lay.own_len)
        want = DE.token_positions(OS.bound_segments(lay, policy), np.zeros(lay.n_branches, np.int64))
        assert np.array_equal(got, want)
    bad = segs.copy()
    bad["dyn"][offs[1] - 1] = -1                     # branch 0 loses its OWN segment
    with pytest.raises(orion.OrionError):
        orion.context_base(offs, bad, lay.own_len)


# ------------------------------------------------------------------ plan parsing (test side)
HDR = np.dtype([("magic", "<i4"), ("version", "<i4"), ("n_branches", "<i4"), ("hq", "<i4"),
                ("hkv", "<i4"), ("d", "<i4"), ("page", "<i4"), ("group", "<i4"),
                ("n_items", "<i4"), ("n_partials", "<i4"), ("n_rows", "<i4"), ("n_readers", "<i4"),
                ("items_off", "<i8"), ("readers_off", "<i8"), ("comb_off_off", "<i8"),
                ("comb_slot_off", "<i8"), ("plan_bytes", "<i8"), ("workspace_bytes", "<i8"),
                ("acc_bytes", "<i8"), ("n_pieces", "<i8"), ("unique_tokens", "<i8"),
                ("logical_tokens", "<i8"), ("sm_scale", "<f4"), ("pad", "<i4", 3),
                ("ranges_off", "<i8"), ("n_ranges", "<i4"), ("paired", "<i4"),
                ("streamed_tokens", "<i8"), ("counter_off", "<i8"), ("n_big", "<i4"), ("pad0", "<i4"),
                ("plan_id", "<u8")])
RANGE = np.dtype([(n, "<i4") for n in ("pt_off", "t0", "t1", "dyn", "flags", "r0", "r1", "r2")])
ITEM = np.dtype([(n, "<i4") for n in ("pt_off", "t0", "t1", "dyn", "kv_head", "readers_off",
                                      "row_begin", "n_rows", "slot0", "piece", "p0", "p1")])


def parse_plan(plan):
    h = np.frombuffer(plan, HDR, 1)[0]
    items = np.frombuffer(plan, ITEM, int(h["n_items"]), int(h["items_off"]))
    readers = np.frombuffer(plan, "<i4", int(h["n_readers"]), int(h["readers_off"]))
    coff = np.frombuffer(plan, "<i4", int(h["n_rows"]) + 1, int(h["comb_off_off"]))
    cslot = np.frombuffer(plan, "<i4", int(h["n_partials"]), int(h["comb_slot_off"]))
    return h, items, readers, coff, cslot


def _check_plan_covers(cfg, lay, offs, segs, own_len, flags=0, chunk_tokens=128):
    plan, ws = orion.expand_plan(cfg.hq, cfg.hkv, cfg.d, cfg.page, offs, segs, own_len,
                                 chunk_tokens=chunk_tokens, flags=flags)
    h, items, readers, coff, cslot = parse_plan(plan)
    G = cfg.hq // cfg.hkv
    assert h["magic"] == 0x314e524f and h["n_rows"] == lay.n_branches * cfg.hq
    variant = int(h["pad"][0])                      # 2 = tcgen05 swap-AB: fp16 partials (plan_format.h)
    assert ws >= h["n_partials"] * ((cfg.d * 2 + 4) if variant == 2 else (cfg.d * 4 + 8))
    slot_tokens = {}
    slot_row = {}
    ranges = np.frombuffer(plan, RANGE, int(h["n_ranges"]), int(h["ranges_off"]))
    for it in items:
        if it["p0"] & 2:                             # multi-range item: its ranges' tokens
            rl = [(int(r["pt_off"]), int(r["t0"]), int(r["t1"]), int(r["dyn"]),
                   int(r["r0"]) & 0xffffffff if r["flags"] & 4 else 0xffffffff)   # kRangeMasked
                  for r in ranges[it["pt_off"]:it["pt_off"] + it["p1"]]]
            assert len(rl) >= 1
        else:
            rl = [(int(it["pt_off"]), int(it["t0"]), int(it["t1"]), int(it["dyn"]), 0xffffffff)]
        for r in range(it["row_begin"], it["row_begin"] + it["n_rows"]):
            b = readers[it["readers_off"] + r // G]
            hh = it["kv_head"] * G + r % G
            s = it["slot0"] + r - it["row_begin"]
            toks = []
            for pt, t0, t1, dyn, mask in rl:         # a masked range: only the readers in its mask
                if (mask >> (r // G)) & 1:
                    end = t1 if dyn < 0 else min(t1, own_len[dyn])
                    toks += [(pt, t) for t in range(t0, max(t0, end))]
            assert s not in slot_tokens
            slot_tokens[s] = toks
            slot_row[s] = b * cfg.hq + hh
    assert sorted(slot_tokens) == list(range(h["n_partials"]))
    for row in range(h["n_rows"]):
        b, hh = divmod(row, cfg.hq)
        got = []
        for s in cslot[coff[row]:coff[row + 1]]:
            assert slot_row[s] == row
            got += slot_tokens[s]
        want = []
        for s in segs[offs[b]:offs[b + 1]]:
            eff = s["len"] if s["dyn"] < 0 else min(max(own_len[s["dyn"]] - s["start"], 0), s["len"])
            want += [(int(s["pt_off"]), t) for t in range(s["start"], s["start"] + eff)]
        assert len(got) == len(set(got)) and sorted(got) == sorted(want)
    return h


@pytest.mark.parametrize("cfgname,policy", [("c1", 0), ("c1", 1), ("c2", 0), ("c3", 1)])
def test_plan_covers_each_context_exactly_once(cfgname, policy):
    cfg = C.CONFIGS[cfgname].with_(n_queries=2, lp=min(C.CONFIGS[cfgname].lp, 256),
                                   t=min(C.CONFIGS[cfgname].t, 96))
    lay = T.make_layout(cfg, ragged=True, extra_tokens=cfg.page)
    offs, segs = _bind_layout(cfg, lay, policy)
    h = _check_plan_covers(cfg, lay, offs, segs, lay.own_len)
    assert h["unique_tokens"] <= h["logical_tokens"]


def test_plan_random_dags_cover():
    rng = random.Random(77)
    for trial in range(25):
        cfg = C.CONFIGS["c1"].with_(lp=rng.choice([1, 16, 70]), t=rng.choice([9, 40, 100]),
                                    lc=rng.choice([0, 3, 8]), page=rng.choice([16, 32]),
                                    hq=rng.choice([2, 4, 6]), hkv=2, n_queries=2)
        n = rng.randint(1, 9)
        lay = T.make_layout(cfg, ragged=True, extra_tokens=rng.choice([0, 20]),
                            dag_override=lambda: W.random_dag(random.Random(trial), n, p=0.4))
        offs, segs = _bind_layout(cfg, lay, trial % 2)
        _check_plan_covers(cfg, lay, offs, segs, lay.own_len)


def test_plan_sharing_counts_c4():
    cfg = C.CONFIGS["c4"].with_(n_queries=1)
    lay = T.make_layout(cfg)
    offs, segs = _bind_layout(cfg, lay, 0)
    plan, ws = orion.expand_plan(cfg.hq, cfg.hkv, cfg.d, cfg.page, offs, segs, lay.own_len)
    st = orion.plan_stats(plan)
    # unique tokens per kv head = prefix + all point segments (capacity); logical/unique ~ 7.6
    assert st["unique_tokens"] == cfg.lp + 16 * cfg.t
    assert 7.0 < st["logical_tokens"] / st["unique_tokens"] < 8.0


def test_plan_errors():
    S = _lib.SEG_DTYPE
    # overlapping segments in one branch list
    segs = np.array([(0, 0, 10, -1), (0, 5, 10, -1)], S)
    with pytest.raises(orion.OrionError) as ei:
        orion.expand_plan(4, 2, 64, 16, np.array([0, 2], np.int32), segs)
    assert ei.value.code == _lib.ERR_INVALID_ARG
    # one page run growing with two branches
    segs = np.array([(0, 0, 10, 0), (0, 0, 10, 1)], S)
    with pytest.raises(orion.OrionError) as ei:
        orion.expand_plan(4, 2, 64, 16, np.array([0, 1, 2], np.int32), segs)
    assert ei.value.code == _lib.ERR_UNSUPPORTED
    # unsupported head_dim / page size
    segs = np.array([(0, 0, 10, -1)], S)
    for d, p in ((96, 16), (64, 24)):
        with pytest.raises(orion.OrionError) as ei:
            orion.expand_plan(4, 2, d, p, np.array([0, 1], np.int32), segs)
        assert ei.value.code == _lib.ERR_UNSUPPORTED
    # empty context
    segs = np.array([(0, 0, 0, -1)], S)
    with pytest.raises(orion.OrionError) as ei:
        orion.expand_plan(4, 2, 64, 16, np.array([0, 1], np.int32), segs)
    assert ei.value.code == _lib.ERR_INVALID_ARG
    # zero-length segments are skipped
    segs = np.array([(0, 0, 0, -1), (3, 0, 5, -1)], S)
    plan, _ = orion.expand_plan(4, 2, 64, 16, np.array([0, 2], np.int32), segs)
    assert orion.plan_stats(plan)["unique_tokens"] == 5


def test_device_entry_points_validate_without_gpu():
    import ctypes
    L = _lib.lib()
    shape = _lib.AttnShape(4, 2, 64, 16, 0.0)
    assert L.orion_kv_append(ctypes.byref(shape), 1, None, None, None, None, None, None, None, 8,
                             None, 0, None) == _lib.ERR_INVALID_ARG
    assert L.orion_expand_attn(ctypes.byref(shape), 1, None, None, None, None, None, 1, None,
                               None, None, None, None, 0, None) == _lib.ERR_INVALID_ARG
    bad = _lib.AttnShape(4, 2, 80, 16, 0.0)
    assert L.orion_kv_append(ctypes.byref(bad), 1, None, None, None, None, None, None, None, 8,
                             None, 0, None) == _lib.ERR_UNSUPPORTED
    fake = ctypes.c_void_p(16)                       # num_pages < 1 is refused before any launch
    assert L.orion_kv_append(ctypes.byref(shape), 1, fake, fake, fake, fake, fake, fake, fake, 0,
                             fake, 0, None) == _lib.ERR_INVALID_ARG


# ------------------------------------------------------------------ point-prefill plans
def _check_prefill_plan(cfg, lay, offs, segs, own_len, flags=0):
    """Row (b, i, h) of a prefill plan has exactly one partial, from one reader-stationary item whose
    ranges are b's list except OWN (same order and extents) followed by the causal own range
    [0, Lc) of its run (the kernel limits row i to [0, i]).  Paired (default): item 2u records in
    t1 how many leading ranges it shares with item 2u+1 (same kv head, equal spans), and the plan
    streams those once per pair (ORION_PLAN_PAIR)."""
    lc = cfg.lc
    plan, ws = orion.expand_plan(cfg.hq, cfg.hkv, cfg.d, cfg.page, offs, segs, own_len,
                                 prefill_rows=lc, flags=flags)
    h, items, readers, coff, cslot = parse_plan(plan)
    ranges = np.frombuffer(plan, RANGE, int(h["n_ranges"]), int(h["ranges_off"]))
    G = cfg.hq // cfg.hkv
    R = lc * G
    assert h["n_rows"] == lay.n_branches * lc * cfg.hq and int(h["pad"][2]) == lc
    assert int(h["pad"][0]) == 0                     # rows-on-lanes tcgen05 kernel
    slot = {}
    for it in items:
        assert it["p0"] == 2 and it["n_rows"] <= 128          # kItemRanges
        rg = ranges[it["pt_off"]:it["pt_off"] + it["p1"]]
        b = readers[it["readers_off"]]
        lst = segs[offs[b]:offs[b + 1]]
        want = [(int(sg["pt_off"]), int(sg["start"]), int(sg["start"] + sg["len"]), int(sg["dyn"]), 0)
                for sg in lst[:-1] if sg["len"] > 0]
        own = lst[-1]
        assert own["dyn"] == b
        want.append((int(own["pt_off"]), int(own["start"]), int(own["start"]) + lc, -1, 1))
        assert [tuple(int(x) for x in r)[:5] for r in rg] == want
        for r in range(it["row_begin"], it["row_begin"] + it["n_rows"]):
            assert r < R
            i, hh = r // G, it["kv_head"] * G + r % G
            slot[it["slot0"] + r - it["row_begin"]] = (b * lc + i) * cfg.hq + hh
    assert sorted(slot) == list(range(h["n_partials"]))
    for row in range(h["n_rows"]):
        ss = cslot[coff[row]:coff[row + 1]]
        assert len(ss) == 1 and slot[int(ss[0])] == row
    paired = bool(flags & orion.PLAN_PAIR)
    assert int(h["paired"]) == int(paired)
    lists = [[tuple(int(x) for x in r)[:5] for r in ranges[it["pt_off"]:it["pt_off"] + it["p1"]]]
             for it in items]
    streamed = sum(r[2] - r[1] for lst in lists for r in lst)
    if paired:
        for u in range(0, len(items) - 1, 2):
            a, b = lists[u], lists[u + 1]
            n_sh = 0
            if items[u]["kv_head"] == items[u + 1]["kv_head"]:
                while n_sh < min(len(a), len(b)) and a[n_sh] == b[n_sh]:
                    n_sh += 1
            assert int(items[u]["t1"]) == n_sh
            streamed -= sum(r[2] - r[1] for r in a[:n_sh])
    assert int(h["streamed_tokens"]) == streamed
    return h


@pytest.mark.parametrize("cfgname,policy,hq", [("c1", 0, 4), ("c1", 1, 4), ("c2", 0, 32), ("c3", 1, 28)])
def test_prefill_plan_covers_context_and_causal_own(cfgname, policy, hq):
    cfg = C.CONFIGS[cfgname].with_(n_queries=2, lp=min(C.CONFIGS[cfgname].lp, 256),
                                   t=min(C.CONFIGS[cfgname].t, 96), hq=hq)
    lay = T.make_layout(cfg, ragged=True, extra_tokens=cfg.page)
    offs, segs = _bind_layout(cfg, lay, policy)
    _check_prefill_plan(cfg, lay, offs, segs, lay.own_len)
    _check_prefill_plan(cfg, lay, offs, segs, lay.own_len, flags=orion.PLAN_PAIR)


def test_prefill_pairs_share_the_prefix_closed_form():
    # Edgeless DAG (every list = [PREFIX, OWN]), even point count: every pair is two readers of
    # one query and kv head sharing exactly the prefix, so the paired plan streams
    # Hkv * (sum_b (Lp + Lc) - (n_branches / 2) * Lp) token rows, the unpaired one Hkv * sum_b (Lp + Lc).
    cfg = C.CONFIGS["c1"].with_(n_queries=3, lp=200, t=64, lc=16, page=16, hq=8, hkv=2)
    lay = T.make_layout(cfg, dag_override=lambda: W.wide(6))
    offs, segs = _bind_layout(cfg, lay, 0)
    B = lay.n_branches
    h = _check_prefill_plan(cfg, lay, offs, segs, lay.own_len, flags=orion.PLAN_PAIR)
    assert int(h["streamed_tokens"]) == cfg.hkv * (B * (cfg.lp + cfg.lc) - (B // 2) * cfg.lp)
    h = _check_prefill_plan(cfg, lay, offs, segs, lay.own_len)
    assert int(h["streamed_tokens"]) == cfg.hkv * B * (cfg.lp + cfg.lc)


def test_prefill_plan_errors():
    import ctypes
    cfg = C.CONFIGS["c1"]
    lay = T.make_layout(cfg)
    offs, segs = _bind_layout(cfg, lay, 0)
    with pytest.raises(orion.OrionError) as ei:          # the mma.sync kernel has no causal rows
        orion.expand_plan(cfg.hq, cfg.hkv, cfg.d, cfg.page, offs, segs, lay.own_len,
                          prefill_rows=cfg.lc, flags=orion.PLAN_MMA_SYNC)
    assert ei.value.code == _lib.ERR_UNSUPPORTED
    with pytest.raises(orion.OrionError) as ei:          # OWN shorter than Lc
        orion.expand_plan(cfg.hq, cfg.hkv, cfg.d, cfg.page, offs, segs, lay.own_len,
                          prefill_rows=int(segs["len"].max()) + 1)
    assert ei.value.code == _lib.ERR_INVALID_ARG
    # the two attention entry points refuse the other kind of plan before touching the device
    L = _lib.lib()
    shape = _lib.AttnShape(cfg.hq, cfg.hkv, cfg.d, cfg.page, 0.0)
    pre, _ = orion.expand_plan(cfg.hq, cfg.hkv, cfg.d, cfg.page, offs, segs, lay.own_len,
                               prefill_rows=cfg.lc)
    dec, _ = orion.expand_plan(cfg.hq, cfg.hkv, cfg.d, cfg.page, offs, segs, lay.own_len)
    fake = ctypes.c_void_p(16)
    args = (fake, fake, None, fake, fake, 1, fake, fake)
    assert L.orion_expand_attn(ctypes.byref(shape), lay.n_branches, *args, _lib.ptr(pre), fake, fake,
                               1 << 30, None) == _lib.ERR_INVALID_ARG
    assert L.orion_point_prefill_attn(ctypes.byref(shape), lay.n_branches, *args, _lib.ptr(dec), fake,
                                      fake, 1 << 30, None) == _lib.ERR_INVALID_ARG
    assert b"prefill" in L.orion_last_error()


@pytest.mark.parametrize("hq,hkv", [(128, 1), (256, 2), (96, 1)])
@pytest.mark.parametrize("flags", [0, 16])          # hybrid (default) / ORION_PLAN_NO_HYBRID
def test_plan_splits_rows_of_wide_groups(hq, hkv, flags):
    """G = Hq / Hkv above a kernel's row limit (64 swap-AB, 128 rows-on-lanes): one reader's rows
    alone exceed an item, so the planner must split them into row blocks (never an item with more
    rows than its kernel handles), and every row is still covered exactly once."""
    cfg = C.CONFIGS["c1"].with_(hq=hq, hkv=hkv, d=128, page=16, lp=80, t=48, lc=8, n_queries=2,
                                dag="mixed8")
    lay = T.make_layout(cfg, ragged=True, extra_tokens=16)
    offs, segs = _bind_layout(cfg, lay, 0)
    h = _check_plan_covers(cfg, lay, offs, segs, lay.own_len, flags=flags)
    plan, _ = orion.expand_plan(cfg.hq, cfg.hkv, cfg.d, cfg.page, offs, segs, lay.own_len, flags=flags)
    h, items, *_ = parse_plan(plan)
    nb = int(h["n_big"])
    assert (items["n_rows"][:nb] <= 128).all() and (items["n_rows"][nb:] <= 64).all()
    assert (nb > 0) == (flags == 0 and hq // hkv in (96, 128))


def test_chain_plan_merges_history_per_reader_block():
    # Dependent chain under ANCESTORS: point j reads the full runs of points 1..j-1.  With fixed
    # reader blocks, a block's shared history becomes multi-range items (kItemRanges) -- far fewer
    # partials than one per (ancestor, reader) -- and every context is still covered exactly once.
    cfg = C.CONFIGS["c5c"].with_(n_queries=1, lp=512, t=96, lc=16, dag="chain64")
    lay = T.make_layout(cfg, dag_override=lambda: W.chain(48, 2))
    offs, segs = _bind_layout(cfg, lay, 0)
    # fixed 512-token chunking (an explicit chunk_tokens turns off the small-step split)
    merged, _ = orion.expand_plan(cfg.hq, cfg.hkv, cfg.d, cfg.page, offs, segs, lay.own_len,
                                  flags=orion.PLAN_NO_HYBRID, chunk_tokens=512)
    hybrid, _ = orion.expand_plan(cfg.hq, cfg.hkv, cfg.d, cfg.page, offs, segs, lay.own_len,
                                  chunk_tokens=512)
    plain, _ = orion.expand_plan(cfg.hq, cfg.hkv, cfg.d, cfg.page, offs, segs, lay.own_len,
                                 flags=orion.PLAN_NO_MERGE, chunk_tokens=512)
    hm, im, *_ = parse_plan(merged)
    hh, ih, *_ = parse_plan(hybrid)
    hp, ip, *_ = parse_plan(plain)
    assert (im["p0"] & 2).any() and not (ip["p0"] & 2).any()
    assert hm["n_partials"] * 2 < hp["n_partials"]            # 3x fewer at this size
    assert hh["n_partials"] < hp["n_partials"]                # 128-row blocks: 1.8x fewer
    for h in (hm, hh):
        assert h["unique_tokens"] == hp["unique_tokens"] and h["logical_tokens"] == hp["logical_tokens"]
    # hybrid: the big items (65..128 rows) come first, every other item has <= 64 rows
    nb = int(hh["n_big"])
    assert nb > 0 and (ih["n_rows"][:nb] > 64).all() and (ih["n_rows"][:nb] <= 128).all()
    assert (ih["n_rows"][nb:] <= 64).all() and hm["n_big"] == 0
    _check_plan_covers(cfg, lay, offs, segs, lay.own_len)
    _check_plan_covers(cfg, lay, offs, segs, lay.own_len, flags=orion.PLAN_NO_HYBRID)


@pytest.mark.parametrize("nb", [1, 2, 8])
def test_small_step_spreads_over_the_sms(nb):
    """A latency-bound running set (c2: 1-8 branches of one query) is cut into about two items
    per SM (chunks of >= one 64-token tile) instead of a few 8K-token merged items; an explicit
    chunk_tokens keeps the fixed chunking; coverage holds either way."""
    cfg = C.CONFIGS["c2"]
    lay = T.make_layout(cfg)
    offs, segs = _bind_layout(cfg, lay, 0)
    sel = np.arange(nb, dtype=np.int32)
    so, sg = orion.select_branches(offs, segs, lay.own_len, sel)
    own = np.ascontiguousarray(lay.own_len[sel], np.int32)
    adaptive, _ = orion.expand_plan(cfg.hq, cfg.hkv, cfg.d, cfg.page, so, sg, own, num_sms=148)
    fixed, _ = orion.expand_plan(cfg.hq, cfg.hkv, cfg.d, cfg.page, so, sg, own, num_sms=148, chunk_tokens=512)
    ha, ia, *_ = parse_plan(adaptive)
    hf, if_, *_ = parse_plan(fixed)
    assert ha["unique_tokens"] == hf["unique_tokens"] and ha["logical_tokens"] == hf["logical_tokens"]
    assert hf["n_items"] < 148 <= ha["n_items"] <= 4 * 148
    from types import SimpleNamespace
    _check_plan_covers(cfg, SimpleNamespace(n_branches=nb), so, sg, own, chunk_tokens=0)


def test_step_launches():
    """orion_step_launches: 1 kernel per orion_expand_step on a short step of the swap-AB kernel
    (the append and the combine fused into the split launch), 3 on a long one (c4's 64 queries: the separate
    append overlaps the split's prologue), 4 on a hybrid plan with both split kernels, 1 for a
    point-prefill plan.  Host only (148 SMs without a GPU)."""
    from paper_2510_24390_b200 import _lib

    def launches(plan):
        n = np.zeros(1, np.int32)
        _lib.check(orion.lib().orion_step_launches(_lib.ptr(plan), _lib.ptr(n)))
        return int(n[0])

    def plan_of(cfgname, nq, **kw):
        cfg = C.CONFIGS[cfgname].with_(n_queries=nq)
        lay = T.make_layout(cfg)
        offs, segs = _bind_layout(cfg, lay, 0)
        return orion.expand_plan(cfg.hq, cfg.hkv, cfg.d, cfg.page, offs, segs, lay.own_len, **kw)[0], cfg

    assert launches(plan_of("c4", 2)[0]) == 1
    assert launches(plan_of("c4", 64)[0]) == 3
    hyb, _ = plan_of("c5c", 1)
    assert orion.plan_stats(hyb)["n_big"] > 0 and launches(hyb) == 4
    pre, cfg = plan_of("c2", 1, prefill_rows=C.CONFIGS["c2"].lc)
    assert launches(pre) == 1
    with pytest.raises(orion.OrionError):
        launches(np.zeros(256, np.uint8))
