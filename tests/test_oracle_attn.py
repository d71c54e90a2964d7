"""Pins for oracle O2/O3/O3'/O4: closed forms, fp64 SDPA library
equivalences, a second independent (masked-pool) formulation, invariances."""
import random

import numpy as np
import pytest
import torch

from oracle import attention as A, dag as D, step as S, append as AP, bind as BD
from workloads import dags as W, configs as C, tensors as T
from tests.oracle_helpers import u16, f64, contiguous, sdpa_decode


def small_cfg(**kw):
    base = C.CONFIGS["c1"].with_(lp=80, t=40, lc=8, page=16)
    return base.with_(**kw)


def test_bf16_widening_exact():
    x = T.bf16_randn_u16((4096,), 3)
    assert np.array_equal(A.bf16_to_f64(u16(x)), f64(x).numpy())


def test_single_token_context_is_v_row():
    cfg = small_cfg()
    lay = T.make_layout(cfg, dag_override=lambda: W.wide(2))
    ten = T.make_qkv(cfg, lay)
    k, v, q = u16(ten["k_cache"][0]), u16(ten["v_cache"][0]), u16(ten["q"][0])
    pages = lay.pages_of(lay.point_pt_off[0], lay.point_cap[0])
    bound = [[(pages, 5, 1)], [(pages, 0, 1)]]
    out, lse = A.expand_attn(q, k, v, bound, cfg.page)
    kf, vf, qf = f64(ten["k_cache"][0]), f64(ten["v_cache"][0]), f64(ten["q"][0])
    for b, pos in ((0, 5), (1, 0)):
        for h in range(cfg.hq):
            g = h // cfg.g
            assert np.array_equal(out[b, h], vf[pages[0], g, pos].numpy())
            want = float(torch.dot(qf[b, h], kf[pages[0], g, pos])) / np.sqrt(cfg.d)
            assert abs(lse[b, h] - want) < 1e-12


def test_constant_k_gives_mean_v_and_constant_v_gives_v():
    cfg = small_cfg()
    lay = T.make_layout(cfg)
    ten = T.make_qkv(cfg, lay)
    kc = ten["k_cache"][0].clone()
    kc[:] = kc[0, 0, 0]                       # every key row identical
    out, _ = S.expand_step(lay, u16(ten["q"][0]), u16(kc), u16(ten["v_cache"][0]))
    vc = ten["v_cache"][0]
    for b in range(lay.n_branches):
        qi = lay.branch_query[b]
        # diamond ANCESTORS lists: rebuild each context as contiguous runs and average V
        lists = D.segment_lists(*W.diamond())[b + 1]
        rows = []
        for kind, pnt in lists:
            if kind == D.SEG_PREFIX:
                rows.append(contiguous(vc, lay.page_table, lay.prefix_pt_off[qi], cfg.lp, cfg.page))
            else:
                bb = lay.branch0[qi] + pnt - 1
                full = contiguous(vc, lay.page_table, lay.point_pt_off[bb], lay.own_len[bb], cfg.page)
                rows.append(full[:lay.content_len[bb]] if kind == D.SEG_CONTENT else full)
        mean = torch.cat(rows, 0).mean(0)     # [Hkv, d]
        for h in range(cfg.hq):
            assert np.allclose(out[b, h], mean[h // cfg.g].numpy(), atol=1e-12, rtol=0)
    vconst = ten["v_cache"][0].clone()
    vconst[:] = vconst[3, 1, 2]
    out, _ = S.expand_step(lay, u16(ten["q"][0]), u16(ten["k_cache"][0]), u16(vconst))
    assert np.allclose(out, f64(vconst[0, 0, 0]).numpy()[None, None, :], atol=1e-12, rtol=0)


@pytest.mark.parametrize("page", [16, 32, 64])
@pytest.mark.parametrize("kind", [2, 1])
def test_chain_equals_causal_decode_sdpa(page, kind):
    # Dependent chain under ANCESTORS == ordinary causal decode over [prefix | S_1 | ... | S_n]
    # (north_star; reading S6/S7).  Contextual chain == decode over [prefix | P_1..P_{j-1} | S_j].
    cfg = small_cfg(page=page, hq=8, hkv=2)
    n = 5
    lay = T.make_layout(cfg, dag_override=lambda: W.chain(n, kind), ragged=True)
    ten = T.make_qkv(cfg, lay, q_scale=4.0)
    out, lse = S.expand_step(lay, u16(ten["q"][0]), u16(ten["k_cache"][0]), u16(ten["v_cache"][0]))
    kc, vc, q = ten["k_cache"][0], ten["v_cache"][0], f64(ten["q"][0])
    kp = contiguous(kc, lay.page_table, lay.prefix_pt_off[0], cfg.lp, page)
    vp = contiguous(vc, lay.page_table, lay.prefix_pt_off[0], cfg.lp, page)
    ks, vs = [kp], [vp]
    for j in range(n):
        kj = contiguous(kc, lay.page_table, lay.point_pt_off[j], lay.own_len[j], page)
        vj = contiguous(vc, lay.page_table, lay.point_pt_off[j], lay.own_len[j], page)
        ref = sdpa_decode(q[j], torch.cat(ks + [kj]), torch.cat(vs + [vj]))
        assert np.allclose(out[j], ref.numpy(), atol=1e-12, rtol=1e-10)
        lc = lay.content_len[j]
        ks.append(kj if kind == 2 else kj[:lc])
        vs.append(vj if kind == 2 else vj[:lc])


def test_eq3_chain_uses_output_span_only():
    cfg = small_cfg(hq=4, hkv=4)
    n = 4
    lay = T.make_layout(cfg, dag_override=lambda: W.chain(n, 2), ragged=True)
    ten = T.make_qkv(cfg, lay)
    out, _ = S.expand_step(lay, u16(ten["q"][0]), u16(ten["k_cache"][0]), u16(ten["v_cache"][0]),
                           policy=D.PARENTS_EQ3)
    kc, vc, q = ten["k_cache"][0], ten["v_cache"][0], f64(ten["q"][0])
    kp = contiguous(kc, lay.page_table, lay.prefix_pt_off[0], cfg.lp, cfg.page)
    vp = contiguous(vc, lay.page_table, lay.prefix_pt_off[0], cfg.lp, cfg.page)
    for j in range(n):
        kj = contiguous(kc, lay.page_table, lay.point_pt_off[j], lay.own_len[j], cfg.page)
        vj = contiguous(vc, lay.page_table, lay.point_pt_off[j], lay.own_len[j], cfg.page)
        kk, vv = [kp], [vp]
        if j > 0:
            kpar = contiguous(kc, lay.page_table, lay.point_pt_off[j - 1], lay.own_len[j - 1], cfg.page)
            vpar = contiguous(vc, lay.page_table, lay.point_pt_off[j - 1], lay.own_len[j - 1], cfg.page)
            lc = lay.content_len[j - 1]
            kk.append(kpar[lc:])
            vv.append(vpar[lc:])
        ref = sdpa_decode(q[j], torch.cat(kk + [kj]), torch.cat(vv + [vj]))
        assert np.allclose(out[j], ref.numpy(), atol=1e-12, rtol=1e-10)


def test_wide_equals_prefix_plus_own():
    cfg = small_cfg(hq=6, hkv=2)
    lay = T.make_layout(cfg, dag_override=lambda: W.wide(3))
    ten = T.make_qkv(cfg, lay, sink=True)
    out, lse = S.expand_step(lay, u16(ten["q"][0]), u16(ten["k_cache"][0]), u16(ten["v_cache"][0]))
    kc, vc, q = ten["k_cache"][0], ten["v_cache"][0], f64(ten["q"][0])
    for j in range(3):
        ks = torch.cat([contiguous(kc, lay.page_table, lay.prefix_pt_off[0], cfg.lp, cfg.page),
                        contiguous(kc, lay.page_table, lay.point_pt_off[j], lay.own_len[j], cfg.page)])
        vs = torch.cat([contiguous(vc, lay.page_table, lay.prefix_pt_off[0], cfg.lp, cfg.page),
                        contiguous(vc, lay.page_table, lay.point_pt_off[j], lay.own_len[j], cfg.page)])
        ref = sdpa_decode(q[j], ks, vs)
        assert np.allclose(out[j], ref.numpy(), atol=1e-12, rtol=1e-10)
        # lse closed form: log-sum-exp of the scores, through torch.logsumexp
        kr = ks.permute(1, 0, 2).repeat_interleave(cfg.g, 0)
        s = torch.einsum("hd,hnd->hn", q[j], kr) / np.sqrt(cfg.d)
        assert np.allclose(lse[j], torch.logsumexp(s, -1).numpy(), atol=1e-12)


def _masked_pool(lay, cfg, qi, policy):
    """Pool = every token of the query in storage order; mask from span membership."""
    n = int(lay.n_points[qi]); b0 = int(lay.branch0[qi])
    pool, where = [], {}
    prefix_pages = lay.pages_of(lay.prefix_pt_off[qi], lay.prefix_len[qi])
    for t in range(lay.prefix_len[qi]):
        where[("P", t)] = len(pool); pool.append((prefix_pages[t // cfg.page], t % cfg.page))
    for k in range(1, n + 1):
        b = b0 + k - 1
        pages = lay.pages_of(lay.point_pt_off[b], lay.point_cap[b])
        for t in range(lay.own_len[b]):
            where[(k, t)] = len(pool); pool.append((pages[t // cfg.page], t % cfg.page))
    lists = D.segment_lists(n, lay.edges[qi], policy)
    mask = np.zeros((n, len(pool)), dtype=bool)
    for j in range(1, n + 1):
        for kind, k in lists[j]:
            if kind == D.SEG_PREFIX:
                span = [("P", t) for t in range(lay.prefix_len[qi])]
            else:
                bk = b0 + k - 1
                lo = lay.content_len[bk] if kind == D.SEG_OUTPUT else 0
                hi = lay.content_len[bk] if kind == D.SEG_CONTENT else lay.own_len[bk]
                span = [(k, t) for t in range(lo, hi)]
            for key in span:
                assert not mask[j - 1, where[key]]
                mask[j - 1, where[key]] = True
    return pool, mask


@pytest.mark.parametrize("policy", [D.ANCESTORS, D.PARENTS_EQ3])
def test_masked_pool_second_oracle(policy):
    rng = random.Random(21)
    for trial in range(6):
        n = rng.randint(1, 6)
        dagf = (lambda nn=n, s=trial: W.random_dag(random.Random(100 + s), nn, p=0.5))
        cfg = small_cfg(hq=4, hkv=2, page=16, seed=300 + trial)
        lay = T.make_layout(cfg, dag_override=dagf, ragged=True)
        ten = T.make_qkv(cfg, lay, q_scale=2.0)
        q, k, v = u16(ten["q"][0]), u16(ten["k_cache"][0]), u16(ten["v_cache"][0])
        out, lse = S.expand_step(lay, q, k, v, policy=policy)
        pool, mask = _masked_pool(lay, cfg, 0, policy)
        out2, lse2 = A.masked_pool_attn(q, k, v, pool, mask, cfg.page)
        assert np.allclose(out, out2, rtol=1e-12, atol=1e-13)
        assert np.allclose(lse, lse2, rtol=1e-12, atol=1e-13)


def test_page_permutation_invariance():
    cfg = small_cfg()
    lay = T.make_layout(cfg, contiguous=True)
    ten = T.make_qkv(cfg, lay)
    q, k, v = u16(ten["q"][0]), u16(ten["k_cache"][0]), u16(ten["v_cache"][0])
    out, lse = S.expand_step(lay, q, k, v)
    perm = np.random.default_rng(7).permutation(lay.num_pages)
    k2 = np.empty_like(k); v2 = np.empty_like(v)
    k2[perm] = k; v2[perm] = v                       # physical page p moves to perm[p]
    lay.page_table = perm[lay.page_table].astype(np.int32)
    out2, lse2 = S.expand_step(lay, q, k2, v2)
    assert np.array_equal(out, out2) and np.array_equal(lse, lse2)


def test_append_matches_contiguous_view():
    cfg = small_cfg()
    lay = T.make_layout(cfg, ragged=True, extra_tokens=cfg.page)
    ten = T.make_qkv(cfg, lay)
    kc = ten["k_cache"][0]
    new = ten["k_new"][0]
    cache2, own2 = AP.kv_append(u16(kc), u16(new), lay.page_table, lay.point_pt_off, lay.own_len, cfg.page)
    assert np.array_equal(own2, lay.own_len + 1)
    c2 = torch.from_numpy(cache2.view(np.int16)).view(torch.bfloat16)
    for b in range(lay.n_branches):
        seg = contiguous(c2, lay.page_table, lay.point_pt_off[b], own2[b], cfg.page)
        assert torch.equal(seg[lay.own_len[b]], f64(new[b]))
        old = contiguous(kc, lay.page_table, lay.point_pt_off[b], lay.own_len[b], cfg.page)
        assert torch.equal(seg[:lay.own_len[b]], old)
    diff = (u16(kc) != cache2).any(axis=-1)          # [pages, Hkv, P]
    assert diff.sum() <= lay.n_branches * cfg.hkv    # only the written slots can differ
    # rewrite mode overwrites the last token and keeps lengths
    cache3, own3 = AP.kv_append(u16(kc), u16(new), lay.page_table, lay.point_pt_off, lay.own_len,
                                cfg.page, rewrite=True)
    assert np.array_equal(own3, lay.own_len)
    c3 = torch.from_numpy(cache3.view(np.int16)).view(torch.bfloat16)
    for b in range(lay.n_branches):
        seg = contiguous(c3, lay.page_table, lay.point_pt_off[b], lay.own_len[b], cfg.page)
        assert torch.equal(seg[lay.own_len[b] - 1], f64(new[b]))


def test_bind_closed_forms():
    lists = {1: [(0, 0), (1, 2), (2, 3), (3, 4), (4, 1)]}
    pp = {1: [9], 2: [5], 3: [6, 7], 4: [8]}
    out = BD.bind_segments(lists, [1, 2], 100, pp, {1: 4, 2: 3, 3: 5, 4: 2}, {1: 10, 2: 11, 3: 12, 4: 13})
    assert out[1] == [([1, 2], 0, 100), ([5], 0, 3), ([6, 7], 0, 12), ([8], 2, 11), ([9], 0, 10)]
