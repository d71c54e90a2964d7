"""Pins for oracle O5 (point-prefill attention, oracle/prefill.py): each test fixes the result by
something other than O5's own code -- fp64 torch SDPA with an explicit causal mask over the
concatenated sequence, the already-pinned decode oracle O3, and closed forms -- so a dropped
dependency span, an off-by-one in the causal limit or a transposed head mapping fails one."""
import numpy as np
import pytest
import torch

from oracle import dag as D, prefill as PF, step as S
from workloads import dags as W, configs as C, tensors as T
from tests.oracle_helpers import u16, f64, contiguous


def small_cfg(**kw):
    return C.CONFIGS["c1"].with_(lp=80, t=40, lc=8, page=16).with_(**kw)


def q_pre(cfg, lay, seed=5, scale=1.0):
    """[B, Lc, Hq, d] bf16 query rows of the content tokens (synthetic, seeded)."""
    return T.bf16_randn_u16((lay.n_branches, cfg.lc, cfg.hq, cfg.d), seed, "cpu", scale=scale)


def sdpa_prefill(q_rows, k_seq, v_seq, n_ctx):
    """q [Lc, Hq, d]; k/v [n_ctx + Lc, Hkv, d] -> out [Lc, Hq, d]: query i sits at position n_ctx + i
    of the sequence and sees positions <= n_ctx + i (torch SDPA, fp64, boolean mask)."""
    lc, hq, d = q_rows.shape
    hkv = k_seq.shape[1]
    g = hq // hkv
    k = k_seq.permute(1, 0, 2).repeat_interleave(g, dim=0)       # [Hq, n, d]
    v = v_seq.permute(1, 0, 2).repeat_interleave(g, dim=0)
    q = q_rows.permute(1, 0, 2)                                   # [Hq, Lc, d]
    n = k_seq.shape[0]
    mask = torch.arange(n)[None, :] <= (n_ctx + torch.arange(lc))[:, None]   # [Lc, n]
    out = torch.nn.functional.scaled_dot_product_attention(q, k, v, attn_mask=mask)
    return out.permute(1, 0, 2)


@pytest.mark.parametrize("kind", [2, 1])
@pytest.mark.parametrize("page", [16, 32])
def test_chain_prefill_equals_causal_sdpa(kind, page):
    # Dependent chain, ANCESTORS: Pre(j) sees [prefix | S_1 | ... | S_{j-1}] then P_j causally,
    # i.e. an ordinary causal prefill of P_j after the concatenated history (reading S7).
    # Contextual chain: [prefix | P_1 | ... | P_{j-1}] then P_j.
    cfg = small_cfg(page=page, hq=8, hkv=2)
    n = 4
    lay = T.make_layout(cfg, dag_override=lambda: W.chain(n, kind), ragged=True)
    ten = T.make_qkv(cfg, lay)
    qp = q_pre(cfg, lay, scale=3.0)
    out, _ = PF.point_prefill(lay, u16(qp), u16(ten["k_cache"][0]), u16(ten["v_cache"][0]))
    kc, vc = ten["k_cache"][0], ten["v_cache"][0]
    ks = [contiguous(kc, lay.page_table, lay.prefix_pt_off[0], cfg.lp, page)]
    vs = [contiguous(vc, lay.page_table, lay.prefix_pt_off[0], cfg.lp, page)]
    for j in range(n):
        kj = contiguous(kc, lay.page_table, lay.point_pt_off[j], lay.own_len[j], page)
        vj = contiguous(vc, lay.page_table, lay.point_pt_off[j], lay.own_len[j], page)
        lc = cfg.lc
        n_ctx = sum(x.shape[0] for x in ks)
        ref = sdpa_prefill(f64(qp[j]), torch.cat(ks + [kj[:lc]]), torch.cat(vs + [vj[:lc]]), n_ctx)
        assert np.allclose(out[j], ref.numpy(), atol=1e-12, rtol=1e-10)
        ks.append(kj if kind == 2 else kj[:lc])
        vs.append(vj if kind == 2 else vj[:lc])


@pytest.mark.parametrize("dagf", [W.diamond, W.fig4, W.mixed8])
@pytest.mark.parametrize("policy", [D.ANCESTORS, D.PARENTS_EQ3])
def test_last_content_row_equals_decode_at_own_len_lc(dagf, policy):
    # The last content token of P_j sees exactly what a decode query of j sees when own_len_j = Lc
    # (same dependency spans, own tokens [0, Lc)): O5's last row == the pinned decode oracle O3.
    cfg = small_cfg(hq=6, hkv=3)
    lay = T.make_layout(cfg, dag_override=dagf, ragged=True)
    ten = T.make_qkv(cfg, lay)
    qp = q_pre(cfg, lay)
    k, v = u16(ten["k_cache"][0]), u16(ten["v_cache"][0])
    out, lse = PF.point_prefill(lay, u16(qp), k, v, policy=policy)
    for b in range(lay.n_branches):
        own = lay.own_len.copy()
        own[b] = cfg.lc
        ref, ref_lse = S.expand_step(lay, u16(qp[:, cfg.lc - 1]), k, v, policy=policy, branches=[b],
                                     own_len=own)
        assert np.allclose(out[b, cfg.lc - 1], ref[0], atol=1e-12, rtol=1e-10)
        assert np.allclose(lse[b, cfg.lc - 1], ref_lse[0], atol=1e-12)


def test_empty_context_first_row_is_own_v_row():
    # No prefix, no dependencies: content token 0 attends to itself only -> exactly V of token 0,
    # lse = scale * q.k_0.
    cfg = small_cfg(lp=0, hq=4, hkv=2)
    lay = T.make_layout(cfg, dag_override=lambda: W.wide(3))
    ten = T.make_qkv(cfg, lay)
    qp = q_pre(cfg, lay)
    out, lse = PF.point_prefill(lay, u16(qp), u16(ten["k_cache"][0]), u16(ten["v_cache"][0]))
    kc, vc = f64(ten["k_cache"][0]), f64(ten["v_cache"][0])
    for b in range(lay.n_branches):
        pg = int(lay.page_table[lay.point_pt_off[b]])
        for h in range(cfg.hq):
            g = h // (cfg.hq // cfg.hkv)
            assert np.array_equal(out[b, 0, h], vc[pg, g, 0].numpy())
            want = float(torch.dot(f64(qp[b, 0, h]), kc[pg, g, 0])) / np.sqrt(cfg.d)
            assert abs(lse[b, 0, h] - want) < 1e-12


def test_constant_keys_give_running_mean_of_values():
    # Identical keys: row i's weights are uniform over (context + i + 1) tokens.
    cfg = small_cfg(hq=4, hkv=2)
    lay = T.make_layout(cfg, dag_override=W.fig4)
    ten = T.make_qkv(cfg, lay)
    kc = ten["k_cache"][0].clone()
    kc[:] = kc[0, 0, 0]
    qp = q_pre(cfg, lay)
    out, _ = PF.point_prefill(lay, u16(qp), u16(kc), u16(ten["v_cache"][0]))
    vc = ten["v_cache"][0]
    lists = D.segment_lists(*W.fig4())
    for b in range(lay.n_branches):
        rows = []
        for kind, pnt in lists[b + 1][:-1]:
            if kind == D.SEG_PREFIX:
                rows.append(contiguous(vc, lay.page_table, lay.prefix_pt_off[0], cfg.lp, cfg.page))
            else:
                full = contiguous(vc, lay.page_table, lay.point_pt_off[pnt - 1], lay.own_len[pnt - 1], cfg.page)
                rows.append(full[:lay.content_len[pnt - 1]] if kind == D.SEG_CONTENT else full)
        own = contiguous(vc, lay.page_table, lay.point_pt_off[b], cfg.lc, cfg.page)
        for i in range(cfg.lc):
            mean = torch.cat(rows + [own[:i + 1]], 0).mean(0)
            for h in range(cfg.hq):
                assert np.allclose(out[b, i, h], mean[h // 2].numpy(), atol=1e-12, rtol=0)
