"""GPU parity of the point-prefill attention (orion_point_prefill_attn)
against the fp64 oracle O5 on the same seeded bytes.  Gates as for decode (north_star):
out max-abs <= 2e-2 and rel-L2 <= 5e-3; lse abs <= 5e-3."""
import numpy as np
import pytest
import torch

import paper_2510_24390_b200 as orion
from oracle import prefill as OP
from workloads import configs as C, tensors as T, dags as W
from tests.gpu_helpers import MAX_ABS, REL_L2, LSE_ABS, u16

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run_prefill(cfg, lay, ten, qp, policy=0, interleaved=False, flags=0):
    dev = torch.device("cuda")
    queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i],
                    prefix_pt_off=int(lay.prefix_pt_off[i]), prefix_len=int(lay.prefix_len[i]))
               for i in range(lay.n_queries)]
    points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
    batch = orion.ExpansionBatch(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, lay.page_table,
                                 lay.own_len, policy=policy, device=dev, prefill_rows=cfg.lc,
                                 kv_interleaved=interleaved, flags=flags)
    if interleaved:
        kv = torch.stack([ten["k_cache"][0], ten["v_cache"][0]], dim=2).to(dev).contiguous()
        kc, vc = kv[:, :, 0], kv[:, :, 1]
    else:
        kc = ten["k_cache"][0].to(dev).contiguous()
        vc = ten["v_cache"][0].to(dev).contiguous()
    q = qp.to(dev).contiguous()
    out = torch.empty_like(q)
    lse = torch.empty(q.shape[:3], dtype=torch.float32, device=dev)
    batch.attend(q, out, kc, vc, lse)
    torch.cuda.synchronize()
    return out, lse, batch


def check(cfg, lay, ten, qp, policy=0, branches=None, interleaved=False, flags=0):
    out, lse, batch = run_prefill(cfg, lay, ten, qp, policy, interleaved, flags)
    if branches is None:
        branches = list(range(lay.n_branches))
    if len(branches) > 32:            # larger configs: the same oracle, in worker processes
        from tests.oracle_pool import point_prefill_parallel
        ref, ref_lse = point_prefill_parallel(lay, u16(qp), u16(ten["k_cache"][0]),
                                              u16(ten["v_cache"][0]), policy=policy, branches=branches)
    else:
        ref, ref_lse = OP.point_prefill(lay, u16(qp), u16(ten["k_cache"][0]), u16(ten["v_cache"][0]),
                                        policy=policy, branches=branches)
    o = out[branches].float().cpu().numpy().astype(np.float64)
    assert np.isfinite(o).all()
    diff = o - ref
    max_abs = float(np.abs(diff).max())
    rel = float(np.linalg.norm(diff) / np.linalg.norm(ref))
    lse_err = float(np.abs(lse[branches].cpu().numpy() - ref_lse).max())
    assert max_abs <= MAX_ABS, (max_abs, rel, lse_err)
    assert rel <= REL_L2, (max_abs, rel, lse_err)
    assert lse_err <= LSE_ABS, (max_abs, rel, lse_err)
    return batch


def q_pre(cfg, lay, seed=5, scale=1.0):
    return T.bf16_randn_u16((lay.n_branches, cfg.lc, cfg.hq, cfg.d), seed, "cpu", scale=scale)


PAIRING = [0, orion.PLAN_PAIR]   # one item per pass (default) / paired items sharing K/V tiles (split_pair.cu)


@pytest.mark.parametrize("flags", PAIRING)
@pytest.mark.parametrize("dagf", [W.diamond, W.fig4, W.mixed8, lambda: W.chain(5, 2)])
@pytest.mark.parametrize("policy", [0, 1])
@pytest.mark.parametrize("d", [64, 128])
def test_small_dags(dagf, policy, d, flags):
    cfg = C.CONFIGS["c1"].with_(lp=150, t=90, lc=8, page=16, d=d, hq=8, hkv=2)
    lay = T.make_layout(cfg, ragged=True, dag_override=dagf)
    ten = T.make_qkv(cfg, lay)
    check(cfg, lay, ten, q_pre(cfg, lay), policy, flags=flags)


@pytest.mark.parametrize("flags", PAIRING)
@pytest.mark.parametrize("lc,hq,hkv", [(32, 8, 2), (32, 32, 8), (16, 28, 4), (64, 8, 4), (40, 8, 2)])
def test_row_blocks_and_causal_spans(lc, hq, hkv, flags):
    # R = Lc*G rows per reader: 64 / 128 / 112 / 128 / 160 (> one 128-row MMA tile: two row blocks
    # and a causal limit crossing the block boundary -- paired, the two blocks of one reader share
    # every range, the causal own range included); Lc up to a whole 64-token tile
    cfg = C.CONFIGS["c1"].with_(lp=300, t=200, lc=lc, page=32, d=128, hq=hq, hkv=hkv)
    lay = T.make_layout(cfg, ragged=True, dag_override=W.mixed8)
    ten = T.make_qkv(cfg, lay, q_scale=2.0)
    check(cfg, lay, ten, q_pre(cfg, lay, scale=3.0), flags=flags)


@pytest.mark.parametrize("dagf,hq,hkv", [(lambda: W.chain(5, 2), 4, 1), (W.fig4, 8, 2), (lambda: W.wide(7), 8, 4)])
def test_pairs_odd_and_across_kv_heads(dagf, hq, hkv):
    # An odd item count (the last pair unit has no second item), pairs straddling two kv heads (no
    # shared range: every tile unique, alternating), pairs of different queries' readers.
    cfg = C.CONFIGS["c1"].with_(n_queries=3, lp=130, t=100, lc=16, page=16, d=128, hq=hq, hkv=hkv)
    lay = T.make_layout(cfg, ragged=True, dag_override=dagf)
    ten = T.make_qkv(cfg, lay, q_scale=2.0)
    batch = check(cfg, lay, ten, q_pre(cfg, lay, scale=2.0), flags=orion.PLAN_PAIR)
    assert batch.stats["paired"] == 1


def test_paired_equals_unpaired_within_rounding():
    # Both kernels compute the same rows from the same plan geometry; they differ only in the
    # order of fp32 accumulation (one O per row vs two alternating-tile accumulators merged).
    cfg = C.CONFIGS["c1"].with_(lp=400, t=160, lc=32, page=64, d=128, hq=8, hkv=2)
    lay = T.make_layout(cfg, ragged=True, dag_override=W.mixed8)
    ten = T.make_qkv(cfg, lay)
    qp = q_pre(cfg, lay, scale=2.0)
    o1, l1, b1 = run_prefill(cfg, lay, ten, qp, flags=orion.PLAN_PAIR)
    o2, l2, b2 = run_prefill(cfg, lay, ten, qp)
    assert b1.stats["paired"] == 1 and b2.stats["paired"] == 0
    assert b1.stats["streamed_tokens"] < b2.stats["streamed_tokens"]
    assert float((o1.float() - o2.float()).abs().max()) <= 1e-2
    assert float((l1 - l2).abs().max()) <= LSE_ABS   # P rounded to bf16 against different running maxima


def test_sink_and_peaky_queries():
    cfg = C.CONFIGS["c1"].with_(lp=500, t=120, lc=24, page=64, d=128, hq=8, hkv=2)
    lay = T.make_layout(cfg, ragged=True, dag_override=W.diamond)
    ten = T.make_qkv(cfg, lay, sink=True)
    check(cfg, lay, ten, q_pre(cfg, lay, scale=4.0))


def test_c2_full():
    cfg = C.CONFIGS["c2"]
    lay = T.make_layout(cfg, ragged=True)
    ten = T.make_qkv(cfg, lay)
    check(cfg, lay, ten, q_pre(cfg, lay))


def test_c4_eight_queries_every_point():
    """c4's shapes (mixed16, 4K prefix, 512 tok/point, 32/8 heads) on an 8-query batch: every point,
    content row and head against O5 (128 points x 32 rows x 32 heads)."""
    cfg = C.CONFIGS["c4"].with_(n_queries=8)
    lay = T.make_layout(cfg)
    ten = T.make_qkv(cfg, lay)
    check(cfg, lay, ten, q_pre(cfg, lay))


def test_prefill_last_row_matches_decode_kernel():
    # The method's identity (pin of O5) through both CUDA paths: with every point at own_len = Lc,
    # the last content row of the prefill and a decode step of q = that row read the same context.
    from oracle import step as OS
    from tests.gpu_helpers import batch_for
    cfg = C.CONFIGS["c1"].with_(lp=200, t=96, lc=32, page=32, d=128, hq=8, hkv=2)
    lay = T.make_layout(cfg, dag_override=W.mixed8)
    lay.own_len[:] = cfg.lc
    ten = T.make_qkv(cfg, lay)
    qp = q_pre(cfg, lay)
    pre, _, _ = run_prefill(cfg, lay, ten, qp)
    dev = torch.device("cuda")
    q = qp[:, cfg.lc - 1].contiguous()
    out = torch.empty(q.shape, dtype=q.dtype, device=dev)
    batch_for(cfg, lay).attend(q.to(dev), out, ten["k_cache"][0].to(dev), ten["v_cache"][0].to(dev))
    torch.cuda.synchronize()
    ref, _ = OS.expand_step(lay, u16(q), u16(ten["k_cache"][0]), u16(ten["v_cache"][0]))
    assert float(np.abs(out.float().cpu().numpy() - ref).max()) <= MAX_ABS
    assert float(np.abs(pre[:, cfg.lc - 1].float().cpu().numpy() - ref).max()) <= MAX_ABS


@pytest.mark.parametrize("flags", PAIRING)
def test_split_plus_combine_equals_direct_prefill(flags):
    # orion_expand_split + orion_expand_combine on a prefill plan (fp32 partials, one per row)
    # reproduce orion_point_prefill_attn's direct-output epilogue bit for bit.
    cfg = C.CONFIGS["c1"].with_(lp=300, t=120, lc=32, page=32, d=128, hq=8, hkv=2)
    lay = T.make_layout(cfg, ragged=True, dag_override=W.mixed8)
    ten = T.make_qkv(cfg, lay)
    qp = q_pre(cfg, lay, scale=2.0)
    out, lse, batch = run_prefill(cfg, lay, ten, qp, flags=flags)
    dev = torch.device("cuda")
    kc = ten["k_cache"][0].to(dev).contiguous()
    vc = ten["v_cache"][0].to(dev).contiguous()
    out2 = torch.empty_like(out)
    lse2 = torch.empty_like(lse)
    batch.split(qp.to(dev).contiguous(), kc, vc)
    batch.combine(out2, lse2)
    torch.cuda.synchronize()
    assert torch.equal(out, out2) and torch.equal(lse, lse2)


def test_prefill_interleaved_kv_layout():
    cfg = C.CONFIGS["c1"].with_(lp=300, t=120, lc=32, page=32, d=128, hq=8, hkv=2)
    lay = T.make_layout(cfg, ragged=True, dag_override=W.mixed8)
    ten = T.make_qkv(cfg, lay)
    check(cfg, lay, ten, q_pre(cfg, lay, scale=2.0), interleaved=True)


@pytest.mark.parametrize("flags", PAIRING)
def test_prefill_grid_size_does_not_change_results(flags):
    # Atomic item (or pair-unit) hand-out: a 3-CTA grid and the full grid give the same bytes.
    cfg = C.CONFIGS["c1"].with_(n_queries=2, lp=300, t=120, lc=32, page=32, d=128, hq=8, hkv=2)
    lay = T.make_layout(cfg, ragged=True, dag_override=W.mixed8)
    ten = T.make_qkv(cfg, lay)
    qp = q_pre(cfg, lay, scale=2.0)
    dev = torch.device("cuda")
    res = []
    for num_sms in (0, 3):
        queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i],
                        prefix_pt_off=int(lay.prefix_pt_off[i]), prefix_len=int(lay.prefix_len[i]))
                   for i in range(lay.n_queries)]
        points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
        batch = orion.ExpansionBatch(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, lay.page_table,
                                     lay.own_len, device=dev, prefill_rows=cfg.lc, flags=flags,
                                     num_sms=num_sms)
        q = qp.to(dev).contiguous()
        out = torch.empty_like(q)
        lse = torch.empty(q.shape[:3], dtype=torch.float32, device=dev)
        batch.attend(q, out, ten["k_cache"][0].to(dev).contiguous(), ten["v_cache"][0].to(dev).contiguous(), lse)
        torch.cuda.synchronize()
        res.append((out.cpu(), lse.cpu()))
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])
