"""T2 — GPU parity of the CUDA path (C ABI) against the fp64 oracle on the same seeded bytes.
Gates (north_star): append bit-exact; out max-abs <= 2e-2 and rel-L2 <= 5e-3; lse abs <= 5e-3."""
import random

import numpy as np
import pytest
import torch

import paper_2510_24390_b200 as orion
from workloads import configs as C, tensors as T, dags as W
from tests.gpu_helpers import check_parity, run_step, u16, batch_for

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


KERNELS = [0, orion.PLAN_MMA_SYNC]     # tcgen05 (default) and the legacy mma.sync split kernel


@pytest.mark.parametrize("flags", KERNELS)
@pytest.mark.parametrize("policy", [0, 1])
@pytest.mark.parametrize("variant", ["plain", "peaky", "sink", "contiguous", "ragged"])
def test_c1_diamond(policy, variant, flags):
    cfg = C.CONFIGS["c1"]
    lay = T.make_layout(cfg, contiguous=variant == "contiguous", ragged=variant == "ragged",
                        extra_tokens=cfg.page)
    ten = T.make_qkv(cfg, lay, q_scale=4.0 if variant == "peaky" else 1.0, sink=variant == "sink")
    check_parity(cfg, lay, ten, policy, flags=flags)


@pytest.mark.parametrize("flags", KERNELS)
@pytest.mark.parametrize("page", [16, 32, 64])
@pytest.mark.parametrize("hq,hkv,d", [(4, 2, 64), (8, 8, 128), (28, 4, 128), (32, 4, 64)])
def test_shapes_pages_ragged(page, hq, hkv, d, flags):
    cfg = C.CONFIGS["c1"].with_(hq=hq, hkv=hkv, d=d, page=page, lp=300, t=150, lc=20, n_queries=2,
                                dag="mixed8")
    lay = T.make_layout(cfg, ragged=True, extra_tokens=page)
    ten = T.make_qkv(cfg, lay, q_scale=2.0)
    check_parity(cfg, lay, ten, 0, chunk_tokens=128, flags=flags)


@pytest.mark.parametrize("flags", KERNELS)
def test_c2_full_layer(flags):
    cfg = C.CONFIGS["c2"]
    lay = T.make_layout(cfg, extra_tokens=cfg.page)
    ten = T.make_qkv(cfg, lay)
    check_parity(cfg, lay, ten, 0, flags=flags)


@pytest.mark.parametrize("policy", [0, 1])
def test_c3_full_layer(policy):
    cfg = C.CONFIGS["c3"]
    lay = T.make_layout(cfg, extra_tokens=cfg.page)
    ten = T.make_qkv(cfg, lay, q_scale=2.0)
    check_parity(cfg, lay, ten, policy)


def _sample(lay, k, seed):
    rng = random.Random(seed)
    return sorted(rng.sample(range(lay.n_branches), k))


def _full_size(name, n_queries=None, **kw):
    cfg = C.CONFIGS[name]
    if n_queries:
        cfg = cfg.with_(n_queries=n_queries)
    lay = T.make_layout(cfg, extra_tokens=cfg.page)
    ten = T.make_qkv(cfg, lay, device="cuda", **kw)       # generated on the GPU (fast), same bytes
    return cfg, lay, {k: v.cpu() for k, v in ten.items()}


@pytest.mark.parametrize("policy", [0, 1])
def test_c4_full_size_every_branch(policy):
    """The bench workload at full size (64 queries x mixed16, 4K prefix, 512 tok/point, 1024
    branches x 32 heads), in the bench's launch configuration (default kernel and plan): every
    branch and head element-wise against the oracle (north_star: "matches the CPU oracle on all 5
    configs")."""
    cfg, lay, ten = _full_size("c4")
    r = check_parity(cfg, lay, ten, policy)
    print(f"c4 policy {policy}: max_abs {r['max_abs']:.2e} rel_l2 {r['rel_l2']:.2e} "
          f"worst branch {r['worst_branch_rel']:.2e} lse {r['lse_err']:.2e}")


@pytest.mark.parametrize("variant", ["peaky", "sink"])
def test_c4_full_size_peaky_and_sink(variant):
    """S18: at c4's context lengths N(0,1) data gives outputs of ~1/sqrt(n_eff), so the absolute
    gate says little; q x 4 (peaky softmax) and an attention sink (prefix token 0's K x 8) make the
    outputs O(0.1-1) and exercise the running-max rescaling."""
    cfg, lay, ten = _full_size("c4", q_scale=4.0 if variant == "peaky" else 1.0, sink=variant == "sink")
    check_parity(cfg, lay, ten, 0)


def test_c4_full_size_mma_sync_sampled():
    cfg, lay, ten = _full_size("c4")
    check_parity(cfg, lay, ten, 0, branches=_sample(lay, 24, 4) + [lay.n_branches - 1],
                 flags=orion.PLAN_MMA_SYNC)


@pytest.mark.parametrize("flags", [0, orion.PLAN_NO_HYBRID])
@pytest.mark.parametrize("policy", [0, 1])
@pytest.mark.parametrize("name", ["c5w", "c5c"])
def test_c5_per_gpu_share_every_branch(name, policy, flags):
    """c5 (BASELINE configs[4]) at one GPU's share of the 8-GPU run (8 queries x wide-64 / chain-64,
    8K prefix, 512 branches): every branch and head; the default hybrid plan (>64-row items on the
    rows-on-lanes kernel) and the swap-AB-only plan."""
    cfg, lay, ten = _full_size(name, n_queries=8, q_scale=2.0)
    r = check_parity(cfg, lay, ten, policy, flags=flags)
    print(f"{name} policy {policy}: max_abs {r['max_abs']:.2e} rel_l2 {r['rel_l2']:.2e} "
          f"worst branch {r['worst_branch_rel']:.2e}")


@pytest.mark.parametrize("name", ["c5w", "c5c"])
def test_c5_per_gpu_share_mma_sync_sampled(name):
    cfg, lay, ten = _full_size(name, n_queries=8, q_scale=2.0)
    check_parity(cfg, lay, ten, 0, branches=_sample(lay, 12, 5) + [63, lay.n_branches - 1],
                 flags=orion.PLAN_MMA_SYNC)


@pytest.mark.parametrize("flags", [0, orion.PLAN_NO_HYBRID])
@pytest.mark.parametrize("hq,hkv", [(128, 1), (96, 1), (64, 2)])
def test_wide_head_groups(hq, hkv, flags):
    """G = Hq / Hkv at or above the kernels' row limits: one reader's rows are split into
    row blocks (or form one 128-row item on the rows-on-lanes kernel) -- every row written."""
    cfg = C.CONFIGS["c1"].with_(hq=hq, hkv=hkv, d=128, page=32, lp=260, t=90, lc=16, n_queries=2,
                                dag="mixed8")
    lay = T.make_layout(cfg, ragged=True, extra_tokens=32)
    ten = T.make_qkv(cfg, lay, q_scale=2.0)
    check_parity(cfg, lay, ten, 0, chunk_tokens=128, flags=flags)


@pytest.mark.parametrize("policy", [0, 1])
def test_hybrid_c3_and_chain(policy):
    """Hybrid plans (both kernels in one step) on c3 and a Dependent chain of 40 points."""
    cfg = C.CONFIGS["c3"].with_(lp=1000)
    lay = T.make_layout(cfg, ragged=True, extra_tokens=cfg.page)
    check_parity(cfg, lay, T.make_qkv(cfg, lay, q_scale=2.0), policy)
    cfg = C.CONFIGS["c5c"].with_(n_queries=2, lp=700, t=80, lc=16)
    lay = T.make_layout(cfg, ragged=True, extra_tokens=cfg.page, dag_override=lambda: W.chain(40, 2))
    r = check_parity(cfg, lay, T.make_qkv(cfg, lay, q_scale=2.0), policy)
    assert r["res"]["batch"].stats["n_items"] > 0


def test_page_permutation_bitwise_and_determinism():
    cfg = C.CONFIGS["c2"].with_(lp=1024)
    lay = T.make_layout(cfg, contiguous=True, extra_tokens=cfg.page)
    ten = T.make_qkv(cfg, lay)
    a = run_step(cfg, lay, ten)
    b = run_step(cfg, lay, ten)
    assert torch.equal(a["out"], b["out"]) and torch.equal(a["lse"], b["lse"])
    perm = torch.from_numpy(np.random.default_rng(3).permutation(lay.num_pages))
    ten2 = dict(ten)
    for key in ("k_cache", "v_cache"):
        x = torch.empty_like(ten[key])
        x[:, perm] = ten[key]
        ten2[key] = x
    lay2 = T.make_layout(cfg, contiguous=True, extra_tokens=cfg.page)
    lay2.page_table = perm.numpy()[lay.page_table].astype(np.int32)
    c = run_step(cfg, lay2, ten2)
    assert torch.equal(a["out"], c["out"]) and torch.equal(a["lse"], c["lse"])


@pytest.mark.parametrize("world", [2, 3])
def test_strong_shards_bitwise(world):
    """SURVEY.md §8(e) bitwise check: each rank's sub-batch (shard.rank_queries, strong mode) gives
    exactly the single-GPU outputs of its queries -- queries share no work, so nothing can differ.
    With fixed chunking (explicit chunk_tokens): the planner's small-step split adapts the chunk
    length to a batch's total work, which a shard changes."""
    from paper_2510_24390_b200 import shard
    cfg = C.CONFIGS["c3"].with_(lp=1024, t=200)
    lay = T.make_layout(cfg, ragged=True, extra_tokens=cfg.page)
    ten = T.make_qkv(cfg, lay)
    full = run_step(cfg, lay, ten, chunk_tokens=512)
    for rank in range(world):
        qs = shard.rank_queries(cfg.n_queries, rank, world, "strong")
        sub, br = T.subset_layout(lay, qs)
        idx = torch.from_numpy(br)
        ten_r = dict(ten)
        for key in ("q", "k_new", "v_new"):
            ten_r[key] = ten[key][:, idx]
        got = run_step(cfg, sub, ten_r, chunk_tokens=512)
        assert torch.equal(got["out"], full["out"][idx.cuda()])
        assert torch.equal(got["lse"], full["lse"][idx.cuda()])


def test_advance_three_steps_and_rewrite():
    cfg = C.CONFIGS["c1"].with_(lp=200, t=70, lc=8, hq=8, hkv=2, d=128)
    lay = T.make_layout(cfg, ragged=True, extra_tokens=3 * cfg.page)
    ten = T.make_qkv(cfg, lay, layers=3)
    from oracle import append as OA, step as OS
    dev = torch.device("cuda")
    batch = batch_for(cfg, lay)
    kc, vc = ten["k_cache"][0].to(dev), ten["v_cache"][0].to(dev)
    k_ref, v_ref, own = u16(ten["k_cache"][0]), u16(ten["v_cache"][0]), lay.own_len.copy()
    for step in range(3):
        q, kn, vn = (ten[x][step].to(dev).contiguous() for x in ("q", "k_new", "v_new"))
        out = torch.empty_like(q)
        batch.step(q, kn, vn, kc, vc, out)
        k_ref, own2 = OA.kv_append(k_ref, u16(ten["k_new"][step]), lay.page_table, lay.point_pt_off, own, cfg.page)
        v_ref, _ = OA.kv_append(v_ref, u16(ten["v_new"][step]), lay.page_table, lay.point_pt_off, own, cfg.page)
        own = own2
        ref, _ = OS.expand_step(lay, u16(ten["q"][step]), k_ref, v_ref, own_len=own)
        torch.cuda.synchronize()
        assert np.array_equal(batch.own_len.cpu().numpy(), own)
        assert np.array_equal(u16(kc), k_ref) and np.array_equal(u16(vc), v_ref)
        o = out.float().cpu().numpy()
        assert np.abs(o - ref).max() <= 2e-2
        assert np.linalg.norm(o - ref) / np.linalg.norm(ref) <= 5e-3
    # rewrite mode keeps lengths and rewrites the last slot
    q, kn, vn = (ten[x][0].to(dev).contiguous() for x in ("q", "k_new", "v_new"))
    batch.step(q, kn, vn, kc, vc, torch.empty_like(q), mode=orion.APPEND_REWRITE)
    torch.cuda.synchronize()
    assert np.array_equal(batch.own_len.cpu().numpy(), own)


def test_append_capacity_guard():
    cfg = C.CONFIGS["c1"]
    lay = T.make_layout(cfg)
    lay.point_cap[:] = lay.own_len                 # capacity == own_len: no room to append
    ten = T.make_qkv(cfg, lay)
    res = run_step(cfg, lay, ten)
    assert np.array_equal(res["own_len"], lay.own_len)
    assert torch.equal(res["k_cache"].cpu(), ten["k_cache"][0])


def test_single_token_contexts_bitwise_v():
    # closed form on the GPU: a one-token context returns that V row exactly (P = 1).
    cfg = C.CONFIGS["c1"].with_(lp=0, t=1, lc=0)
    lay = T.make_layout(cfg, dag_override=lambda: W.wide(5), extra_tokens=0)
    lay.own_len[:] = 0
    ten = T.make_qkv(cfg, lay)
    lay.point_cap[:] = 64
    res = run_step(cfg, lay, ten)
    kc = res["v_cache"].cpu()
    for b in range(5):
        page = lay.page_table[lay.point_pt_off[b]]
        for h in range(cfg.hq):
            assert torch.equal(res["out"][b, h].cpu(), kc[page, h // cfg.g, 0])


@pytest.mark.parametrize("cfgname,flags", [("c2", 0), ("c3", 0), ("c1", 0), ("c2", orion.PLAN_MMA_SYNC),
                                           ("c2", orion.PLAN_ROWS_ON_LANES)])
def test_interleaved_kv_layout(cfgname, flags):
    # K and V of a (page, kv head) adjacent in one [pages][Hkv][2][P][d] array (kv_interleaved):
    # append bit-exact into the interleaved blocks, attention within the gates, every kernel.
    cfg = C.CONFIGS[cfgname]
    if cfgname == "c3":
        cfg = cfg.with_(n_queries=4)
    lay = T.make_layout(cfg, ragged=True, extra_tokens=cfg.page)
    ten = T.make_qkv(cfg, lay, q_scale=2.0)
    check_parity(cfg, lay, ten, flags=flags, interleaved=True)


@pytest.mark.parametrize("flags", [0, orion.PLAN_ROWS_ON_LANES, orion.PLAN_MMA_SYNC])
def test_grid_size_does_not_change_results(flags):
    # Items are handed out by an atomic counter (any CTA may run any item); each item's arithmetic
    # and its partial slots are fixed by the plan, so a 3-CTA grid (the ring wraps many times) and
    # the full grid must give the same bytes.  Fixed chunking: the planner's small-step split
    # would otherwise size the chunks for the SM count.
    cfg = C.CONFIGS["c2"].with_(layers=1)
    lay = T.make_layout(cfg, ragged=True)
    ten = T.make_qkv(cfg, lay)
    dev = torch.device("cuda")
    outs = []
    for num_sms in (0, 3):
        queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i],
                        prefix_pt_off=int(lay.prefix_pt_off[i]), prefix_len=int(lay.prefix_len[i]))
                   for i in range(lay.n_queries)]
        points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
        batch = orion.ExpansionBatch(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, lay.page_table,
                                     lay.own_len, device=dev, flags=flags, num_sms=num_sms, chunk_tokens=512)
        q = ten["q"][0].to(dev).contiguous()
        out = torch.empty_like(q)
        lse = torch.empty(q.shape[:2], dtype=torch.float32, device=dev)
        batch.attend(q, out, ten["k_cache"][0].to(dev).contiguous(), ten["v_cache"][0].to(dev).contiguous(), lse)
        torch.cuda.synchronize()
        outs.append((out.cpu(), lse.cpu()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("flags", [0, orion.PLAN_ROWS_ON_LANES])
@pytest.mark.parametrize("chunk", [0, 64])
def test_empty_items(flags, chunk):
    """Own runs chunked past their current length give items that are empty at run time (their
    dynamic ranges end before t0): c2 with 448 extra capacity tokens per point, the small-step
    split (chunk 0) or explicit 64-token chunks.  Both kernels write neutral partials for them
    (the rows-on-lanes kernel in its scheduler warp, outside the item ring) and match the oracle."""
    cfg = C.CONFIGS["c2"]
    lay = T.make_layout(cfg, ragged=True, extra_tokens=7 * cfg.page)
    ten = T.make_qkv(cfg, lay)
    check_parity(cfg, lay, ten, chunk_tokens=chunk, flags=flags)


@pytest.mark.parametrize("cfgname,mode,extra", [("c2", orion.APPEND_ADVANCE, {}), ("c2", orion.APPEND_REWRITE, {}),
                                                ("c3", orion.APPEND_ADVANCE, {"n_queries": 4}),
                                                ("c4", orion.APPEND_ADVANCE, {"n_queries": 2}),
                                                ("c5c", orion.APPEND_ADVANCE, {"n_queries": 1})])
def test_expand_step_equals_append_then_attn(cfgname, mode, extra):
    """orion_expand_step (the append inside the swap-AB split launch; on c5's hybrid plan the two
    calls) gives bitwise the outputs, lse, caches and lengths of orion_kv_append followed by
    orion_expand_attn.  Ragged own runs with spare capacity, so appended rows land in partially
    filled pages that the same launch's items read."""
    cfg = C.CONFIGS[cfgname].with_(**extra)
    lay = T.make_layout(cfg, ragged=True, extra_tokens=cfg.page)
    ten = T.make_qkv(cfg, lay)
    a = run_step(cfg, lay, ten, mode=mode, fused=True)
    b = run_step(cfg, lay, ten, mode=mode, fused=False)
    assert np.array_equal(a["own_len"], b["own_len"])
    for key in ("out", "lse", "k_cache", "v_cache"):
        x, y = a[key], b[key]
        assert torch.equal(x.view(torch.int16) if x.dtype == torch.bfloat16 else x,
                           y.view(torch.int16) if y.dtype == torch.bfloat16 else y), key
