"""§8(f) rank 3 under load: the expansion step keeps parity while a co-scheduled prefill load
(cuBLAS bf16 GEMMs of a Llama-3-8B layer prefill -- the compute-bound Pre-stage work of PAPER.md:220,
392) runs beside it, (a) on disjoint SM partitions (green contexts, paper_2510_24390_b200/partition.py)
and (b) on a low-priority stream of the same context.  Inputs reach the partition's stream through
an explicit event (streams of different contexts are unordered); outputs are read after both
partitions' streams are synchronised.  Gates as tests/gpu_helpers.py (north_star)."""
import numpy as np
import pytest
import torch

import paper_2510_24390_b200 as orion
from oracle import step as OS
from workloads import configs as C, tensors as T
from tests.gpu_helpers import MAX_ABS, REL_L2, LSE_ABS, batch_for, oracle_after_append, errors, u16

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _setup():
    cfg = C.CONFIGS["c3"].with_(n_queries=4)
    lay = T.make_layout(cfg, ragged=True, extra_tokens=cfg.page)
    ten = T.make_qkv(cfg, lay, q_scale=2.0)
    k2, v2, own = oracle_after_append(cfg, lay, ten)
    ref, ref_lse = OS.expand_step(lay, u16(ten["q"][0]), k2, v2, own_len=own)
    dev = torch.device("cuda")
    dt = {k: ten[k][0].to(dev).contiguous() for k in ("k_cache", "v_cache", "q", "k_new", "v_new")}
    return cfg, lay, ten, dt, ref, ref_lse, own, k2, v2


def _load(n=24):
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    x = torch.randn((4096, 4096), generator=g, device=dev, dtype=torch.bfloat16)
    w = torch.randn((4096, 14336), generator=g, device=dev, dtype=torch.bfloat16) * 0.02
    o = torch.empty((4096, 14336), device=dev, dtype=torch.bfloat16)

    def run():
        for _ in range(n):
            torch.matmul(x, w, out=o)
    return run


def _check(res_out, res_lse, batch, kc, vc, ref, ref_lse, own, k2, v2):
    torch.cuda.synchronize()
    assert np.array_equal(batch.own_len.cpu().numpy(), own)
    assert np.array_equal(u16(kc), k2) and np.array_equal(u16(vc), v2)
    max_abs, rel, _ = errors(res_out, ref)
    assert max_abs <= MAX_ABS and rel <= REL_L2, (max_abs, rel)
    assert float(np.abs(res_lse.cpu().numpy() - ref_lse).max()) <= LSE_ABS


def test_expansion_on_green_partition_with_prefill_load():
    try:
        from paper_2510_24390_b200.partition import SmPartition
        part = SmPartition(100)
    except Exception as exc:                          # no green contexts on this driver / image
        pytest.skip(f"green contexts unavailable: {type(exc).__name__}: {exc}")
    try:
        cfg, lay, ten, dt, ref, ref_lse, own, k2, v2 = _setup()
        batch = batch_for(cfg, lay)
        batch = orion.ExpansionBatch.from_segments(cfg.hq, cfg.hkv, cfg.d, cfg.page, batch.seg_offsets,
                                                   batch.segs, lay.point_pt_off, lay.point_cap,
                                                   lay.page_table, lay.own_len, num_sms=part.sms[0])
        out = torch.empty_like(dt["q"])
        lse = torch.empty(dt["q"].shape[:2], dtype=torch.float32, device=dt["q"].device)
        load = _load()
        part.sync_before()                            # inputs copied on the default stream
        with torch.cuda.stream(part.second):
            load()                                    # prefill GEMMs on the other partition
        batch.step(dt["q"], dt["k_new"], dt["v_new"], dt["k_cache"], dt["v_cache"], out, lse,
                   stream=part.first)
        with torch.cuda.stream(part.second):
            load()
        batch.step(dt["q"], dt["k_new"], dt["v_new"], dt["k_cache"], dt["v_cache"], out, lse,
                   mode=orion.APPEND_REWRITE, stream=part.first)   # same slot again, same answer
        part.synchronize()
        _check(out, lse, batch, dt["k_cache"], dt["v_cache"], ref, ref_lse, own, k2, v2)
    finally:
        part.close()


def test_expansion_under_stream_priorities_with_prefill_load():
    cfg, lay, ten, dt, ref, ref_lse, own, k2, v2 = _setup()
    batch = batch_for(cfg, lay)
    hi = torch.cuda.Stream(priority=-1)
    lo = torch.cuda.Stream(priority=0)
    out = torch.empty_like(dt["q"])
    lse = torch.empty(dt["q"].shape[:2], dtype=torch.float32, device=dt["q"].device)
    load = _load()
    hi.wait_stream(torch.cuda.current_stream())
    lo.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(lo):
        load()
    batch.step(dt["q"], dt["k_new"], dt["v_new"], dt["k_cache"], dt["v_cache"], out, lse, stream=hi)
    with torch.cuda.stream(lo):
        load()
    batch.step(dt["q"], dt["k_new"], dt["v_new"], dt["k_cache"], dt["v_cache"], out, lse,
               mode=orion.APPEND_REWRITE, stream=hi)
    _check(out, lse, batch, dt["k_cache"], dt["v_cache"], ref, ref_lse, own, k2, v2)


def test_release_append_skips_out_of_range_page():
    """Release build: an own-run page id outside [0, num_pages) is never written (the debug build
    reports it, tests/test_check_build.py); the other branches append normally."""
    cfg = C.CONFIGS["c1"].with_(d=128, hq=8, hkv=2)
    lay = T.make_layout(cfg, ragged=True, extra_tokens=cfg.page)
    ten = T.make_qkv(cfg, lay)
    bad = lay.page_table.copy()
    bad[int(lay.point_pt_off[1]) + int(lay.own_len[1]) // cfg.page] = lay.num_pages + 3
    dev = torch.device("cuda")
    batch = batch_for(cfg, lay)
    batch.page_table = torch.from_numpy(bad).to(dev)
    kc, vc = ten["k_cache"][0].to(dev).contiguous(), ten["v_cache"][0].to(dev).contiguous()
    before = u16(kc)
    batch.append(ten["k_new"][0].to(dev).contiguous(), ten["v_new"][0].to(dev).contiguous(), kc, vc)
    torch.cuda.synchronize()
    lay.page_table = bad
    want = lay.own_len + 1
    want[1] -= 1
    assert np.array_equal(batch.own_len.cpu().numpy(), want)
    got = u16(kc)
    # every other branch's slot holds its new row; nothing else changed
    for b in range(lay.n_branches):
        if b == 1:
            continue
        pg = bad[lay.point_pt_off[b] + lay.own_len[b] // cfg.page]
        assert np.array_equal(got[pg, :, lay.own_len[b] % cfg.page], u16(ten["k_new"][0])[b])
    diff = np.argwhere((got != before).any(axis=-1))
    assert len(diff) == (lay.n_branches - 1) * cfg.hkv


def test_fused_step_on_a_partition_smaller_than_its_grid():
    """orion_expand_step on a short step fuses append, split and combine into one cooperative
    launch (its CTAs wait on each other).  A plan built for the whole GPU (148 CTAs) stepped on a
    16-SM green-context partition cannot have every CTA resident: the cooperative launch is
    refused and the call runs append + attention instead -- same results, no hang."""
    try:
        from paper_2510_24390_b200.partition import SmPartition
        part = SmPartition(16)
    except Exception as exc:                          # no green contexts on this driver / image
        pytest.skip(f"green contexts unavailable: {type(exc).__name__}: {exc}")
    try:
        cfg, lay, ten, dt, ref, ref_lse, own, k2, v2 = _setup()
        batch = batch_for(cfg, lay)                   # planned for the whole device
        assert batch.step_launches() == 1             # a short step: fused when it fits
        out = torch.empty_like(dt["q"])
        lse = torch.empty(dt["q"].shape[:2], dtype=torch.float32, device=dt["q"].device)
        part.sync_before()
        batch.step(dt["q"], dt["k_new"], dt["v_new"], dt["k_cache"], dt["v_cache"], out, lse,
                   stream=part.first)
        part.synchronize()
        _check(out, lse, batch, dt["k_cache"], dt["v_cache"], ref, ref_lse, own, k2, v2)
    finally:
        part.close()
