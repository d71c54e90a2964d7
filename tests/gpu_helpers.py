"""Shared driver for the GPU parity tests: run one expansion decode step of a workloads.Layout
through the CUDA path (paper_2510_24390_b200, C ABI) and through the oracle, on the same bytes."""
import numpy as np
import torch

import paper_2510_24390_b200 as orion
from oracle import step as OS, append as OA
from workloads import tensors as T

MAX_ABS = 2e-2      # north_star gate (BASELINE.json): max-abs error of out
REL_L2 = 5e-3       # north_star gate: relative L2 error of out over the whole tensor
LSE_ABS = 5e-3      # lse (fp32) vs the oracle's fp64 log-sum-exp, natural log


def u16(t):
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def batch_for(cfg, lay, policy=0, chunk_tokens=0, device="cuda", flags=0, interleaved=False):
    queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i],
                    prefix_pt_off=int(lay.prefix_pt_off[i]), prefix_len=int(lay.prefix_len[i]))
               for i in range(lay.n_queries)]
    points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
    return orion.ExpansionBatch(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, lay.page_table,
                                lay.own_len, policy=policy, device=device, chunk_tokens=chunk_tokens,
                                flags=flags, kv_interleaved=interleaved)


def run_step(cfg, lay, ten, policy=0, mode=orion.APPEND_ADVANCE, chunk_tokens=0, layer=0, flags=0,
             interleaved=False, fused=True):
    """Returns dict(out, lse, k_cache, v_cache, own_len) from the GPU after one step.  interleaved:
    the caches live in one [pages][Hkv][2][P][d] array (K/V views of it are passed)."""
    dev = torch.device("cuda")
    batch = batch_for(cfg, lay, policy, chunk_tokens, flags=flags, interleaved=interleaved)
    if interleaved:
        kv = torch.stack([ten["k_cache"][layer], ten["v_cache"][layer]], dim=2).to(dev).contiguous()
        kc, vc = kv[:, :, 0], kv[:, :, 1]
    else:
        kc = ten["k_cache"][layer].to(dev).contiguous()
        vc = ten["v_cache"][layer].to(dev).contiguous()
    q = ten["q"][layer].to(dev).contiguous()
    kn = ten["k_new"][layer].to(dev).contiguous()
    vn = ten["v_new"][layer].to(dev).contiguous()
    out = torch.empty_like(q)
    lse = torch.empty(q.shape[:2], dtype=torch.float32, device=dev)
    batch.step(q, kn, vn, kc, vc, out, lse, mode=mode, fused=fused)
    torch.cuda.synchronize()
    return dict(out=out, lse=lse, k_cache=kc, v_cache=vc, own_len=batch.own_len.cpu().numpy(),
                batch=batch)


def oracle_after_append(cfg, lay, ten, layer=0, rewrite=False):
    k2, own = OA.kv_append(u16(ten["k_cache"][layer]), u16(ten["k_new"][layer]), lay.page_table,
                           lay.point_pt_off, lay.own_len, cfg.page, rewrite=rewrite)
    v2, _ = OA.kv_append(u16(ten["v_cache"][layer]), u16(ten["v_new"][layer]), lay.page_table,
                         lay.point_pt_off, lay.own_len, cfg.page, rewrite=rewrite)
    return k2, v2, own


def errors(out_gpu, ref):
    o = out_gpu.float().cpu().numpy().astype(np.float64)
    diff = o - ref
    max_abs = float(np.abs(diff).max())
    rel = float(np.linalg.norm(diff) / max(np.linalg.norm(ref), 1e-30))
    per_branch = np.linalg.norm(diff.reshape(diff.shape[0], -1), axis=1) / np.maximum(
        np.linalg.norm(ref.reshape(ref.shape[0], -1), axis=1), 1e-30)
    return max_abs, rel, float(per_branch.max())


def check_parity(cfg, lay, ten, policy=0, branches=None, mode=orion.APPEND_ADVANCE, chunk_tokens=0,
                 flags=0, interleaved=False):
    """Full GPU step vs oracle on `branches` (default all).  Asserts the gates; returns errors."""
    res = run_step(cfg, lay, ten, policy, mode, chunk_tokens, flags=flags, interleaved=interleaved)
    rewrite = mode == orion.APPEND_REWRITE
    k2, v2, own = oracle_after_append(cfg, lay, ten, rewrite=rewrite)
    assert np.array_equal(res["own_len"], own)
    assert np.array_equal(u16(res["k_cache"]), k2), "K1 append not bit-exact (K)"
    assert np.array_equal(u16(res["v_cache"]), v2), "K1 append not bit-exact (V)"
    if branches is None:
        branches = list(range(lay.n_branches))
    if len(branches) > 128:           # full-size configs: the same oracle, in worker processes
        from tests.oracle_pool import expand_step_parallel
        ref, ref_lse = expand_step_parallel(lay, u16(ten["q"][0]), k2, v2, policy=policy,
                                            branches=branches, own_len=own)
    else:
        ref, ref_lse = OS.expand_step(lay, u16(ten["q"][0]), k2, v2, policy=policy, branches=branches,
                                      own_len=own)
    out = res["out"][branches]
    max_abs, rel, worst = errors(out, ref)
    lse_err = float(np.abs(res["lse"][branches].cpu().numpy() - ref_lse).max())
    assert np.isfinite(out.float().cpu().numpy()).all()
    assert max_abs <= MAX_ABS and rel <= REL_L2, (max_abs, rel, worst)
    assert lse_err <= LSE_ABS, lse_err
    return dict(max_abs=max_abs, rel_l2=rel, worst_branch_rel=worst, lse_err=lse_err, res=res)
