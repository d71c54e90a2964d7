"""GPU parity of the expansion driver (paper_2510_24390_b200.expansion):
a whole expansion of small DAG batches, round by round, against the oracles -- schedule O6
(bit-exact), append O4 (bit-exact cache), prefill O5 and decode O3 (north_star gates) on the
evolving cache, with every oracle input generated on the host, never read back from the GPU."""
import numpy as np
import pytest
import torch

from paper_2510_24390_b200.expansion import Expansion
from oracle import append as OA, expansion as OE, prefill as OP, step as OS
from workloads import configs as C, tensors as T, dags as W
from tests.gpu_helpers import MAX_ABS, REL_L2, u16

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def gate(got, ref):
    o = got.float().cpu().numpy().astype(np.float64)
    assert np.isfinite(o).all()
    d = o - ref
    assert float(np.abs(d).max()) <= MAX_ABS
    assert float(np.linalg.norm(d) / np.linalg.norm(ref)) <= REL_L2


@pytest.mark.parametrize("dagf,policy", [(W.fig4, 0), (W.mixed8, 0), (W.mixed8, 1), (W.diamond, 1)])
def test_whole_expansion_matches_oracles(dagf, policy):
    cfg = C.CONFIGS["c1"].with_(n_queries=2, lp=96, t=21, lc=8, page=16, d=128, hq=8, hkv=2)
    lay = T.make_layout(cfg, dag_override=dagf)
    ten = T.make_qkv(cfg, lay)
    dev = torch.device("cuda")
    tokens = np.full(lay.n_branches, cfg.t - cfg.lc, np.int32)
    tokens[1::3] = 3                                  # ragged: some points stop early
    queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i],
                    prefix_pt_off=int(lay.prefix_pt_off[i]), prefix_len=int(lay.prefix_len[i]))
               for i in range(lay.n_queries)]
    points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
    ex = Expansion(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, lay.page_table, cfg.lc,
                   tokens, policy=policy, device=dev)
    kc = ten["k_cache"][0].to(dev).contiguous()
    vc = ten["v_cache"][0].to(dev).contiguous()
    k_ref, v_ref = u16(ten["k_cache"][0]), u16(ten["v_cache"][0])
    want = OE.batch_schedule([(int(lay.n_points[i]), lay.edges[i], int(lay.branch0[i]))
                              for i in range(lay.n_queries)], tokens)
    rnd = 0
    while True:
        pre, dec = ex.next_round()
        if len(pre) == 0 and len(dec) == 0:
            break
        assert (list(pre), list(dec)) == want[rnd]
        if len(pre):
            qp = T.bf16_randn_u16((len(pre), cfg.lc, cfg.hq, cfg.d), 1000 + rnd, "cpu", scale=2.0)
            out = torch.empty((len(pre), cfg.lc, cfg.hq, cfg.d), dtype=torch.bfloat16, device=dev)
            ex.prefill(pre, [qp.to(dev)], [kc], [vc], [out])
            q_full = np.zeros((lay.n_branches, cfg.lc, cfg.hq, cfg.d), np.uint16)
            q_full[pre] = u16(qp)
            ref, _ = OP.point_prefill(lay, q_full, k_ref, v_ref, policy=policy, branches=list(pre),
                                      own_len=ex.own_len)
            gate(out, ref)
        if len(dec):
            own_before = ex.own_len[dec].copy()
            qd = T.bf16_randn_u16((len(dec), cfg.hq, cfg.d), 2000 + rnd, "cpu", scale=2.0)
            kn = T.bf16_randn_u16((len(dec), cfg.hkv, cfg.d), 3000 + rnd, "cpu")
            vn = T.bf16_randn_u16((len(dec), cfg.hkv, cfg.d), 4000 + rnd, "cpu")
            out = torch.empty((len(dec), cfg.hq, cfg.d), dtype=torch.bfloat16, device=dev)
            ex.decode(dec, [qd.to(dev)], [kn.to(dev)], [vn.to(dev)], [kc], [vc], [out])
            k_ref, own2 = OA.kv_append(k_ref, u16(kn), lay.page_table, lay.point_pt_off[dec],
                                       own_before, cfg.page)
            v_ref, _ = OA.kv_append(v_ref, u16(vn), lay.page_table, lay.point_pt_off[dec],
                                    own_before, cfg.page)
            assert np.array_equal(own2, ex.own_len[dec])
            q_full = np.zeros((lay.n_branches, cfg.hq, cfg.d), np.uint16)
            q_full[dec] = u16(qd)
            ref, _ = OS.expand_step(lay, q_full, k_ref, v_ref, policy=policy, branches=list(dec),
                                    own_len=ex.own_len)
            gate(out, ref)
        rnd += 1
    torch.cuda.synchronize()
    assert rnd == len(want)
    assert np.array_equal(u16(kc.cpu()), k_ref) and np.array_equal(u16(vc.cpu()), v_ref)
    assert (ex.own_len == cfg.lc + tokens).all()


@pytest.mark.parametrize("dagf,policy", [(W.mixed8, 0), (W.fig4, 1)])
def test_graph_replay_equals_eager(dagf, policy):
    """Decode rounds replayed from a CUDA graph (captured once per running set) give bitwise the
    eager launches' outputs and caches, over a whole ragged expansion of 2 layers; the round's
    input tensors keep their addresses and are refilled in place each round."""
    cfg = C.CONFIGS["c1"].with_(n_queries=2, lp=96, t=21, lc=8, page=16, d=128, hq=8, hkv=2)
    lay = T.make_layout(cfg, dag_override=dagf)
    ten = T.make_qkv(cfg, lay)
    dev = torch.device("cuda")
    tokens = np.full(lay.n_branches, cfg.t - cfg.lc, np.int32)
    tokens[1::3] = 3
    queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i],
                    prefix_pt_off=int(lay.prefix_pt_off[i]), prefix_len=int(lay.prefix_len[i]))
               for i in range(lay.n_queries)]
    points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
    L, B = 2, lay.n_branches
    arms = []
    for _ in range(2):
        ex = Expansion(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, lay.page_table, cfg.lc,
                       tokens, policy=policy, device=dev)
        kc = [ten["k_cache"][0].to(dev).contiguous() for _ in range(L)]
        vc = [ten["v_cache"][0].to(dev).contiguous() for _ in range(L)]
        bufs = {n: [torch.empty((B, h, cfg.d), dtype=torch.bfloat16, device=dev) for _ in range(L)]
                for n, h in (("q", cfg.hq), ("k", cfg.hkv), ("v", cfg.hkv), ("o", cfg.hq))}
        arms.append((ex, kc, vc, bufs))
    rnd = 0
    while True:
        rounds = [a[0].next_round() for a in arms]
        pre, dec = rounds[0]
        assert all(np.array_equal(r[0], pre) and np.array_equal(r[1], dec) for r in rounds)
        if len(pre) == 0 and len(dec) == 0:
            break
        outs = []
        for gi, (ex, kc, vc, bufs) in enumerate(arms):
            if len(pre):
                qp = T.bf16_randn_u16((len(pre), cfg.lc, cfg.hq, cfg.d), 1000 + rnd, "cpu").to(dev)
                op = torch.empty_like(qp)
                ex.prefill(pre, [qp] * L, kc, vc, [op] * L)
            if len(dec):
                n = len(dec)
                for l in range(L):
                    for nm, h, sd in (("q", cfg.hq, 2000), ("k", cfg.hkv, 3000), ("v", cfg.hkv, 4000)):
                        bufs[nm][l][:n].copy_(T.bf16_randn_u16((n, h, cfg.d), sd + 10 * rnd + l, "cpu").to(dev))
                view = lambda nm: [t[:n] for t in bufs[nm]]
                ex.decode(dec, view("q"), view("k"), view("v"), kc, vc, view("o"), graph=gi == 1)
                outs.append(torch.stack([t[:n] for t in bufs["o"]]).cpu())
        if len(dec):
            assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16)), f"round {rnd}"
        rnd += 1
    torch.cuda.synchronize()
    for l in range(L):
        assert torch.equal(arms[0][1][l].view(torch.int16), arms[1][1][l].view(torch.int16))
        assert torch.equal(arms[0][2][l].view(torch.int16), arms[1][2][l].view(torch.int16))
    assert arms[1][0].captures == arms[1][0].rebuilds >= 2
