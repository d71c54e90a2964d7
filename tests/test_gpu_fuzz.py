"""Seeded GPU fuzz of the decode step and the point prefill against the oracles: random DAGs (all
three edge kinds), GQA groups 1/2/4/7/8, head_dim 64/128, every supported page size 16..256,
both policies, piece chunking, ragged lengths.  Same gates as the parity tests (north_star)."""
import random

import numpy as np
import pytest
import torch

import paper_2510_24390_b200 as orion
from oracle import prefill as OP, step as OS
from workloads import configs as C, tensors as T, dags as W
from tests.gpu_helpers import MAX_ABS, REL_L2, check_parity, u16
from tests.test_gpu_prefill import run_prefill

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def fuzz_cfg(seed):
    rng = random.Random(seed)
    g = rng.choice([1, 2, 4, 7, 8])
    hkv = rng.choice([1, 2, 4]) if g != 7 else rng.choice([1, 4])
    page = rng.choice([16, 32, 64, 128, 256])
    lc = rng.choice([4, 8, 16])
    cfg = C.CONFIGS["c1"].with_(hq=g * hkv, hkv=hkv, d=rng.choice([64, 128]), page=page,
                                lp=rng.choice([1, 37, 200, 513]), t=lc + rng.randint(2, 150), lc=lc,
                                n_queries=rng.randint(1, 3), seed=seed)
    n = rng.randint(1, 9)
    dag = lambda: W.random_dag(random.Random(seed * 31), n, p=rng.choice([0.2, 0.5]), null_frac=0.1)
    return rng, cfg, dag


@pytest.mark.parametrize("seed", range(40))
def test_fuzz_decode(seed):
    rng, cfg, dag = fuzz_cfg(seed)
    lay = T.make_layout(cfg, ragged=True, extra_tokens=cfg.page, dag_override=dag)
    ten = T.make_qkv(cfg, lay, q_scale=rng.choice([1.0, 3.0]), sink=rng.random() < 0.3)
    check_parity(cfg, lay, ten, policy=rng.choice([0, 1]), chunk_tokens=rng.choice([0, 64, 192]))


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_prefill(seed):
    rng, cfg, dag = fuzz_cfg(1000 + seed)
    lay = T.make_layout(cfg, ragged=True, dag_override=dag)
    ten = T.make_qkv(cfg, lay)
    policy = rng.choice([0, 1])
    qp = T.bf16_randn_u16((lay.n_branches, cfg.lc, cfg.hq, cfg.d), seed, "cpu", scale=2.0)
    # odd seeds run the paired kernel (ORION_PLAN_PAIR: shared K/V tiles, alternating tails)
    out, lse, _ = run_prefill(cfg, lay, ten, qp, policy, flags=orion.PLAN_PAIR if seed % 2 else 0)
    ref, _ = OP.point_prefill(lay, u16(qp), u16(ten["k_cache"][0]), u16(ten["v_cache"][0]), policy=policy)
    o = out.float().cpu().numpy().astype(np.float64)
    assert np.isfinite(o).all()
    assert float(np.abs(o - ref).max()) <= MAX_ABS
    assert float(np.linalg.norm(o - ref) / np.linalg.norm(ref)) <= REL_L2
