"""Small multi-item parity probes (used with ORION_DEBUG_GRID=1 to force many items per CTA)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import configs as C, tensors as T, dags as W
from tests.gpu_helpers import run_step, oracle_after_append, u16, errors
from oracle import step as OS

def probe(tag, cfg, dagf=None):
    lay = T.make_layout(cfg, extra_tokens=cfg.page, dag_override=dagf)
    ten = T.make_qkv(cfg, lay, q_scale=2.0)
    res = run_step(cfg, lay, ten)
    k2, v2, own = oracle_after_append(cfg, lay, ten)
    ref, _ = OS.expand_step(lay, u16(ten["q"][0]), k2, v2, own_len=own)
    ma, rel, worst = errors(res["out"], ref)
    print(f"{tag}: items={res['batch'].stats['n_items']} max_abs={ma:.2e} rel={rel:.2e}", flush=True)

base = C.CONFIGS["c1"].with_(hq=8, hkv=2, d=128, page=64)
probe("wide2 lp128 t64", base.with_(lp=128, t=64, lc=8, n_queries=1), lambda: W.wide(2))
probe("wide2 lp256 t130", base.with_(lp=256, t=130, lc=8, n_queries=1), lambda: W.wide(2))
probe("wide3 lp512 t200", base.with_(lp=512, t=200, lc=8, n_queries=1), lambda: W.wide(3))
probe("diamond lp300", base.with_(lp=300, t=150, lc=20, n_queries=1), None)
probe("mixed8 2q", base.with_(lp=300, t=150, lc=20, n_queries=2, dag="mixed8"), None)
