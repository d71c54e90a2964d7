"""Quick GPU parity probe for one config/kernel variant (prints errors instead of asserting)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_24390_b200 as orion
from workloads import configs as C, tensors as T
from tests.gpu_helpers import run_step, oracle_after_append, u16, errors
from oracle import step as OS

def probe(name, flags, **kw):
    cfg = C.CONFIGS[name].with_(**kw) if kw else C.CONFIGS[name]
    lay = T.make_layout(cfg, extra_tokens=cfg.page)
    ten = T.make_qkv(cfg, lay, q_scale=2.0)
    t0 = time.time()
    res = run_step(cfg, lay, ten, flags=flags)
    k2, v2, own = oracle_after_append(cfg, lay, ten)
    br = list(range(min(lay.n_branches, 16)))
    ref, ref_lse = OS.expand_step(lay, u16(ten["q"][0]), k2, v2, branches=br, own_len=own)
    o = res["out"][br]
    ma, rel, worst = errors(o, ref)
    lse = res["lse"][br].cpu().numpy()
    print(f"{name} flags={flags} {kw}: max_abs={ma:.3e} rel={rel:.3e} worst_branch={worst:.3e} "
          f"lse_err={np.abs(lse-ref_lse).max():.3e} nan={np.isnan(o.float().cpu().numpy()).sum()} "
          f"items={res['batch'].stats['n_items']} ({time.time()-t0:.1f}s)", flush=True)

if __name__ == "__main__":
    for spec in sys.argv[1:]:
        name, flags = spec.split(":")
        probe(name, int(flags))
