"""orion_expand_step's co-residency check on a plain stream and on green-context streams (small
c3 step), one call each, no load: exercises the driver entry points before the full tests."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from workloads import configs as C, tensors as T
from tests.gpu_helpers import batch_for
from paper_2510_24390_b200.partition import SmPartition

cfg = C.CONFIGS["c3"].with_(n_queries=4)
lay = T.make_layout(cfg, ragged=True, extra_tokens=cfg.page)
ten = T.make_qkv(cfg, lay)
dev = torch.device("cuda")
dt = {k: ten[k][0].to(dev).contiguous() for k in ("k_cache", "v_cache", "q", "k_new", "v_new")}
batch = batch_for(cfg, lay)
out = torch.empty_like(dt["q"])
batch.step(dt["q"], dt["k_new"], dt["v_new"], dt["k_cache"], dt["v_cache"], out, mode=1)
torch.cuda.synchronize()
print("plain stream ok", float(out.float().abs().mean()))
for n in (100, 16):
    part = SmPartition(n)
    part.sync_before()
    batch.step(dt["q"], dt["k_new"], dt["v_new"], dt["k_cache"], dt["v_cache"], out, mode=1, stream=part.first)
    part.synchronize()
    print("partition", part.sms, "ok", float(out.float().abs().mean()))
    part.close()
