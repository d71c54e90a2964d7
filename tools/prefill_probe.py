"""Point-prefill probe: c4-shaped prefill attention on a few queries, timed (and traced when run
with ORION_LIB=paper_2510_24390_b200/liborion_trace.so)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_24390_b200 as orion
from workloads import configs as C, tensors as T

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 16
flags = orion.PLAN_PAIR if "pair" in sys.argv[2:] else 0
cfg = C.CONFIGS["c4"].with_(n_queries=nq)
lay = T.make_layout(cfg)
dev = torch.device("cuda")
queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i], prefix_pt_off=int(lay.prefix_pt_off[i]),
                prefix_len=int(lay.prefix_len[i])) for i in range(lay.n_queries)]
points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
batch = orion.ExpansionBatch(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, lay.page_table, lay.own_len,
                             device=dev, prefill_rows=cfg.lc, flags=flags)
kc = torch.randn((lay.num_pages, cfg.hkv, cfg.page, cfg.d), device=dev).to(torch.bfloat16)
vc = torch.randn_like(kc)
q = torch.randn((lay.n_branches, cfg.lc, cfg.hq, cfg.d), device=dev).to(torch.bfloat16)
out = torch.empty_like(q)
for _ in range(2):
    batch.attend(q, out, kc, vc)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    batch.attend(q, out, kc, vc)
e1.record()
torch.cuda.synchronize()
st = batch.stats
ms = e0.elapsed_time(e1) / 5
ctx = st["logical_tokens"] - lay.n_branches * cfg.lc
flop = cfg.hq * cfg.d * 4.0 * (cfg.lc * ctx + lay.n_branches * cfg.lc * (cfg.lc + 1) / 2)
print(f"prefill nq={nq} {'paired' if flags else 'unpaired'}: {ms:.3f} ms, {flop / ms / 1e9:.0f} TFLOP/s, items {st['n_items']}, "
      f"streamed {st['streamed_tokens'] * cfg.d * 4 / 1e9:.1f} GB K/V")
