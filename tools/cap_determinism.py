import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2510_24390_b200 as orion
from workloads import configs as C, tensors as T
cfg = C.CONFIGS["c4"].with_(n_queries=16)
lay = T.make_layout(cfg)
queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i], prefix_pt_off=int(lay.prefix_pt_off[i]),
                prefix_len=int(lay.prefix_len[i])) for i in range(lay.n_queries)]
points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
g = torch.Generator(device="cuda"); g.manual_seed(1)
kc = torch.randn((lay.num_pages, cfg.hkv, cfg.page, cfg.d), generator=g, device="cuda").to(torch.bfloat16)
vc = torch.randn_like(kc)
q = torch.randn((lay.n_branches, cfg.hq, cfg.d), generator=g, device="cuda").to(torch.bfloat16)
outs = {}
for cap in (0, 148, 116, 32, 7):
    b = orion.ExpansionBatch(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, lay.page_table, lay.own_len, num_sms=cap)
    o = torch.empty_like(q); b.attend(q, o, kc, vc); torch.cuda.synchronize(); outs[cap] = o
    o2 = torch.empty_like(q); b.attend(q, o2, kc, vc); torch.cuda.synchronize()
    print(cap, "repeat equal", torch.equal(o, o2), "vs cap0", torch.equal(o, outs[0]), float((o.float()-outs[0].float()).abs().max()))
