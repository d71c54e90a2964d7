import sys, torch, numpy as np
sys.path.insert(0, "/root/repo")
import bench as BM
from workloads import configs as WC, tensors as WT
import paper_2510_24390_b200 as orion
nq = int(sys.argv[1])
args = BM.parse(["--no-e2e"])
cfg = WC.CONFIGS["c4"].with_(n_queries=nq)
dev = torch.device("cuda", 0)
lay = WT.make_layout(cfg, seed=cfg.seed)
tens = BM.alloc_tensors(args, cfg, lay, 32, dev, 7)
kc, vc, q, kn, vn, out = tens
batch = BM.batch_of(args, cfg, lay, dev)
REW = orion.APPEND_REWRITE
def step(mode):
    for l in range(32):
        if "a" in mode: batch.append(kn[l], vn[l], kc[l], vc[l], mode=REW)
        if "s" in mode: batch.split(q[l], kc[l], vc[l])
        if "c" in mode: batch.combine(out[l])
s = torch.cuda.current_stream()
for mode in ("asc", "s", "as", "sc", "a", "c"):
    for _ in range(3): step(mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10): step(mode)
    e1.record(s); torch.cuda.synchronize()
    print(f"nq={nq} mode={mode:4s} us/layer {e0.elapsed_time(e1) / 10 / 32 * 1e3:8.1f}")
