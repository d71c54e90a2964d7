import sys, time, torch, numpy as np
sys.path.insert(0, "/root/repo")
import bench as BM
from workloads import configs as WC, tensors as WT
args = BM.parse(["--no-e2e"])
cfg = WC.CONFIGS["c4"]
dev = torch.device("cuda", 0)
lay = WT.make_layout(cfg, seed=cfg.seed)
tens = BM.alloc_tensors(args, cfg, lay, 32, dev, 7)
kc, vc, q, kn, vn, out = tens
batch = BM.batch_of(args, cfg, lay, dev)
import paper_2510_24390_b200 as orion
REW = orion.APPEND_REWRITE
def step(mode):
    for l in range(32):
        batch.append(kn[l], vn[l], kc[l], vc[l], mode=REW)
        if mode == "split":
            batch.split(q[l], kc[l], vc[l]); batch.combine(out[l])
        else:
            batch.attend(q[l], out[l], kc[l], vc[l])
s = torch.cuda.current_stream()
for mode in ("split", "attend", "split", "attend"):
    for _ in range(3): step(mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(20): step(mode)
    e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(mode, "ms/step", round(ms, 3), "tok/s", round(1024 / ms * 1e3))
# with events inside (as bench.time_steps)
el, sm, spl, _, _ = BM.time_steps(batch, 32, tens, 20, 3, s)
print("bench.time_steps (events per layer)", round(el / 20, 3), "split_us", round(np.mean(spl) * 1e3, 1))
