"""Decode-round launch probe on a small running set (c2-like): 32 layers of append + split +
combine launched eagerly vs replayed from a CUDA graph; per-round device time and, with the
torch profiler, per-kernel device time in both modes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_24390_b200 as orion
from workloads import configs as C, tensors as T

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = C.CONFIGS["c2"]
lay = T.make_layout(cfg)
dev = torch.device("cuda")
queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i], prefix_pt_off=int(lay.prefix_pt_off[i]),
                prefix_len=int(lay.prefix_len[i])) for i in range(lay.n_queries)]
points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
batch = orion.ExpansionBatch(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, lay.page_table,
                             lay.own_len, device=dev)
sel = np.arange(nb, dtype=np.int32)
so, sg = orion.select_branches(batch.seg_offsets, batch.segs, np.asarray(lay.own_len, np.int32), sel)
pts = points[sel]
b = orion.ExpansionBatch.from_segments(cfg.hq, cfg.hkv, cfg.d, cfg.page, so, sg, pts[:, 0], pts[:, 2],
                                       lay.page_table, np.asarray(lay.own_len, np.int32)[sel], device=dev)
L = cfg.layers
kc = [torch.randn((lay.num_pages, cfg.hkv, cfg.page, cfg.d), device=dev).to(torch.bfloat16) for _ in range(L)]
vc = [torch.randn_like(k) for k in kc]
q = [torch.randn((nb, cfg.hq, cfg.d), device=dev).to(torch.bfloat16) for _ in range(L)]
kn = [torch.randn((nb, cfg.hkv, cfg.d), device=dev).to(torch.bfloat16) for _ in range(L)]
vn = [torch.randn_like(k) for k in kn]
out = [torch.empty_like(x) for x in q]
print("plan", b.stats["n_items"], "items", b.stats.get("n_big", 0), "big")


def rnd(s=None):
    for l in range(L):
        b.step(q[l], kn[l], vn[l], kc[l], vc[l], out[l], mode=orion.APPEND_REWRITE, stream=s)


def timeit(f, n=50):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3, (time.perf_counter() - t0) / n * 1e6


g = torch.cuda.CUDAGraph()
cs = torch.cuda.Stream()
cs.wait_stream(torch.cuda.current_stream())
with torch.cuda.graph(g, stream=cs, capture_error_mode="thread_local"):
    rnd(cs)
for name, f in (("eager", rnd), ("graph", g.replay)):
    dev_us, host_us = timeit(f)
    print(f"{name}: {dev_us:.1f} us/round device, {host_us:.1f} us/round host, {dev_us / (3 * L):.2f} us/launch")
from torch.profiler import profile, ProfilerActivity
for name, f in (("eager", rnd), ("graph", g.replay)):
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        for _ in range(10):
            f()
        torch.cuda.synchronize()
    tot = {}
    for ev in p.events():
        if ev.device_type.name == "CUDA":
            k = ev.name.split("(")[0][:40]
            tot.setdefault(k, []).append(ev.device_time)
    print(name, {k: (len(v), round(sum(v) / len(v), 2)) for k, v in tot.items()})
