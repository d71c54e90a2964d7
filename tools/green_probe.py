"""Feasibility probe: green contexts (SM partitions) with torch GEMMs and the orion kernels.
Creates a green context over N SMs, wraps its stream for torch, runs a GEMM and an orion decode
step on it, and compares timings / results with the primary context's stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import cuda.bindings.driver as d


def chk(r):
    err = r[0] if isinstance(r, tuple) else r
    if int(err) != 0:
        raise RuntimeError(f"CUDA driver error {err}")
    return r[1:] if isinstance(r, tuple) and len(r) > 2 else (r[1] if isinstance(r, tuple) else None)


torch.zeros(1, device="cuda")
dev = chk(d.cuDeviceGet(0))
res = chk(d.cuDeviceGetDevResource(dev, d.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
print("SMs:", res.sm.smCount)
want = int(sys.argv[1]) if len(sys.argv) > 1 else 32
out = d.cuDevSmResourceSplitByCount(1, res, 0, want)
print("split:", [type(x).__name__ for x in out])
err, groups, ng, rem = out
assert int(err) == 0, err
print("group SMs:", groups[0].sm.smCount, "remaining:", rem.sm.smCount)
streams = {}
for name, r in (("small", groups[0]), ("rest", rem)):
    desc = chk(d.cuDevResourceGenerateDesc([r], 1))
    g = chk(d.cuGreenCtxCreate(desc, dev, d.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
    st = chk(d.cuGreenCtxStreamCreate(g, d.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
    streams[name] = torch.cuda.ExternalStream(int(st))

a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
b = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)


def time_on(s, f, n=5):
    with torch.cuda.stream(s):
        f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(n):
            f()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


gemm = lambda: a @ b
print("gemm primary ms:", time_on(torch.cuda.current_stream(), gemm))
print("gemm small ms:", time_on(streams["small"], gemm))
print("gemm rest ms:", time_on(streams["rest"], gemm))

import paper_2510_24390_b200 as orion
from workloads import configs as C, tensors as T
cfg = C.CONFIGS["c4"].with_(n_queries=16)
lay = T.make_layout(cfg)
queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i], prefix_pt_off=int(lay.prefix_pt_off[i]),
                prefix_len=int(lay.prefix_len[i])) for i in range(lay.n_queries)]
points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
res_out = {}
for name, s, cap in (("primary", torch.cuda.current_stream(), 0), ("small", streams["small"], groups[0].sm.smCount),
                     ("rest", streams["rest"], rem.sm.smCount)):
    batch = orion.ExpansionBatch(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, lay.page_table, lay.own_len,
                                 num_sms=cap)
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    kc = torch.randn((lay.num_pages, cfg.hkv, cfg.page, cfg.d), generator=g, device="cuda").to(torch.bfloat16)
    vc = torch.randn_like(kc)
    q = torch.randn((lay.n_branches, cfg.hq, cfg.d), generator=g, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    ms = time_on(s, lambda: batch.attend(q, out, kc, vc, stream=s))
    res_out[name] = out.clone()
    print(f"orion attend on {name} (grid cap {cap}): {ms:.3f} ms")
print("results equal:", torch.equal(res_out["primary"], res_out["small"]), torch.equal(res_out["primary"], res_out["rest"]))
