"""Which SM count does the driver report for a green-context stream's context?  (cuStreamGetCtx +
cuCtxGetDevResource, as orion_expand_step's co-residency check does.)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from cuda.bindings import driver as d
from paper_2510_24390_b200.partition import SmPartition

torch.zeros(1, device="cuda")
for n in (16, 100):
    part = SmPartition(n)
    for name, st in (("first", part.first), ("second", part.second), ("torch default", torch.cuda.current_stream())):
        err, ctx = d.cuStreamGetCtx(st.cuda_stream)
        err2, res = d.cuCtxGetDevResource(ctx, d.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM)
        print(f"partition {n}: {name}: sms {part.sms}, stream ctx SM count = {res.sm.smCount if not int(err2) else err2}")
    part.close()
