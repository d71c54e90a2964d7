"""Dev: run one point-prefill parity case (default: the R = 128-row, 8-kv-head layout) and print the
error against oracle O5; with ORION_LIB=...liborion_trace.so a stuck mbarrier prints its offset."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from workloads import configs as C, tensors as T, dags as W
from tests import test_gpu_prefill as TP

lc, hq, hkv = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (32, 32, 8)))
cfg = C.CONFIGS["c1"].with_(lp=300, t=200, lc=lc, page=32, d=128, hq=hq, hkv=hkv)
lay = T.make_layout(cfg, ragged=True, dag_override=W.mixed8)
ten = T.make_qkv(cfg, lay, q_scale=2.0)
TP.check(cfg, lay, ten, TP.q_pre(cfg, lay, scale=3.0))
print("ok")
