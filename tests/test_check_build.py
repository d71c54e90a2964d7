"""T6 — the ORION_CHECK debug library (`make check` -> liborion_check.so, csrc/kernels.cu
check_plan_kernel): the device content checks include/orion.h leaves out of the release build
(SURVEY.md §8(b) "Content checks (page ids in range) run only in the ORION_CHECK debug build").
CPU: it exports the same symbols.  GPU (subprocess with ORION_LIB): valid steps pass the checks
and stay parity-green; a page table naming a page outside [0, num_pages) is reported as
ORION_ERR_INVALID_ARG instead of the silent zero-fill of an out-of-range TMA box."""
import ctypes
import os
import subprocess
import sys

import pytest

from paper_2510_24390_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK_LIB = os.path.join(ROOT, "paper_2510_24390_b200", "liborion_check.so")


def _need_lib():
    if not os.path.exists(CHECK_LIB):
        pytest.fail(f"{CHECK_LIB} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")


def test_check_library_exports_every_symbol():
    _need_lib()
    L = ctypes.CDLL(CHECK_LIB)
    for name in _lib.EXPORTED_SYMBOLS:
        assert hasattr(L, name), name


SCRIPT = r'''
import numpy as np, torch
import paper_2510_24390_b200 as orion
from paper_2510_24390_b200 import _lib
from workloads import configs as C, tensors as T
from tests.gpu_helpers import check_parity, run_step
assert _lib.LIB_PATH.endswith("liborion_check.so"), _lib.LIB_PATH
for cfg in (C.CONFIGS["c1"], C.CONFIGS["c1"].with_(d=128, hq=8, hkv=2)):
    lay = T.make_layout(cfg, ragged=True, extra_tokens=cfg.page)
    ten = T.make_qkv(cfg, lay, q_scale=2.0)
    check_parity(cfg, lay, ten, 0)                       # valid plan: passes the checks, parity-green
    bad = lay.page_table.copy()
    bad[int(lay.prefix_pt_off[0])] = lay.num_pages + 7   # a prefix page every branch reads
    lay.page_table = bad
    try:
        run_step(cfg, lay, ten, 0)
    except orion.OrionError as e:
        assert e.code == _lib.ERR_INVALID_ARG and "ORION_CHECK" in str(e) and "page id" in str(e), str(e)
    else:
        raise AssertionError("out-of-range page id not reported")
# a device plan that is not a copy of the host plan (stale / foreign) is reported
cfg = C.CONFIGS["c1"].with_(d=128, hq=8, hkv=2)
lay = T.make_layout(cfg, ragged=True, extra_tokens=cfg.page)
ten = T.make_qkv(cfg, lay)
from tests.gpu_helpers import batch_for
a = batch_for(cfg, lay, chunk_tokens=64)
b = batch_for(cfg, lay, chunk_tokens=512, flags=orion.PLAN_NO_MERGE)
dev = torch.device("cuda")
q = ten["q"][0].to(dev); out = torch.empty_like(q)
kc, vc = ten["k_cache"][0].to(dev), ten["v_cache"][0].to(dev)
try:
    orion.expand_attn(cfg.hq, cfg.hkv, cfg.d, cfg.page, q, out, None, kc, vc, a.page_table, a.own_len,
                      a.h_plan, b.d_plan, a.workspace)
except orion.OrionError as e:
    assert e.code == _lib.ERR_INVALID_ARG and "d_plan" in str(e), str(e)
else:
    raise AssertionError("mismatched device plan not reported")
# an append whose own-run page id lies outside the caches is reported (never written)
bad = lay.page_table.copy()
bad[int(lay.point_pt_off[1])] = lay.num_pages + 3
c = batch_for(cfg, lay)
c.page_table = torch.from_numpy(bad).to(dev)
kn, vn = ten["k_new"][0].to(dev), ten["v_new"][0].to(dev)
try:
    c.append(kn, vn, kc, vc)
except orion.OrionError as e:
    assert e.code == _lib.ERR_INVALID_ARG and "outside [0, num_pages)" in str(e), str(e)
else:
    raise AssertionError("out-of-range append page not reported")
print("CHECK_BUILD_OK")
'''


@pytest.mark.gpu
def test_check_build_catches_bad_page_ids():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _need_lib()
    env = dict(os.environ, ORION_LIB=CHECK_LIB, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "CHECK_BUILD_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
