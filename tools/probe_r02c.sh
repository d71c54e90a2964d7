#!/bin/bash
ORION_LIB=paper_2510_24390_b200/liborion_check.so timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or shapes or wide or hybrid" > gpurun_out/pc_check.log 2>&1
echo "check rc=$?"; tail -2 gpurun_out/pc_check.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pc_all.log 2>&1
echo "all gpu rc=$?"; tail -4 gpurun_out/pc_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/pc_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/pc_smoke.log
