#!/bin/bash
P=paper_2510_24390_b200
ORION_LIB=$P/liborion_check.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "empty_items or interleaved" --timeout 120 > gpurun_out/t_empty.log 2>&1
echo "check rc=$?"; tail -2 gpurun_out/t_empty.log
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_expansion.py tests/test_gpu_prefill.py -x -q --timeout 400 > gpurun_out/t_small.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/t_small.log
for nb in 1 2 8; do echo "nb=$nb"; timeout 120 python tools/graph_probe.py $nb 2>&1 | grep -E "plan|round"; done
bash tools/ab_r02.sh $P/liborion_prev.so $P/liborion.so c4 1 --queries 8
