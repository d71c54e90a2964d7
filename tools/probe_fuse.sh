#!/bin/bash
P=paper_2510_24390_b200
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 -k "expand_step" > gpurun_out/t_f1.log 2>&1
echo "fused tests rc=$?"; tail -3 gpurun_out/t_f1.log | cut -c1-400
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_expansion.py tests/test_gpu_costream.py tests/test_gpu_decoder.py -x -q --timeout 400 > gpurun_out/t_f2.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/t_f2.log | cut -c1-400
bash tools/ab_multi.sh 2 liborion_prev liborion
for nb in 1 2 8; do echo "nb=$nb"; timeout 120 python tools/graph_probe.py $nb 2>&1 | grep -E "round"; done
