#!/bin/bash
# super-tile rows-on-lanes kernel: watchdog build on the rol tests first, then release parity, then A/B
P=paper_2510_24390_b200
ORION_LIB=$P/liborion_check.so timeout 600 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_parity.py -x -q --timeout 120 -k "hybrid or prefill or rows_on_lanes or empty or interleaved or grid or c1" > gpurun_out/t_st1.log 2>&1
echo "check rc=$?"; tail -3 gpurun_out/t_st1.log | cut -c1-300
[ "$1" == "quick" ] && exit 0
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q --timeout 300 > gpurun_out/t_st2.log 2>&1
echo "release rc=$?"; tail -3 gpurun_out/t_st2.log | cut -c1-300
bash tools/ab_rol.sh 2 liborion_prev liborion
