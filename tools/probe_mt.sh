#!/bin/bash
P=paper_2510_24390_b200
ORION_LIB=$P/liborion_mt.so timeout 60 python tools/prefill_probe.py 16 2>&1 | tail -1; echo "mt probe rc=$?"
ORION_LIB=$P/liborion_mtcheck.so timeout 600 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_parity.py -x -q --timeout 120 -k "hybrid or prefill or rows_on_lanes or empty or interleaved or grid" > gpurun_out/t_mt.log 2>&1
echo "mt tests rc=$?"; tail -2 gpurun_out/t_mt.log
bash tools/ab_rol.sh 2 liborion liborion_qe liborion_mt liborion_mtqe
