#!/bin/bash
# full validation: -m gpu suite, smoke, default bench line, reference arm
timeout 2400 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/gpu_all.log 2>&1
echo "gpu tests rc=$?"; tail -3 gpurun_out/gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/ref_bench.json 2> gpurun_out/ref_bench.err; echo "ref rc=$?"
