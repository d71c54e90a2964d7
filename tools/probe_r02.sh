#!/bin/bash
# dev probe: correctness under the watchdog build, then the release build, then c5/c4 timings
NOX="--no-cpu-baseline --no-prefill --no-e2e --no-model --no-expansion --no-point-prefill"
ORION_LIB=paper_2510_24390_b200/liborion_check.so timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or shapes or c2 or grid or wide or hybrid" > gpurun_out/p_check.log 2>&1
echo "check rc=$?"; tail -3 gpurun_out/p_check.log
[ "$1" == "quick" ] && exit 0
[ "$1" != "bench" ] && timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_prefill.py -x -q > gpurun_out/p_rel.log 2>&1
[ "$1" != "bench" ] && { echo "release rc=$?"; tail -3 gpurun_out/p_rel.log; }
for c in c5w c5c; do
  timeout 300 python bench.py --config $c --queries 8 --steps 10 --warmup 3 $NOX > gpurun_out/p_$c.json 2> gpurun_out/p_$c.err
done
timeout 300 python bench.py --steps 10 --warmup 3 $NOX > gpurun_out/p_c4.json 2> gpurun_out/p_c4.err
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-prefill --no-e2e --no-model --no-expansion --no-shares --no-c5 --layers 4 > gpurun_out/p_pp.json 2> gpurun_out/p_pp.err
python -c "import json;d=json.loads(open('gpurun_out/p_pp.json').read().strip().splitlines()[-1]);pp=d['point_prefill'];print('prefill ms/layer', round(pp['ms_per_layer'],3), 'frac', round(pp['roofline']['frac'],3))"
for c in c5w c5c; do
  ORION_LIB=paper_2510_24390_b200/liborion_trace.so timeout 300 python bench.py --config $c --queries 8 --layers 2 --steps 1 --warmup 0 $NOX > gpurun_out/p_trace_$c.txt 2>&1
done
