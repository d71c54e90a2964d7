#!/bin/bash
# FMA-pipe exp2 offload in the rows-on-lanes softmax: prefill + c5 chain A/B over the fraction
P=paper_2510_24390_b200
NOX="--no-cpu-baseline --no-prefill --no-e2e --no-model --no-expansion --no-point-prefill --no-shares --no-c5"
for r in 1 2; do
for L in prev p0 liborion p3 p4; do
  F=$P/liborion_$L.so; [ $L == liborion ] && F=$P/liborion.so
  echo -n "$L "; ORION_LIB=$F timeout 300 python tools/prefill_probe.py 64 2>&1 | tail -1
  ORION_LIB=$F timeout 300 python bench.py --config c5c --queries 8 --steps 10 --warmup 3 $NOX > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);r=d['roofline']
print('   c5c', round(d['value']), 'split_us', round(r['split_ms_per_launch']*1e3,1), 'mhz', d['clocks']['sm_mhz'])"
done; done
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_parity.py -x -q --timeout 400 > gpurun_out/t_poly.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/t_poly.log
