#!/bin/bash
# interleaved same-box A/B of two library builds on a config: tools/ab_r02.sh libA libB config [rounds] [extra args]
A=$1; B=$2; CFG=$3; R=${4:-3}; shift 4
NOX="--no-cpu-baseline --no-prefill --no-e2e --no-model --no-expansion --no-point-prefill --no-shares --no-c5"
for i in $(seq 1 $R); do
  for L in $A $B; do
    ORION_LIB=$L timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 $NOX "$@" > gpurun_out/ab.json 2>/dev/null
    python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);r=d['roofline']
print('$L'.split('/')[-1], '$CFG', round(d['value']), round(d['ms_per_step'],3), 'split_us', round(r['split_ms_per_launch']*1e3,1), 'mhz', d['clocks']['sm_mhz'])"
  done
done
