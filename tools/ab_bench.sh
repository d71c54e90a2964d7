#!/bin/bash
# Interleaved A/B of two builds of the library on the default bench (power-cap clock drift makes
# back-to-back single runs differ by +-2%).  Usage: tools/ab_bench.sh libA.so libB.so [rounds] [extra bench args]
A=$1; B=$2; R=${3:-3}; shift 3
for i in $(seq 1 $R); do
  for L in $A $B; do
    ORION_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-prefill --no-e2e "$@" > gpurun_out/ab.log 2>&1
    python -c "
import json,sys;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);r=d['roofline']
print('$L'.split('/')[-1], round(d['value']), round(d['ms_per_step'],3), 'split_ms', round(r['split_ms_per_launch'],4), 'share', round(r['split_share_of_step'],4), 'mhz', d['clocks']['sm_mhz'])"
  done
done
