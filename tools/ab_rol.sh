#!/bin/bash
# same-box A/B of rows-on-lanes kernel variants: prefill (64 queries) + c5 chain + c5 wide
# usage: tools/ab_rol.sh rounds lib1 lib2 ...   (names under paper_2510_24390_b200/, without .so)
P=paper_2510_24390_b200
R=$1; shift
NOX="--no-cpu-baseline --no-prefill --no-e2e --no-model --no-expansion --no-point-prefill --no-shares --no-c5"
for r in $(seq 1 $R); do
for L in "$@"; do
  F=$P/$L.so
  echo -n "$L "; ORION_LIB=$F timeout 300 python tools/prefill_probe.py 64 2>&1 | tail -1
  for c in c5c c5w; do
  ORION_LIB=$F timeout 300 python bench.py --config $c --queries 8 --steps 10 --warmup 3 $NOX > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);r=d['roofline']
print('   $c', round(d['value']), 'split_us', round(r['split_ms_per_launch']*1e3,1), 'mhz', d['clocks']['sm_mhz'])"
  done
done; done
