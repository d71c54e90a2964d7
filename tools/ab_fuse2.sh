#!/bin/bash
# same-box A/B: default fuse threshold vs fusing every step (liborion_fall.so)
P=paper_2510_24390_b200
NOX="--no-cpu-baseline --no-prefill --no-e2e --no-model --no-expansion --no-point-prefill --no-shares --no-c5"
for r in 1 2; do
  for L in liborion liborion_fall; do
    for q in 4 8 16 64; do
      ORION_LIB=$P/$L.so timeout 300 python bench.py --queries $q --steps 10 --warmup 3 $NOX > gpurun_out/ab.json 2>/dev/null
      python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$L', 'q=$q', round(d['value']), d['gpu_launches'])"
    done
  done
done
