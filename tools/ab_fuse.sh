#!/bin/bash
# same-box A/B: region A through orion_expand_step (fused append) vs the three calls
NOX="--no-cpu-baseline --no-prefill --no-e2e --no-model --no-expansion --no-point-prefill --no-shares --no-c5"
for r in 1 2 3; do
  for U in "" "--unfused"; do
    for spec in "c4" "c4 --queries 8" "c4 --queries 2"; do
      timeout 300 python bench.py --config $spec --steps 10 --warmup 3 $NOX $U > gpurun_out/ab.json 2>/dev/null
      python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('${U:-fused}', '$spec', round(d['value']), round(d['ms_per_step'],3), d['gpu_launches'])"
    done
  done
done
