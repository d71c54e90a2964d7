#!/bin/bash
NOX="--no-cpu-baseline --no-prefill --no-e2e --no-model --no-expansion --no-point-prefill"
for c in c5w c5c; do
  timeout 300 python bench.py --config $c --queries 8 --steps 10 --warmup 3 --kernel rol $NOX > gpurun_out/pb_rol_$c.json 2> gpurun_out/pb_rol_$c.err
done
timeout 300 python bench.py --steps 10 --warmup 3 --kernel rol $NOX > gpurun_out/pb_rol_c4.json 2> gpurun_out/pb_rol_c4.err
