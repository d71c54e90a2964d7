#!/bin/bash
# round-2 evidence refresh: the default bench line, then the c5 chain launch list + full capture
NOX="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-model --no-expansion --no-point-prefill --no-prefill --no-shares --no-c5"
M="--clock-control none"
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
echo "bench rc=$?"
C5C="python bench.py --config c5c --queries 8 $NOX"
$C5C > gpurun_out/plain_c5c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum $M -c 300 --csv --log-file gpurun_out/launches_c5c.csv $C5C > gpurun_out/ncu_l3.log 2>&1 && \
  ncu --set full $M --import-source on -k regex:split_t -s 40 -c 2 -o gpurun_out/prof_c5c $C5C > gpurun_out/ncu_f3.log 2>&1
echo "c5c rc=$?"
for r in gpurun_out/prof_c5c; do
  ncu -i $r.ncu-rep --page raw --csv > ${r}_raw.csv; ncu -i $r.ncu-rep --page details --csv > ${r}_details.csv
done
