#!/bin/bash
# ncu evidence for profiles/r02: launch lists (device time per launch, cold + serialised) and one
# `--set full` capture per top kernel, each after the same command exited 0 without ncu.
NOX="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-model --no-expansion --no-point-prefill --no-prefill --no-shares --no-c5"
C4="python bench.py $NOX"
C5W="python bench.py --config c5w --queries 8 $NOX"
C5C="python bench.py --config c5c --queries 8 $NOX"
C4S="python bench.py --queries 8 $NOX"
PP="python tools/prefill_probe.py 16"
M="--clock-control none"
$C4 > gpurun_out/plain_c4.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum $M -c 300 --csv --log-file gpurun_out/launches_c4.csv $C4 > gpurun_out/ncu_l1.log 2>&1 && \
  ncu --set full $M --import-source on -k regex:split_tct -s 40 -c 1 -o gpurun_out/prof_c4_tct $C4 > gpurun_out/ncu_f1.log 2>&1
echo "c4 rc=$?"
$C5W > gpurun_out/plain_c5w.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum $M -c 300 --csv --log-file gpurun_out/launches_c5w.csv $C5W > gpurun_out/ncu_l2.log 2>&1 && \
  ncu --set full $M --import-source on -k regex:split_t -s 40 -c 2 -o gpurun_out/prof_c5w $C5W > gpurun_out/ncu_f2.log 2>&1
echo "c5w rc=$?"
$C5C > gpurun_out/plain_c5c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum $M -c 300 --csv --log-file gpurun_out/launches_c5c.csv $C5C > gpurun_out/ncu_l3.log 2>&1 && \
  ncu --set full $M --import-source on -k regex:split_t -s 40 -c 2 -o gpurun_out/prof_c5c $C5C > gpurun_out/ncu_f3.log 2>&1
echo "c5c rc=$?"
$C4S > gpurun_out/plain_c4s.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum $M -c 300 --csv --log-file gpurun_out/launches_c4_8q.csv $C4S > gpurun_out/ncu_l4.log 2>&1
echo "c4 8q rc=$?"
$PP > gpurun_out/plain_pp.log 2>&1 && \
  ncu --set full $M --import-source on -k regex:split_tc -s 2 -c 1 -o gpurun_out/prof_prefill $PP > gpurun_out/ncu_f5.log 2>&1
echo "prefill rc=$?"
ls -la gpurun_out/*.ncu-rep
