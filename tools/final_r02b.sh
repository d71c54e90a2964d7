#!/bin/bash
# round-2 final evidence: default bench line + reference arm, then launch lists and ncu captures
NOX="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-model --no-expansion --no-point-prefill --no-prefill --no-shares --no-c5"
M="--clock-control none"
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/ref_bench.json 2> gpurun_out/ref_bench.err; echo "ref rc=$?"
cap() {   # name, command, kernel regex, count
  local name=$1 cmd=$2 kre=$3 cnt=$4
  $cmd > gpurun_out/plain_$name.log 2>&1 || { echo "$name plain failed"; return; }
  ncu --metrics gpu__time_duration.sum $M -c 300 --csv --log-file gpurun_out/launches_$name.csv $cmd > gpurun_out/ncu_l_$name.log 2>&1
  ncu --set full $M --import-source on -k regex:$kre -s 40 -c $cnt -o gpurun_out/prof_$name $cmd > gpurun_out/ncu_f_$name.log 2>&1
  ncu -i gpurun_out/prof_$name.ncu-rep --page raw --csv > gpurun_out/prof_${name}_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_$name.ncu-rep --page details --csv > gpurun_out/prof_${name}_details.csv 2>/dev/null
  echo "$name captured"
}
cap c4 "python bench.py $NOX" "split_tct|combine16" 2
cap c4_8q "python bench.py --queries 8 $NOX" "split_tct" 1
cap c5w "python bench.py --config c5w --queries 8 $NOX" "split_t" 2
cap c5c "python bench.py --config c5c --queries 8 $NOX" "split_t" 2
python tools/prefill_probe.py 64 > gpurun_out/plain_pf.log 2>&1 && \
  ncu --set full $M --import-source on -k regex:split_tc -s 2 -c 1 -o gpurun_out/prof_prefill python tools/prefill_probe.py 64 > gpurun_out/ncu_f_pf.log 2>&1 && \
  ncu -i gpurun_out/prof_prefill.ncu-rep --page raw --csv > gpurun_out/prof_prefill_raw.csv && \
  ncu -i gpurun_out/prof_prefill.ncu-rep --page details --csv > gpurun_out/prof_prefill_details.csv && echo "prefill captured"
