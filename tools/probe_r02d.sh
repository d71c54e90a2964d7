#!/bin/bash
# prefill item order A/B + graph-decode expansion tests + c2 expansion leg + prefill DRAM capture
P=paper_2510_24390_b200
bash tools/ab_prefill.sh $P/liborion_prev.so $P/liborion.so 16 2
bash tools/ab_prefill.sh $P/liborion_prev.so $P/liborion.so 64 2
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_expansion.py -x -q > gpurun_out/t_pe.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/t_pe.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-prefill --no-e2e --no-model --no-point-prefill --no-shares --no-c5 > gpurun_out/exp.json 2> gpurun_out/exp.err
echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/exp.json').read().strip().splitlines()[-1])
e=d['expansion_run']; print('c4 exp', round(e['value']), e['graph_captures'], round(e['us_per_round'],1))
c=d['expansion_run_c2']
for k in ('eager','graph'): print('c2', k, round(c[k]['value']), round(c[k]['us_per_round'],1), c[k]['rounds'])
print('speedup', round(c['graph_speedup'],2))
PY
ncu --set full --clock-control none -k regex:split_tc -s 2 -c 1 -o gpurun_out/prof_pf2 python tools/prefill_probe.py 16 > gpurun_out/ncu_pf2.log 2>&1
ncu -i gpurun_out/prof_pf2.ncu-rep --page raw --csv > gpurun_out/prof_pf2_raw.csv
echo "ncu rc=$?"
