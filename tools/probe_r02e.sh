#!/bin/bash
# small-step split A/B (c2 running sets, c4 8-query share) + parity of the adaptive plans
P=paper_2510_24390_b200
for nb in 1 2 8; do for L in $P/liborion_prev.so $P/liborion.so; do
  echo "$(basename $L) nb=$nb"; ORION_LIB=$L timeout 120 python tools/graph_probe.py $nb 2>&1 | grep -E "plan|round"
done; done
bash tools/ab_r02.sh $P/liborion_prev.so $P/liborion.so c4 2 --queries 8
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_expansion.py -x -q > gpurun_out/t_small.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/t_small.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-prefill --no-e2e --no-model --no-point-prefill --no-shares --no-c5 > gpurun_out/exp.json 2> gpurun_out/exp.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/exp.json').read().strip().splitlines()[-1])
e=d['expansion_run']; print('c4 exp', round(e['value']), e['graph_captures'], round(e['us_per_round'],1))
c=d['expansion_run_c2']
for k in ('eager','graph'): print('c2', k, round(c[k]['value']), round(c[k]['us_per_round'],1), c[k]['rounds'])
print('speedup', round(c['graph_speedup'],2))
PY
