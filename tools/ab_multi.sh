#!/bin/bash
# interleaved same-box A/B of several library builds on c4, c4 8-query share, c5 wide/chain, prefill
# usage: tools/ab_multi.sh rounds lib1 lib2 ...   (names under paper_2510_24390_b200/, without .so)
P=paper_2510_24390_b200
R=$1; shift
LIBS="$@"
NOX="--no-cpu-baseline --no-prefill --no-e2e --no-model --no-expansion --no-point-prefill --no-shares --no-c5"
run() {   # lib config extra...
  local F=$1 c=$2; shift 2
  ORION_LIB=$F timeout 300 python bench.py --config $c "$@" --steps 10 --warmup 3 $NOX > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);r=d['roofline']
print(f\"{round(d['value']/1e3,2)}k/{round(r['split_ms_per_launch']*1e3,1)}us\")" 2>/dev/null || echo "FAIL($(tail -1 gpurun_out/ab.err))"
}
for r in $(seq 1 $R); do
for L in $LIBS; do
  F=$P/$L.so
  a=$(run $F c4); b=$(run $F c4 --queries 8); c=$(run $F c5w --queries 8); d=$(run $F c5c --queries 8)
  pf=$(ORION_LIB=$F timeout 300 python tools/prefill_probe.py 64 2>&1 | tail -1 | grep -o "[0-9.]* ms")
  echo "$L | c4 $a | c4q8 $b | c5w $c | c5c $d | prefill $pf"
done; done
