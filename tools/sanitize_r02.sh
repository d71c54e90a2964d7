#!/bin/bash
# compute-sanitizer on the smoke invocation (tiny c1 shapes): memcheck, racecheck, synccheck
for t in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $t --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_$t.log 2>&1
  echo "$t rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|smoke ok|not supported|Error" gpurun_out/san_$t.log | head -5
done
