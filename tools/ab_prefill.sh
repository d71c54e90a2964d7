#!/bin/bash
# same-box A/B of the point prefill between two library builds: tools/ab_prefill.sh libA libB [queries] [rounds]
A=$1; B=$2; NQ=${3:-16}; R=${4:-3}
for i in $(seq 1 $R); do
  for L in $A $B; do
    echo -n "$(basename $L) "; ORION_LIB=$L timeout 300 python tools/prefill_probe.py $NQ 2>&1 | tail -1
  done
done
