#!/bin/bash
# Interleaved A/B of the C4 on-the-fly K4 (F=640, full grid) between two
# builds: tools/ab_k4.sh libA.so libB.so [rounds]
A=$1; B=$2; R=${3:-3}
for r in $(seq $R); do
  for L in $A $B; do
    echo "$L $(SRPB_LIB=$L timeout 300 python tools/c4_probe.py --frames 640 --conv-cands 0 --reps 2 2>&1 | grep -E 'maps=True' | sed 's/.*J=600000: //')"
  done
done
