#!/bin/bash
# usage: tools/solve_sweep.sh "CFG1;CFG2;..." (TFB_SOLVE_CFG strings) -> small-level solve times
IFS=';' read -ra CFGS <<< "$1"
for c in "${CFGS[@]}"; do
  TFB_SOLVE_CFG="$c" timeout 300 python tools/level_timing.py --shape 4096,4096 --reps 2 > gpurun_out/ssv.txt 2>&1
  echo "$c $(grep -o '^  L [0-9] fwd.*' gpurun_out/ssv.txt | awk '{print $4"/"$6}' | tr '\n' ' ')"
done
