#!/bin/bash
# usage: tools/small_sweep.sh "CFG1;CFG2;..."  (TFB_SMALL_CFG strings) -> level times of levels 0-9
IFS=';' read -ra CFGS <<< "$1"
for c in "${CFGS[@]}"; do
  TFB_SMALL_CFG="$c" timeout 300 python tools/level_timing.py --shape 4096,4096 --reps 2 > gpurun_out/ss.txt 2>&1
  echo "$c $(grep -o '^L [0-9] .*t= *[0-9.]*ms' gpurun_out/ss.txt | awk '{print $NF}' | tr '\n' ' ')"
done
