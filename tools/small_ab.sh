#!/bin/bash
# cfg5 (1 RHS) and cfg3 (64 RHS) per-level factor / solve times of the small levels
python tools/level_timing.py --shape 4096,4096 --reps 3 > gpurun_out/sab5.txt 2>&1
grep "^L [0-9] \|factor total\|solve nrhs=1 " gpurun_out/sab5.txt | awk '{print $1,$2,$(NF-4)}' | tr '\n' ' '; echo
grep -A10 "solve nrhs=1 fwd" gpurun_out/sab5.txt | head -11 | tr '\n' ' '; echo
python tools/level_timing.py --nrhs 64 --reps 3 > gpurun_out/sab3.txt 2>&1
grep -A10 "solve nrhs=64 fwd" gpurun_out/sab3.txt | head -11 | tr '\n' ' '; echo
