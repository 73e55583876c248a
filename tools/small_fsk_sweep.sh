#!/bin/bash
# cfg5 per-level factor times for forward-substitution panel thresholds
for k in 16 8 4 2; do
  TFB_SMALL_FSK=$k python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/fsk_$k.json 2>gpurun_out/fsk_$k.err
  python -c "
import json; d=json.load(open('gpurun_out/fsk_$k.json'))
print('fsk=$k', round(d['ms_per_step'],3), 'small L0-9', [round(x,3) for x in d['level_ms'][:10]], round(sum(d['level_ms'][:10]),3), 'solve', round(d['config']['solve_ms'],3))"
done
