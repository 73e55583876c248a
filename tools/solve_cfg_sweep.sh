#!/bin/bash
# single-RHS small-level solve configs (TFB_SOLVE_CFG: G:GPC per class m<=12,24,48,96,256,rest)
for c in "1:128,2:64,4:64,8:32,32:8,128:2" "2:64,2:64,4:64,8:32,32:8,128:2" "1:128,4:32,4:64,8:32,32:8,128:2" \
         "1:128,2:64,8:32,8:32,32:8,128:2" "1:128,2:64,4:64,16:16,32:8,128:2" "1:256,2:128,4:64,8:32,32:8,128:2"; do
  TFB_SOLVE_CFG=$c python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sc.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sc.json')); k=d['kernel_ms_per_step']
print('$c', round(d['ms_per_step'],3), 'solve', round(d['config']['solve_ms'],3), 'fwd_small', k.get('solve_fwd_small'), 'bwd_small', k.get('solve_bwd_small'))"
done
