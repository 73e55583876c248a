#!/bin/bash
# A/B of an environment knob on the bench: tools/ab_env.sh CONFIG VAR v1 v2 ...
cfg=$1; var=$2; shift 2
for v in "$@"; do
  env $var=$v python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${var}_$v.json 2>gpurun_out/ab_${var}_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_${var}_$v.json'))
print('$var=$v', round(d['ms_per_step'],3), 'eager', round(d['config']['eager_ms_per_step'],3), 'levels', [round(x,2) for x in d['level_ms']], 'solve', round(d['config']['solve_ms'],3))" || tail -5 gpurun_out/ab_${var}_$v.err
done
