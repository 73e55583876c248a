#!/bin/bash
# A/B of the concurrent top slices: tools/split_sweep.sh CONFIG "H:FRONTS ..." -> ms per step
c=$1; shift
for hf in $@; do
  h=${hf%%:*}; f=${hf##*:}
  TFB_SPLIT_TOP=$h TFB_SPLIT_FRONTS=$f python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ss_$c.json 2> gpurun_out/ss_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/ss_$c.json')); t=d['config'].get('top_slices')
print('$c', '$hf', round(d['ms_per_step'],3), t and t['levels'])" || tail -3 gpurun_out/ss_$c.err
done
