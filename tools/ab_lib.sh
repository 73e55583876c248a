#!/bin/bash
# A/B of two builds of the library: tools/ab_lib.sh CONFIG LIB1 LIB2 ...
cfg=$1; shift
i=0
for lib in "$@"; do
  i=$((i+1))
  TFB_LIB=$(realpath $lib) python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ablib_$i.json 2>gpurun_out/ablib_$i.err
  python -c "
import json; d=json.load(open('gpurun_out/ablib_$i.json'))
print('$lib', round(d['ms_per_step'],3), 'levels', [round(x,2) for x in d['level_ms']], 'solve', round(d['config']['solve_ms'],3), 'schur', d['kernel_ms_per_step'].get('large_update_kernel<1> (schur)'))" || tail -3 gpurun_out/ablib_$i.err
done
