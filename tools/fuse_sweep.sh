#!/bin/bash
cfg=$1; shift
for fl in $1; do
  TFB_FUSE_LEVELS=$fl python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/fz_${cfg}_${fl}.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/fz_${cfg}_${fl}.json').read().strip().splitlines()[-1]); c=d['config']
print('$cfg fuse=$fl', 'DoF/s %.3e' % d['value'], 'factor %.2f solve %.2f' % (c['factor_ms'], c['solve_ms'])); print(' ', d['level_ms'][:10])" || tail -3 gpurun_out/fz_${cfg}_${fl}.json
done
