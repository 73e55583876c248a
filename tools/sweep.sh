#!/bin/bash
# usage: tools/sweep.sh CONFIG "M1 M2 ..."  -> one summary line per small-front limit
cfg=$1; shift
for sm in $1; do
  python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --small-max-m $sm > gpurun_out/sw_${cfg}_${sm}.json 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/sw_${cfg}_${sm}.json').read().strip().splitlines()[-1]); c=d['config']
print('$cfg', 'small<=$sm', 'DoF/s %.3e' % d['value'], 'ms %.2f' % d['ms_per_step'], 'factor %.2f solve %.2f' % (c['factor_ms'], c['solve_ms']), 'res %.1e' % c['rel_residual']); print(' ', d['level_ms'])" || tail -3 gpurun_out/sw_${cfg}_${sm}.json
done
