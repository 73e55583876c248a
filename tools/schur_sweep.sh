#!/bin/bash
# usage: tools/schur_sweep.sh CONFIG "V1 V2 ..." -> per Schur-GEMM variant timing
cfg=$1; shift
for v in $1; do
  TFB_SCHUR_CFG=$v python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/sc_${cfg}_${v}.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/sc_${cfg}_${v}.json').read().strip().splitlines()[-1]); c=d['config']; k=d['kernel_ms_per_step']
print('$cfg schur_cfg=$v', 'DoF/s %.3e' % d['value'], 'factor %.2f' % c['factor_ms'], 'schur %.2f' % k.get('large_update_kernel<1> (schur)', 0), 'res %.1e' % c['rel_residual'])" || tail -3 gpurun_out/sc_${cfg}_${v}.json
done
