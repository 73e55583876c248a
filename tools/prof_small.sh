#!/bin/bash
# ncu source-level capture of factor_small_kernel on cfg5 level $1 (0-based launch index)
L=${1:-8}
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:factor_small_kernel \
    --launch-skip $L --launch-count 1 -o gpurun_out/small_L$L -f \
    python bench.py --config cfg5 --steps 1 --warmup 0 --no-cpu-baseline --no-graph \
    > gpurun_out/ncu_small_L$L.log 2>&1
echo "ncu rc=$?"
