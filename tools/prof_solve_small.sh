#!/bin/bash
# ncu --set full of the cfg5 single-RHS small-level solve kernels (L2 and L6, both directions)
mkdir -p gpurun_out
for spec in "solve_fwd_small 2" "solve_fwd_small 6" "solve_bwd_small 2"; do
  set -- $spec
ncu --set full --import-source on --clock-control none -k regex:$1 --launch-skip $2 --launch-count 1 \
    -o gpurun_out/$1_$2 -f python bench.py --config cfg5 --steps 1 --warmup 0 --no-cpu-baseline --no-graph \
    > gpurun_out/ncu_$1_$2.log 2>&1
echo "ncu $1 $2 rc=$?"
done
