#!/bin/bash
# ncu --set full of Schur launches on cfg5: L17 (index 7) and the first two L22 chunks (20, 21)
mkdir -p gpurun_out
for i in 7 20 21; do
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:'large_update_kernel<.int.1,' --launch-skip $i --launch-count 1 -o gpurun_out/schur_$i -f \
    python bench.py --config cfg5 --steps 1 --warmup 0 --no-cpu-baseline --no-graph \
    > gpurun_out/ncu_schur_$i.log 2>&1
echo "ncu $i rc=$?"
done
