#!/bin/bash
# bench.py line of every config into gpurun_out/m3 (tools/measure_r02b.sh's bench part)
O=gpurun_out/m3
mkdir -p $O
for c in cfg5 cfg1 cfg2 cfg3 cfg4 cfg3p2; do
  python bench.py --config $c --steps 20 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
echo done
