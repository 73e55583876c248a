#!/bin/bash
# Round-2 final measurement set (GPU box): bench lines of every config, the
# reference arm, the cfg5 ncu launch list + DRAM traffic, the full GPU tests.
set -u
O=gpurun_out/m3
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
python bench.py --steps 20 --warmup 3 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_cfg5_reference.json 2> $O/bench_cfg5_reference.err
for c in cfg1 cfg2 cfg3 cfg4 cfg3p2; do
  python bench.py --config $c --steps 20 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
for c in cfg1 cfg2; do
  python bench.py --impl reference --config $c --steps 5 --warmup 1 > $O/bench_${c}_reference.json 2> $O/bench_${c}_reference.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/cfg5_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_launch.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  --csv --log-file $O/cfg5_traffic.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_traffic.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1
echo done
