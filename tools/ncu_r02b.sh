#!/bin/bash
# cfg5 ncu launch list + DRAM traffic at HEAD (into gpurun_out/m3)
O=gpurun_out/m3
mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/cfg5_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_launch.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  --csv --log-file $O/cfg5_traffic.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_traffic.log 2>&1
echo done
