#!/bin/bash
# DRAM bytes per launch (ncu, replayed per kernel) for the C2 and C3 bench steps.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in C3 C2; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/traffic_$c.csv \
    python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/traffic_$c.log 2>&1
done
