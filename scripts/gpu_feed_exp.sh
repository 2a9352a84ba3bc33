#!/bin/bash
# Conv kernel feed-rate experiment: normal / no MMA / no operand loads (results invalid in 1, 2).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2604_04736_b200.build > gpurun_out/build.log 2>&1
for d in 0 1 2 3; do
  BNN_CONV_DEBUG=$d timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/feed_$d.csv python bench.py --config C3 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/feed_$d.log 2>&1
done
for d in 0 1 2 3; do echo "== dbg $d"; python scripts/launch_list.py gpurun_out/feed_$d.csv 22 | grep "^conv"; done
