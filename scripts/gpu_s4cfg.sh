#!/bin/bash
# the other configs' bench lines (C1, C4, C5, C6) on the current build
cd "$(dirname "$0")/.."
O=gpurun_out/s4/cfg; mkdir -p $O
python -m paper_2604_04736_b200.build > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
for c in C4 C5 C1 C6; do
  timeout 900 python bench.py --config $c --gpus 1 --steps 10 --warmup 3 > $O/bench_$c.log 2>&1; echo "$c rc=$?"
  grep -o '"ms_per_step": [0-9.]*' $O/bench_$c.log | head -1
done
