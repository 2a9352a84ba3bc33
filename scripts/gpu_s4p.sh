#!/bin/bash
# perf-only iteration: C3 bench + launch list of the conv64 kernels
cd "$(dirname "$0")/.."
O=gpurun_out/s4/${1:-p}; mkdir -p $O
python -m paper_2604_04736_b200.build > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 300 python bench.py --gpus 1 --steps 30 --warmup 5 > $O/bench.log 2>&1; echo "bench rc=$?"; grep -o '"ms_per_step": [0-9.]*' $O/bench.log | head -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3.csv python bench.py --config C3 --steps 1 --warmup 1 --profile-run > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
python scripts/launch_list.py $O/launches_C3.csv 8 2>&1 | grep "conv64\|conv3_kernel<0"
