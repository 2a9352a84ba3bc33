#!/bin/bash
# ncu launch list of the C3 bench + full captures of the conv kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu_launches_c3.log 2>&1
B1="python bench.py --config C3 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -s 6 -c 1 \
    -o gpurun_out/prof_convfwd $B1 > gpurun_out/ncu_convfwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_wgrad_tc -s 2 -c 1 \
    -o gpurun_out/prof_convwgrad $B1 > gpurun_out/ncu_convwgrad.log 2>&1
ls -la gpurun_out
