#!/bin/bash
# ncu launch list of the bench command + full captures of the sampled-GEMM kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
B1="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_gemm -s 1 -c 1 \
    -o gpurun_out/prof_fwd $B1 > gpurun_out/ncu_fwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_gemm -s 4 -c 1 \
    -o gpurun_out/prof_dgrad $B1 > gpurun_out/ncu_dgrad.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wgrad_tc -s 0 -c 1 \
    -o gpurun_out/prof_wgrad $B1 > gpurun_out/ncu_wgrad.log 2>&1
ls -la gpurun_out
