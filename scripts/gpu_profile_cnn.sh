#!/bin/bash
# ncu launch list of the C3 bench + full captures of the conv kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu_launches_c3.log 2>&1
B1="python bench.py --config C3 --steps 1 --warmup 0 --no-cpu-baseline"
for k in ${KERNELS:-conv2_wgrad_kernel:4 conv2_kernel:6}; do
  name=${k%%:*}; skip=${k##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$name -s $skip -c 1 \
      -o gpurun_out/prof_${name}_$skip $B1 > gpurun_out/ncu_${name}_$skip.log 2>&1
done
ls -la gpurun_out
