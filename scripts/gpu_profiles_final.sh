#!/bin/bash
# Round-end evidence: ncu launch lists of the C2 and C3 bench commands, one --set full capture
# of each dominant kernel class, the tcgen05 / TMA microbenchmarks.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2604_04736_b200.build > gpurun_out/build.log 2>&1
for c in C2 C3; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/launches_$c.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:wgrad_tc_kernel" -s 1 -c 1 -o gpurun_out/full_c2_wgrad \
  python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/full_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:conv2_wgrad_kernel" -s 0 -c 1 -o gpurun_out/full_c3_wgrad \
  python bench.py --config C3 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/full_c3.log 2>&1
./scripts/mma_bench > gpurun_out/mma_bench.txt 2>&1
./scripts/tma_test > gpurun_out/tma_test.txt 2>&1
ls -la gpurun_out
