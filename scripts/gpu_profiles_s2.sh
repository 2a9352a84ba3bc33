#!/bin/bash
# Evidence refresh: launch lists with DRAM bytes (C2, C3), per-class traffic, one --set full
# capture of the dominant class of each (C2 forward layer 2, C3 stage-1 conv3 dgrad),
# exported to CSV on the box.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2604_04736_b200.build > gpurun_out/build.log 2>&1
for c in C3 C2; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/traffic_$c.csv \
    python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/traffic_$c.log 2>&1
done
python scripts/traffic_summary.py gpurun_out/traffic_C3.csv gpurun_out/traffic_C2.csv > gpurun_out/traffic_summary.txt 2>&1
KREGEX="gen_gemm_kernel<.int.0, .int.2" CFG=C2 SKIP=1 TAG=full_c2_fwd bash scripts/gpu_prof_one.sh
KREGEX="conv3_kernel<.int.1" CFG=C3 SKIP=6 TAG=full_c3_dgrad bash scripts/gpu_prof_one.sh
python scripts/eps_rate.py > gpurun_out/eps_rate.txt 2>&1
ls -la gpurun_out
KREGEX="wgrad_tc_kernel" CFG=C2 SKIP=1 TAG=full_c2_wgrad bash scripts/gpu_prof_one.sh
timeout 300 python bench.py --config C1 --precision fp32 --agg gnll --no-cpu-baseline > gpurun_out/bench_C1_gnll.log 2>&1
