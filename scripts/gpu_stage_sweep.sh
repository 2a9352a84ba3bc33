#!/bin/bash
# tcgen05 issue-rate microbenchmark + conv pipeline-depth sweep on C3.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2604_04736_b200.build > gpurun_out/build.log 2>&1
./scripts/mma_bench > gpurun_out/mma_bench.log 2>&1
for st in 3 4 6 9; do
  BNN_CONV_STAGES=$st timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C3_st$st.log 2>&1
done
cat gpurun_out/mma_bench.log
for st in 3 4 6 9; do python -c "
import json,sys;d=json.loads(open('gpurun_out/bench_C3_st$st.log').readline());print($st, round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['kernel_ms_per_step'].items() if k in ('fwd','dgrad','wgrad')})"; done
