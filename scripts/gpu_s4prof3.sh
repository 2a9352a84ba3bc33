#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/s4/prof3; mkdir -p $O
BNN_NVCC_FLAGS=-DC3_PROF python -m paper_2604_04736_b200.build --force > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 300 python bench.py --gpus 1 --steps 1 --warmup 3 > $O/out.log 2>&1; echo rc=$?
grep "c3<" $O/out.log | tail -48
