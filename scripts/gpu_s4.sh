#!/bin/bash
# Session-4 check: GPU tests, default bench (C3), launch list, ncu --set full of the stem conv
# forward and a stage-1 halo forward.
cd "$(dirname "$0")/.."
O=gpurun_out/s4/${1:-a}; mkdir -p $O
python -m paper_2604_04736_b200.build > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --gpus 1 --steps 30 --warmup 5 > $O/bench_default.log 2>&1; echo "bench rc=$?"
tail -c 1500 $O/bench_default.log
B1="python bench.py --config C3 --steps 1 --warmup 1 --profile-run"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:conv3_kernel<.int.0, .bool.0>" -s 0 -c 1 -o $O/full_stem $B1 > $O/ncu_stem.log 2>&1; echo "ncu stem rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:conv3_kernel<.int.0, .bool.1>" -s 0 -c 1 -o $O/full_s1fwd $B1 > $O/ncu_s1fwd.log 2>&1; echo "ncu s1fwd rc=$?"
