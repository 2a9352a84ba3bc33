#!/bin/bash
# A/B of a compile-time flag on one box: bench ×2 with the default build, ×2 with $1 in BNN_NVCC_FLAGS
cd "$(dirname "$0")/.."
O=gpurun_out/s4/flag; mkdir -p $O
for rep in 1 2; do
for f in "" "$1"; do
  BNN_NVCC_FLAGS="$f" python -m paper_2604_04736_b200.build --force > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
  timeout 300 python bench.py --gpus 1 --steps 40 --warmup 5 > $O/b.log 2>&1
  echo "[$f] rep $rep: $(grep -o '"ms_per_step": [0-9.]*' $O/b.log | head -1)"
done
done
