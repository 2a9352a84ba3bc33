#!/bin/bash
# ncu --set full of the conv64 kernels (the slower launch of each pair)
cd "$(dirname "$0")/.."
O=gpurun_out/s4/${1:-c}; mkdir -p $O
python -m paper_2604_04736_b200.build > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
B1="python bench.py --config C3 --steps 1 --warmup 1 --profile-run"
for m in 0 1; do
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:conv64_kernel<.int.$m>" -s 1 -c 1 -o $O/full_c64_$m $B1 > $O/ncu_c64_$m.log 2>&1; echo "ncu $m rc=$?"
done
