#!/bin/bash
# ncu --set full of the stage-1 conv3 halo kernels (fwd, dgrad) of one C3 step.
cd "$(dirname "$0")/.."
O=gpurun_out/r02; mkdir -p $O
B="python bench.py --config C3 --steps 1 --warmup 1 --profile-run"
for k in "conv3_kernel<.int.0, .bool.1>" "conv3_kernel<.int.1, .bool.1>"; do
  n=$(echo "$k" | tr -dc '0-9a-z')
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$k" -c 1 -o $O/prof_$n $B > $O/ncu_$n.log 2>&1
  echo "$k rc=$?"
  ncu -i $O/prof_$n.ncu-rep --page details --csv > $O/prof_${n}_details.csv 2>/dev/null
done
ls -la $O | tail
