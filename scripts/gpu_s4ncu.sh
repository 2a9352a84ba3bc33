#!/bin/bash
# End-of-round ncu --set full captures of the C3 step's top kernels (one launch each), exported
# as raw CSV for scripts/ncu_summary.py
cd "$(dirname "$0")/.."
O=gpurun_out/s4/ncu; mkdir -p $O
python -m paper_2604_04736_b200.build > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
B1="python bench.py --config C3 --steps 1 --warmup 1 --profile-run"
i=0
# pattern|launches to skip (conv3<1,0>: the 7th of a step is the stride-2 dgrad into 64 channels)
for ks in "conv64_kernel<.int.0>|1" "conv64_kernel<.int.1>|1" "conv64_wgrad_kernel<.bool.1>|1" "stem_fwd_kernel|0" \
          "conv3_kernel<.int.1, .bool.0>|6" "conv2_wgrad_kernel<.int.1>|4" "conv2_kernel<.int.1, .int.2>|1" "conv2_kernel<.int.0, .int.1>|2"; do
  i=$((i+1)); k=${ks%|*}; sk=${ks#*|}
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
     -k "regex:$k" -s $sk -c 1 -o $O/full_$i $B1 > $O/ncu_$i.log 2>&1; echo "ncu $i ($k) rc=$?"
  ncu -i $O/full_$i.ncu-rep --page raw --csv > $O/full_$i.csv 2>/dev/null
done
