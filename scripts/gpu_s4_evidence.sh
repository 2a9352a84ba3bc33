#!/bin/bash
# Session-4 evidence: default bench (C3), reference arm, C2 bench, launch lists (C3, C2) with DRAM
# bytes, the ncu traffic summary, ncu --set full of the conv64 kernels.
cd "$(dirname "$0")/.."
O=gpurun_out/s4/ev; mkdir -p $O
python -m paper_2604_04736_b200.build > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 600 python bench.py --gpus 1 --steps 50 --warmup 5 > $O/bench_default.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 3 > $O/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --config C2 --gpus 1 --steps 100 --warmup 5 > $O/bench_C2.log 2>&1; echo "C2 rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in C3 C2; do
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/launches_$c.csv \
      python bench.py --config $c --steps 2 --warmup 1 --profile-run > $O/ncu_$c.log 2>&1
  echo "$c list rc=$?"
done
python scripts/traffic_summary.py $O/launches_C2.csv $O/launches_C3.csv > $O/traffic.json 2> $O/traffic.err; cat $O/traffic.json | head -5
B1="python bench.py --config C3 --steps 1 --warmup 1 --profile-run"
for k in "conv64_kernel<.int.0>" "conv64_kernel<.int.1>" "conv64_wgrad_kernel<.bool.1>" "stem_fwd_kernel" "conv2_kernel<.int.1, .int.2>"; do
  n=$(echo "$k" | tr -dc '0-9a-z')
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$k" -s 1 -c 1 -o $O/full_$n $B1 > $O/ncu_full_$n.log 2>&1
  echo "$k rc=$?"
done
tail -c 400 $O/bench_default.log
