#!/bin/bash
# Round-2 evidence: launch lists (C3, C2, C7) with per-launch DRAM bytes, the ncu traffic summary
# for bench.py's roofline line, ncu --set full of the C3 dgrad kernels, and the default bench.
cd "$(dirname "$0")/.."
O=gpurun_out/r02/ev; mkdir -p $O
python -m paper_2604_04736_b200.build > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in C3 C2 C7; do
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/launches_$c.csv \
      python bench.py --config $c --steps 2 --warmup 1 --profile-run > $O/ncu_$c.log 2>&1
  echo "$c rc=$?"
done
python scripts/traffic_summary.py $O/launches_C2.csv $O/launches_C3.csv > $O/traffic.json 2> $O/traffic.err; cat $O/traffic.json
B1="python bench.py --config C3 --steps 1 --warmup 1 --profile-run"
for k in "conv3_kernel<.int.1, .bool.1>" "conv2_kernel<.int.1>" "conv2_wgrad_kernel"; do
  n=$(echo "$k" | tr -dc '0-9a-z')
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$k" -s 2 -c 1 -o $O/full_$n $B1 > $O/ncu_full_$n.log 2>&1
  echo "$k rc=$?"
  ncu -i $O/full_$n.ncu-rep --page details --csv > $O/full_${n}_details.csv 2>/dev/null
  ncu -i $O/full_$n.ncu-rep --page raw --csv > $O/full_${n}_raw.csv 2>/dev/null
done
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_default.log 2>&1; echo "bench rc=$?"
tail -c 600 $O/bench_default.log
