#!/bin/bash
# End-of-session evidence: default bench, C2 and C7 benches, reference arm, C3 launch list.
cd "$(dirname "$0")/.."
O=gpurun_out/s4/final; mkdir -p $O
python -m paper_2604_04736_b200.build > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 600 python bench.py --gpus 1 --steps 50 --warmup 5 > $O/bench_default.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --config C2 --gpus 1 --steps 100 --warmup 5 > $O/bench_C2.log 2>&1; echo "C2 rc=$?"
timeout 600 python bench.py --config C7 --precision bf16 --gpus 1 --steps 30 --warmup 5 > $O/bench_C7.log 2>&1; echo "C7 rc=$?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 3 > $O/bench_ref.log 2>&1; echo "ref rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/launches_C3.csv \
    python bench.py --config C3 --steps 2 --warmup 1 --profile-run > $O/ncu_C3.log 2>&1; echo "list rc=$?"
for f in bench_default bench_C2 bench_C7; do grep -o '"ms_per_step": [0-9.]*' $O/$f.log | head -1; done
