#!/bin/bash
# conv64 check: CNN BF16 parity tests, conv64 vs conv3 A/B, bench C3 with and without, launch list.
cd "$(dirname "$0")/.."
O=gpurun_out/s4/${1:-b}; mkdir -p $O
python -m paper_2604_04736_b200.build > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cnn or conv64 or eps_fused or stem or session4" > $O/pytest_cnn.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest_cnn.log
timeout 300 python bench.py --gpus 1 --steps 30 --warmup 5 > $O/bench_c64.log 2>&1; echo "bench rc=$?"; grep -o '"ms_per_step": [0-9.]*' $O/bench_c64.log | head -1; grep -o '"kernel_ms_per_step": {[^}]*}' $O/bench_c64.log
BNN_CONV64=0 timeout 300 python bench.py --gpus 1 --steps 30 --warmup 5 > $O/bench_c3.log 2>&1; echo "bench c3 rc=$?"; grep -o '"ms_per_step": [0-9.]*' $O/bench_c3.log | head -1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_C3.csv python bench.py --config C3 --steps 2 --warmup 1 --profile-run > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
python scripts/launch_list.py $O/launches_C3.csv 12 2>&1 | head -40
