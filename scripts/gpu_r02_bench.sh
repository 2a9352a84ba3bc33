#!/bin/bash
# Round 2: the driver's bench commands (default = C3), the reference arm, C2, and the ncu
# launch list of the C3 step. Logs under gpurun_out/r02/.
cd "$(dirname "$0")/.."
O=gpurun_out/r02; mkdir -p $O
python -m paper_2604_04736_b200.build > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_default.log 2>&1; echo "default rc=$?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --config C2 --steps 100 --warmup 10 --no-cpu-baseline > $O/bench_C2.log 2>&1; echo "C2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_C3.csv python bench.py --config C3 --steps 2 --warmup 1 --profile-run > $O/ncu_launches.log 2>&1
echo "ncu rc=$?"
for f in $O/bench_*.log; do echo "== $f"; tail -c 1500 $f; echo; done
