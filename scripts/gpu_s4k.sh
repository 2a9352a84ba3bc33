#!/bin/bash
# A/B/… of experiment switches on one box: bench (+ launch list of kernels matching $2) per variant
# usage: gpu_s4k.sh TAG PATTERN "VAR=x" "VAR=y" …   ("" = defaults)
cd "$(dirname "$0")/.."
O=gpurun_out/s4/${1:-k}; mkdir -p $O; pat=$2; shift 2
python -m paper_2604_04736_b200.build > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
for rep in 1 2; do
for v in "$@"; do
  tag=$(echo "x$v" | tr -dc 'a-zA-Z0-9')
  env $v timeout 300 python bench.py --gpus 1 --steps 40 --warmup 5 > $O/bench_${tag}_$rep.log 2>&1
  echo "[$v] rep $rep: $(grep -o '"ms_per_step": [0-9.]*' $O/bench_${tag}_$rep.log | head -1)"
done
done
for v in "$@"; do
  tag=$(echo "x$v" | tr -dc 'a-zA-Z0-9')
  [ -z "$pat" ] && continue
  env $v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l_$tag.csv python bench.py --config C3 --steps 1 --warmup 1 --profile-run > /dev/null 2>&1
  echo "[$v]"; python scripts/launch_list.py $O/l_$tag.csv 14 2>&1 | grep "$pat"
done
