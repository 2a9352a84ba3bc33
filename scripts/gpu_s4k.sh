#!/bin/bash
# A/B of an experiment switch: bench + launch list with and without
cd "$(dirname "$0")/.."
O=gpurun_out/s4/${1:-k}; mkdir -p $O
python -m paper_2604_04736_b200.build > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
for v in "" "$2"; do
  tag=$(echo "x$v" | tr -dc 'a-zA-Z0-9')
  env $v timeout 300 python bench.py --gpus 1 --steps 30 --warmup 5 > $O/bench_$tag.log 2>&1; echo "[$v] bench rc=$?"; grep -o '"ms_per_step": [0-9.]*' $O/bench_$tag.log | head -1
  env $v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l_$tag.csv python bench.py --config C3 --steps 1 --warmup 1 --profile-run > /dev/null 2>&1
  python scripts/launch_list.py $O/l_$tag.csv 14 2>&1 | grep "$3"
done
