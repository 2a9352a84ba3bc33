#!/bin/bash
# ViT BF16 iteration: ViT GPU tests, a C7 BF16 bench line, and (NCU=1) the launch list of one step.
cd "$(dirname "$0")/.."
O=gpurun_out/r02; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k vit --no-header -p no:cacheprovider 2>&1 | tail -2
timeout 300 python bench.py --config C7 --precision bf16 --steps 20 --warmup 5 --no-cpu-baseline > $O/b7.log 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02/b7.log").read().strip().splitlines()[-1])
print(round(d["ms_per_step"], 3), {k: round(v, 3) for k, v in d["kernel_ms_per_step"].items()}, "frac", round(d["roofline"]["frac"], 3))
PY
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C7_iter.csv \
    python bench.py --config C7 --precision bf16 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  python scripts/launch_list.py $O/launches_C7_iter.csv 0 2>&1 | head -20
fi
