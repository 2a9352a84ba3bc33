#!/bin/bash
# C3 iteration: CNN GPU tests (unless SKIPT=1), C3 bench summary.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2604_04736_b200.build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
if [ -z "$SKIPT" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "cnn" > gpurun_out/pt_cnn.log 2>&1
  tail -1 gpurun_out/pt_cnn.log
fi
timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C3.log 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_C3.log").read().strip().splitlines()[-1])
print("C3 ms/step", round(d["ms_per_step"], 4), {k: round(v, 4) for k, v in d["kernel_ms_per_step"].items()}, "frac", round(d["roofline"]["frac"], 3))
PY
