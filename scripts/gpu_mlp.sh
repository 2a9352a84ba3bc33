#!/bin/bash
# MLP iteration loop: build, MLP GPU parity tests, C2 bench (logs under gpurun_out/).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2604_04736_b200.build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "${PYK:-not cnn}" > gpurun_out/pt_mlp.log 2>&1
tail -2 gpurun_out/pt_mlp.log
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench_C2.log 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_C2.log").read().strip().splitlines()[-1])
print("C2 ms/step", round(d["ms_per_step"], 4), {k: round(v, 4) for k, v in d["kernel_ms_per_step"].items()}, "frac", round(d["roofline"]["frac"], 3))
PY
