#!/bin/bash
# Iteration helper: CNN GPU tests (unless SKIPT=1) and C3 bench lines (A/B via env in VARIANTS).
cd "$(dirname "$0")/.."
O=gpurun_out/r02; mkdir -p $O
if [ -z "$SKIPT" ]; then
  timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "${TESTK:-cnn}" --no-header -p no:cacheprovider > $O/pt_iter.log 2>&1
  tail -3 $O/pt_iter.log
fi
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then envs=""; else envs="$v"; fi
  env $envs timeout 600 python bench.py --config ${CFG:-C3} --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_iter.log 2>&1
  python - "$v" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/r02/bench_iter.log").read().strip().splitlines()[-1])
print(sys.argv[1], "ms/step", round(d["ms_per_step"], 4), {k: round(v, 3) for k, v in d["kernel_ms_per_step"].items()}, "frac", round(d["roofline"]["frac"], 3), d["roofline"]["kernel"])
PY
done
