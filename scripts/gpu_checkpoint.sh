#!/bin/bash
# Checkpoint of what the driver runs at round end: the full GPU test suite, smoke(), the default
# bench line (C3) and the reference arm. Logs under gpurun_out/ckpt/.
cd "$(dirname "$0")/.."
O=gpurun_out/ckpt; mkdir -p $O
python -m paper_2604_04736_b200.build > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -x --no-header -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/ckpt/bench_default.json", "gpurun_out/ckpt/bench_ref.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, round(d["ms_per_step"], 3), d["value"], d.get("e2e"), d.get("roofline", {}).get("frac"), d.get("clocks", {}).get("reasons"))
PY
