#!/bin/bash
# Final numbers of the session: C2 (default, --optimizer adam, --agg mean), C3, launch list of C2.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2604_04736_b200.build > gpurun_out/build.log 2>&1
timeout 600 python bench.py > gpurun_out/final_C2.log 2>&1
timeout 300 python bench.py --optimizer adam --no-cpu-baseline > gpurun_out/final_C2_adam.log 2>&1
timeout 300 python bench.py --agg mean --no-cpu-baseline > gpurun_out/final_C2_mean.log 2>&1
timeout 600 python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/final_C3.log 2>&1
for f in final_C2 final_C2_adam final_C2_mean final_C3; do
python - gpurun_out/$f.log <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]
print(sys.argv[1], round(d["ms_per_step"], 4), round(d["value"] / 1e6, 3), "M/s e2e", round(d["e2e"]["value"] / 1e6, 3),
      r["kernel"], round(r["frac"], 3), d.get("cpu_baseline", {}).get("value"), d["clocks"])
PY
done
