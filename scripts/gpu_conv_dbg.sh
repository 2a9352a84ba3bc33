#!/bin/bash
# Per-launch µs of the conv kernels of one C3 step under BNN_CONV_DEBUG = 0 (production),
# 1 (no MMAs), 2 (no operand loads), 3 (neither): which part limits each kernel class.
cd "$(dirname "$0")/.."
O=gpurun_out/r02; mkdir -p $O
for d in 0 1 2 3; do
  BNN_CONV_DEBUG=$d timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/dbg$d.csv python bench.py --config C3 --steps 1 --warmup 1 --profile-run > /dev/null 2>&1
done
python - <<'PY'
import csv, collections
def load(p):
    rows = list(csv.reader(open(p)))
    hdr = None; out = []
    for r in rows:
        if "Kernel Name" in r: hdr = r; continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.append((d["Kernel Name"].split("(")[0].replace("void ", "").replace("bnn::", ""), float(d["Metric Value"].replace(",", "")) / 1e3))
    return out
runs = [load(f"gpurun_out/r02/dbg{d}.csv") for d in range(4)]
n = len(runs[0]) // 3  # last of the 3 steps (warm)
for i in range(2 * n, 3 * n):
    name = runs[0][i][0]
    if "conv" in name and "combine" not in name:
        print(f"{name:32s} " + " ".join(f"{r[i][1]:8.1f}" if i < len(r) else "     n/a" for r in runs))
PY
