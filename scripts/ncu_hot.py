"""Top stall-sampled SASS lines of an ncu source-page CSV (ncu -i X --page source --csv --print-source sass)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [dict(zip(h, x)) for x in rows[2:] if len(x) >= len(h) - 1]
k = "Warp Stall Sampling (All Samples)"
val = lambda x: int(x.get(k, "0").replace(",", "") or 0)
tot = sum(val(x) for x in data)
for x in sorted(data, key=lambda x: -val(x))[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{val(x):7d} {100 * val(x) / max(tot, 1):5.1f}%  {x['Address'][-5:]}  {x['Source'].strip()[:100]}")
print("total samples", tot)
