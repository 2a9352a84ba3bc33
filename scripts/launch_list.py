"""Per-kernel launch durations (µs) from an ncu --metrics gpu__time_duration.sum CSV."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
seq = [(d["Kernel Name"].split("(")[0].replace("bnn::", "").replace("void ", ""),
        float(d["Metric Value"].replace(",", "")) / 1e3) for d in data if d["Metric Name"] == "gpu__time_duration.sum"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
tot = collections.defaultdict(float)
for k, v in seq:
    tot[k] += v
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:15]:
    print(f"{v:10.1f} us total  {k}")
for name in sorted({k for k, _ in seq if k.startswith("conv")}):
    print(name, [round(v) for k, v in seq if k == name][:n])
