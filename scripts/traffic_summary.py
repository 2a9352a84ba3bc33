"""profiles/ncu_traffic.json from the ncu CSVs of scripts/gpu_traffic.sh: DRAM bytes per launch,
averaged over the launches of each kernel class that bench.py's roofline line reports."""
import collections
import csv
import json
import sys

CLASSES = {
    "mlp": {"fwd": ["gen_gemm_kernel<0, 2>", "gen_gemm_kernel<0, 4>"], "dgrad": ["gen_gemm_kernel<1, 2>"],
            "wgrad": ["wgrad_tc_kernel"]},
    "cnn": {"fwd": ["conv2_kernel<0, 1>", "conv2_kernel<0, 2>", "conv3_kernel<0, 0>", "conv3_kernel<0, 1>",
                    "conv64_kernel<0>", "stem_fwd_kernel"],
            "dgrad": ["conv2_kernel<1, 1>", "conv2_kernel<1, 2>", "conv3_kernel<1, 0>", "conv3_kernel<1, 1>",
                      "conv64_kernel<1>"],
            "wgrad": ["conv2_wgrad_kernel<1>", "conv2_wgrad_kernel<2>", "conv64_wgrad_kernel<0>", "conv64_wgrad_kernel<1>",
                      "wgrad_split_reduce4_kernel", "wgrad_eps_combine_kernel", "wgrad_eps_combine_lanes_kernel"]},
}


def per_launch(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    launches = collections.OrderedDict()
    for d in data:
        key = d["ID"]
        name = d["Kernel Name"].split("(")[0].replace("bnn::", "").replace("void ", "")
        unit = d.get("Metric Unit", "")
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
        launches.setdefault(key, {"name": name})[d["Metric Name"]] = v * (scale if "bytes" in d["Metric Name"] else 1)
    return list(launches.values())


out = {}
for kind, path in (("cnn", sys.argv[1]), ("mlp", sys.argv[2])):
    L = per_launch(path)
    for cls, names in CLASSES[kind].items():
        sel = [l for l in L if l["name"] in names]
        if not sel:
            continue
        b = [l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0) for l in sel]
        out[f"{kind}:{cls}"] = int(sum(b) / len(b))
        out[f"{kind}:{cls}_note"] = (f"mean dram__bytes_read.sum + dram__bytes_write.sum over {len(sel)} launches "
                                     f"({', '.join(names)}) of the bench command, ncu --clock-control none")
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
