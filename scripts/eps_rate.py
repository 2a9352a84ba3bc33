import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
"""Standalone EPS-v1 generator throughput (bnn_eps_bench: normals generated and summed,
no stores): the measured ALU roofline of the ε regeneration (SURVEY §8(d))."""
import json
import torch
from paper_2604_04736_b200 import native

sink = torch.zeros(148 * 64, device="cuda")
n4 = 1 << 28  # 2^30 normals
res = {}
for grid in (148 * 4, 148 * 8, 148 * 16, 148 * 32):
    for _ in range(2):
        native.eps_bench(n4, 1, sink, grid)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        native.eps_bench(n4, 1, sink, grid)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    res[grid] = 4 * n4 / ms / 1e6  # Gnormal/s
    print(f"grid {grid}: {ms:.3f} ms  {res[grid]:.1f} Gnormal/s")
print(json.dumps({"eps_bench_gnormal_per_s": max(res.values())}))
