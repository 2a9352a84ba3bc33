#!/usr/bin/env python
"""bench.py — ELBO-step throughput (sample·images/s) of the sample-sharded BNN step on B200.

Contract (README/DESIGN.md §7): `python bench.py --gpus N --steps K --warmup W` runs the
BASELINE.json workload; for N>1 it is launched under torchrun (one rank per GPU, NCCL).
Rank 0 prints ONE JSON line. A "step" is one pass of the whole hot path (σ prologue,
sampled forward, loss head, sampled backward with sample-accumulating wgrad, allreduce,
finalize + KL) over one synthetic minibatch.

N=1 workload: C2 = Bayesian MLP 784-1024-1024-10, B=256, S=64 (BASELINE.json configs[1]).
For N>1 the run is weak-scaled: S = 64·N samples sharded over N ranks (same batch per rank).

`--impl reference` times the CPU oracle (oracle/, fp64, all host cores) on a bounded sample
of the same workload — the tier's reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2604_04736_b200 import synth  # noqa: E402
from paper_2604_04736_b200.configs import CONFIGS, MODELS, n_params  # noqa: E402

METRIC = "ELBO-step sample·images/s"


def _env_world():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ====================================================================== reference arm
def cpu_oracle_rate(model, B, D, budget_s=15.0, seed=0x5EED):
    """Time the fp64 oracle (as it stands) on the host cores over a bounded sample of the
    workload: all B examples, S_sample samples; returns (sample·images/s, cores, sample)."""
    import oracle as O
    mu, rho = synth.init_params(model, seed=2)
    x, yc, yr = synth.make_batch(model, B, seed=1)
    cores = os.cpu_count() or 1
    O.lib()
    t0 = time.perf_counter()
    O.elbo_partial(model, mu, rho, x, yc, yr, B, 0, 64, 0, 1, seed, 0)
    t1 = time.perf_counter() - t0
    S_sample = max(1, min(64, int(budget_s / max(t1, 1e-3))))
    t0 = time.perf_counter()
    O.elbo_partial(model, mu, rho, x, yc, yr, B, 0, 64, 0, S_sample, seed, 0)
    dt = time.perf_counter() - t0
    return S_sample * B / dt, cores, f"{S_sample} of 64 samples x {B} images (one step's slice), fp64"


def run_reference(args, world, rank):
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    model = MODELS[cfg["model"]]
    B, S = cfg["B"], cfg["S"] * (world if world > 1 else 1)
    rates = []
    for i in range(args.warmup + args.steps):
        r, cores, sample = cpu_oracle_rate(model, B, cfg["D"], budget_s=args.ref_budget)
        if i >= args.warmup:
            rates.append(r)
    v = statistics.median(rates)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "sample·images/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": S * B / v * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: " + cfg["model"], "global_batch": B,
                       "samples": S},
            "cpu_baseline": {"value": v, "unit": "sample·images/s", "cores": cores,
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "sample·images/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ====================================================================== our arm
def run_ours(args, world, rank, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2604_04736_b200 import native

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    uid = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        obj = [native.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    cfg = CONFIGS[args.config]
    model = MODELS[cfg["model"]]
    B = cfg["B"]
    S_loc = cfg["S"]
    S = S_loc * world  # weak scaling: samples proportional to GPUs
    D = cfg["D"]
    P = n_params(model)

    mu_h, rho_h = synth.init_params(model, seed=2)
    x_h, yc_h, yr_h = synth.make_batch(model, B, seed=1)
    mu = torch.from_numpy(mu_h).to(dev)
    rho = torch.from_numpy(rho_h).to(dev)
    x = torch.from_numpy(x_h).to(dev)
    y = torch.from_numpy(yc_h if yc_h is not None else yr_h).to(dev)
    gmu = torch.empty_like(mu)
    grho = torch.empty_like(rho)
    loss_dev = torch.zeros(1, device=dev)
    stream = torch.cuda.current_stream(dev)
    ctx = native.Context(model, precision=args.precision, mode="sample", rank=rank, world=world,
                         uid=uid, max_B_loc=B, max_S_loc=S_loc, dataset_size=D, device=local_rank,
                         stream=stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step(i):
        ctx.elbo_step(mu, rho, x, y, B, S, 0x5EED, i, grad_mu=gmu, grad_rho=grho,
                      loss_dev=loss_dev, want_loss=False)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches0 = ctx.launch_count()
    ctx.profile(True)
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            ev[i][0].record(stream)
            step(args.warmup + i)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile(False)
    launches = ctx.launch_count() - launches0
    if world > 1:
        dist.barrier()
    times = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(times)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = S * B / (ms_per_step / 1e3)

    # ---------------- end to end through the public API with host buffers
    x_pin = torch.from_numpy(x_h).pin_memory()
    y_pin = torch.from_numpy(yc_h if yc_h is not None else yr_h).pin_memory()
    for i in range(2):
        ctx.elbo_step_host(mu, rho, x_pin, y_pin, B, S, 0x5EED, i, grad_mu=gmu, grad_rho=grho)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e_ms = []
    for i in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.elbo_step_host(mu, rho, x_pin, y_pin, B, S, 0x5EED, i, grad_mu=gmu, grad_rho=grho)
        e_ms.append((time.perf_counter() - t0) * 1e3)
    te = torch.tensor([sum(e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = S * B / (float(te.item()) / args.steps / 1e3)

    if rank == 0:
        peaks, peak_src = _peaks()
        line = {"metric": METRIC, "value": value, "unit": "sample·images/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "bf16" if args.precision == "bf16" else "f32", "data": "synthetic",
                "config": {"workload": f"{args.config}: Bayesian MLP 784-1024-1024-10 (CE)",
                           "global_batch": B, "samples": S, "samples_per_gpu": S_loc,
                           "params": P, "parallelism": f"sample-sharded x{world}",
                           "l2": "flushed between timed steps (256 MiB memset outside events)"},
                "clocks": clk.summary(),
                "e2e": {"value": e2e_value, "unit": "sample·images/s",
                        "h2d_bytes_per_step": int(x_pin.numel() * 4 + y_pin.numel() * 4),
                        "d2h_bytes_per_step": 4},
                "gpu_launches": int(launches),
                "kernel_ms_per_step": {k: v["ms"] / args.steps for k, v in prof.items()}}
        line["roofline"] = roofline(model, B, S_loc, prof, args.steps, peaks, peak_src)
        if world == 1 and not args.no_cpu_baseline:
            r, cores, sample = cpu_oracle_rate(model, B, D, budget_s=args.ref_budget)
            line["cpu_baseline"] = {"value": r, "unit": "sample·images/s", "cores": cores,
                                    "kind": "oracle", "sample": sample}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def roofline(model, B, S_loc, prof, steps, peaks, peak_src):
    """Dominant kernel class vs its bound.

    The sampled-GEMM kernels are ALU-bound by ε regeneration; their unit is
    ε normals generated, and the peak is the issue-slot ceiling derived in DESIGN.md §4:
    148 SMs × 128 lanes × f_clk / (instructions per normal)."""
    w = model["widths"]
    layers = [(w[i + 1], w[i]) for i in range(len(w) - 1)]
    nrm_fwd = S_loc * sum(n * k + n for n, k in layers)          # fwd generates every W_s and b_s
    nrm_dgrad = S_loc * sum(n * k for n, k in layers[1:])        # dgrad skips layer 0
    nrm_wgrad = S_loc * sum(n * k + n for n, k in layers)        # wgrad epilogue (+ bias kernel)
    flops = {"fwd": 2 * B * S_loc * sum(n * k for n, k in layers),
             "dgrad": 2 * B * S_loc * sum(n * k for n, k in layers[1:]),
             "wgrad": 2 * B * S_loc * sum(n * k for n, k in layers)}
    normals = {"fwd": nrm_fwd, "dgrad": nrm_dgrad, "wgrad": nrm_wgrad}
    dom = max(prof, key=lambda k: prof[k]["ms"]) if prof else None
    if dom is None:
        return None
    ms = prof[dom]["ms"] / steps
    instr_per_normal = INSTR_PER_NORMAL
    clk_mhz = peaks.get("sm_max_mhz", 1965.0)
    peak = 148 * 128 * clk_mhz * 1e6 / instr_per_normal / 1e9  # Gnormal/s
    out = {"kernel": dom, "ms_per_step": ms}
    if dom in normals:
        ach = normals[dom] / (ms / 1e3) / 1e9
        out.update({"bound": "alu", "achieved": ach, "peak": peak, "unit": "Gnormal/s",
                    "frac": ach / peak, "traffic": _ncu_traffic(dom),
                    "peak_source": f"derived: 148 SM x 128 lanes x {clk_mhz:.0f} MHz / "
                                   f"{instr_per_normal} SASS instr per normal (DESIGN.md §4)",
                    "tensor_tflops": flops[dom] / (ms / 1e3) / 1e12,
                    "tensor_frac_of_measured": flops[dom] / (ms / 1e3) / 1e12
                    / peaks.get("bf16_tflops", 1590.0)})
    else:
        out.update({"bound": "hbm", "achieved": None, "peak": peaks.get("hbm_gbs"),
                    "unit": "GB/s", "frac": None, "traffic": None})
    return out


# SASS instructions issued per ε normal by the fused generator (eps4 + W build), from
# cuobjdump of the gen kernel; see DESIGN.md §4 and profiles/.
INSTR_PER_NORMAL = 40.0


def _ncu_traffic(kernel):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)).get(kernel)
        except Exception:
            return None
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=["C2"])
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--ref-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world, rank, local_rank = _env_world()
    if args.gpus != world and world != 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local_rank)


if __name__ == "__main__":
    main()
