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

WORKLOAD_NAMES = {
    "mlp_784_1024_1024_10": "Bayesian MLP 784-1024-1024-10 (CE)",
    "mlp_8_16_1": "Bayesian MLP 8-16-1 (MSE)",
    "resnet18_cifar": "ResNet-18-shaped Bayesian CNN, 32x32x3, per-sample crop+flip",
    "mcd_mlp_96_128_128_24": "MC-dropout MLP 96-128-128-24 (p=0.1), MSE of the averaged predictions",
}


def run_plan(config, world, mode_arg=None):
    """Samples / batch per rank for a BASELINE config at `world` GPUs."""
    cfg = CONFIGS[config]
    if config == "C3":  # weak: S = 8 per GPU, same batch everywhere
        S_loc, B = cfg["S_per_gpu"], cfg["B"]
        return dict(S=S_loc * world, S_loc=S_loc, B=B, B_loc=B, K=world, G=1, mode="sample",
                    scaling="weak")
    if config == "C4":  # strong: S = 64 fixed; sample-sharded (default) or data-sharded
        mode = mode_arg or "sample"
        if mode == "data":
            return dict(S=cfg["S"], S_loc=cfg["S"], B=cfg["B"], B_loc=cfg["B"] // world, K=1,
                        G=world, mode="data", scaling="strong")
        return dict(S=cfg["S"], S_loc=cfg["S"] // world, B=cfg["B"], B_loc=cfg["B"], K=world,
                    G=1, mode="sample", scaling="strong")
    if config == "C5":  # hybrid 4 sample groups x 2 data groups (world 8); K = world/2 below 8
        G = 2 if world >= 2 else 1
        K = max(1, world // G)
        return dict(S=cfg["S"], S_loc=cfg["S"] // K, B=cfg["B"], B_loc=cfg["B"] // G, K=K, G=G,
                    mode="hybrid" if world > 1 else "sample", scaling="strong")
    # C1 / C2 / C6: weak scaling, S = S_config per GPU
    S_loc, B = cfg["S"], cfg["B"]
    return dict(S=S_loc * world, S_loc=S_loc, B=B, B_loc=B, K=world, G=1, mode="sample",
                scaling="weak")


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
def cpu_oracle_rate(model, B, D, budget_s=15.0, seed=0x5EED, aug="none"):
    """Time the fp64 oracle (as it stands) on the host cores over a bounded sample of the
    workload: all B examples, S_sample samples; returns (sample·images/s, cores, sample)."""
    import oracle as O
    mu, rho = synth.init_params(model, seed=2)
    x, yc, yr = synth.make_batch(model, B, seed=1)
    cores = os.cpu_count() or 1
    O.lib()
    a = O.AUG_PER_SAMPLE if aug == "per_sample" else O.AUG_NONE
    # probe with a few images, then size the slice to ≈ budget_s of CPU work
    Bp = min(B, 8)
    t0 = time.perf_counter()
    O.elbo_partial(model, mu, rho, x[:Bp], None if yc is None else yc[:Bp],
                   None if yr is None else yr[:Bp], B, 0, 64, 0, 1, seed, 0, a)
    t1 = (time.perf_counter() - t0) / Bp
    n_img = max(1, int(budget_s / max(t1, 1e-6)))
    if n_img >= B:
        S_sample, B_s = max(1, min(64, n_img // B)), B
    else:
        S_sample, B_s = 1, n_img
    t0 = time.perf_counter()
    O.elbo_partial(model, mu, rho, x[:B_s], None if yc is None else yc[:B_s],
                   None if yr is None else yr[:B_s], B, 0, 64, 0, S_sample, seed, 0, a)
    dt = time.perf_counter() - t0
    return S_sample * B_s / dt, cores, (f"{S_sample} sample(s) x {B_s} of {B} images (a slice of "
                                        f"one step), fp64, {cores} threads")


def run_reference(args, world, rank):
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    model = MODELS[cfg["model"]]
    plan = run_plan(args.config, world, args.mode)
    B, S = plan["B"], plan["S"]
    rates = []
    for i in range(args.warmup + args.steps):
        r, cores, sample = cpu_oracle_rate(model, B, cfg["D"], budget_s=args.ref_budget,
                                           aug=cfg.get("aug", "none"))
        if i >= args.warmup:
            rates.append(r)
    v = statistics.median(rates)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "sample·images/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": S * B / v * 1e3, "higher_is_better": True,
            "scaling": plan["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {WORKLOAD_NAMES[cfg['model']]}",
                       "global_batch": B, "samples": S},
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
    distributed = world > 1 or "TORCHELASTIC_RUN_ID" in os.environ
    if distributed:
        dist.init_process_group("nccl", device_id=dev)
        obj = [native.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    cfg = CONFIGS[args.config]
    model = MODELS[cfg["model"]]
    if args.agg == "mean":  # exact aggregation: loss of the mean prediction
        model = dict(model, loss=model["loss"] + "_mean")
    elif args.agg == "gnll":  # Gaussian NLL of the predictive (regression configs, FP32)
        assert model["loss"] == "mse", "--agg gnll needs a regression config (C1)"
        model = dict(model, loss="gnll_mean")
    plan = run_plan(args.config, world, args.mode)
    B, B_loc, S, S_loc, K, G = plan["B"], plan["B_loc"], plan["S"], plan["S_loc"], plan["K"], plan["G"]
    D = cfg["D"]
    P = n_params(model)
    g_idx = rank % G

    mu_h, rho_h = synth.init_params(MODELS[cfg["model"]], seed=2)
    x_h, yc_h, yr_h = synth.make_batch(MODELS[cfg["model"]], B, seed=1)
    # this rank's data-group shard of the global batch
    x_h = x_h[g_idx * B_loc:(g_idx + 1) * B_loc]
    yc_h = None if yc_h is None else yc_h[g_idx * B_loc:(g_idx + 1) * B_loc]
    yr_h = None if yr_h is None else yr_h[g_idx * B_loc:(g_idx + 1) * B_loc]
    mu = torch.from_numpy(mu_h).to(dev)
    rho = torch.from_numpy(rho_h).to(dev)
    x = torch.from_numpy(x_h).to(dev)
    y = torch.from_numpy(yc_h if yc_h is not None else yr_h).to(dev)
    gmu = torch.empty_like(mu)
    grho = torch.empty_like(rho)
    loss_dev = torch.zeros(1, device=dev)
    stream = torch.cuda.current_stream(dev)
    ctx = native.Context(model, precision=args.precision, mode=plan["mode"], K=K, G=G, rank=rank,
                         world=world, uid=uid, max_B_loc=B_loc, max_S_loc=S_loc, dataset_size=D,
                         device=local_rank, stream=stream.cuda_stream, aug=cfg.get("aug", "none"))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    adam = args.optimizer == "adam"
    mom = [torch.zeros_like(mu) for _ in range(4)] if adam else None
    n_upd = [0]

    def step(i):
        if adam:
            # one training step: ELBO gradients + the fused Adam update of μ, ρ
            n_upd[0] += 1
            ctx.elbo_step_adam(mu, rho, x, y, B, S, 0x5EED, i, mom, t=n_upd[0], want_loss=False)
        else:
            ctx.elbo_step(mu, rho, x, y, B, S, 0x5EED, i, grad_mu=gmu, grad_rho=grho,
                          loss_dev=loss_dev, want_loss=False)

    def step_host(i):
        if adam:
            x.copy_(x_pin, non_blocking=True)
            y.copy_(y_pin, non_blocking=True)
            n_upd[0] += 1
            ctx.elbo_step_adam(mu, rho, x, y, B, S, 0x5EED, i, mom, t=n_upd[0], want_loss=True)
        else:
            ctx.elbo_step_host(mu, rho, x_pin, y_pin, B, S, 0x5EED, i, grad_mu=gmu, grad_rho=grho)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches0 = ctx.launch_count()
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            ev[i][0].record(stream)
            step(args.warmup + i)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    launches = ctx.launch_count() - launches0
    # per-kernel-class timing (the roofline line) in separate, untimed steps: the class events
    # the library records around its launches would otherwise sit inside the timed region
    prof_steps = max(3, min(args.steps, 10))
    ctx.profile(True)
    for i in range(prof_steps):
        flush.zero_()
        step(args.warmup + args.steps + i)
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile(False)
    if distributed:
        dist.barrier()
    times = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(times)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = S * B / (ms_per_step / 1e3)

    # ---------------- end to end through the public API with host buffers
    x_pin = torch.from_numpy(x_h).pin_memory()
    y_pin = torch.from_numpy(yc_h if yc_h is not None else yr_h).pin_memory()
    for i in range(2):
        step_host(i)
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    e_ms = []
    for i in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step_host(i)
        e_ms.append((time.perf_counter() - t0) * 1e3)
    te = torch.tensor([sum(e_ms)], dtype=torch.float64, device=dev)
    if distributed:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = S * B / (float(te.item()) / args.steps / 1e3)

    if rank == 0:
        peaks, peak_src = _peaks()
        line = {"metric": METRIC, "value": value, "unit": "sample·images/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": plan["scaling"], "vs_baseline": None,
                "dtype": "bf16" if args.precision == "bf16" else "f32", "data": "synthetic",
                "config": {"workload": f"{args.config}: {WORKLOAD_NAMES[cfg['model']]}",
                           "global_batch": B, "samples": S, "samples_per_gpu": S_loc,
                           "params": P, "parallelism": f"{plan['mode']}-sharded K{K}xG{G}",
                           "loss_aggregation": {"mean": "loss of the mean prediction (exact, PAPER.md:272-281)",
                                                "gnll": "Gaussian NLL of the predictive mean/variance (P:349, P:281)",
                                                "sample": "mean of per-sample losses (Alg. 1 l.9)"}[args.agg],
                           "optimizer": "fused Adam (in the timed step)" if adam else
                                        "none (step returns grad_mu, grad_rho; north_star boundary)",
                           "l2": "flushed between timed steps (256 MiB memset outside events)"},
                "clocks": clk.summary(),
                "e2e": {"value": e2e_value, "unit": "sample·images/s",
                        "h2d_bytes_per_step": int(x_pin.numel() * 4 + y_pin.numel() * 4),
                        "d2h_bytes_per_step": 4},
                "gpu_launches": int(launches),
                "nccl": bool(uid is not None),
                "kernel_ms_per_step": {k: v["ms"] / prof_steps for k, v in prof.items()},
                "kernel_ms_note": f"per kernel class, CUDA events around each launch, {prof_steps} extra "
                                  "untimed steps (profiling off in the timed region)"}
        line["roofline"] = roofline(model, B_loc, S_loc, prof, prof_steps, peaks, peak_src)
        if world == 1 and not args.no_cpu_baseline:
            r, cores, sample = cpu_oracle_rate(MODELS[cfg["model"]], B, D, budget_s=args.ref_budget,
                                               aug=cfg.get("aug", "none"))
            line["cpu_baseline"] = {"value": r, "unit": "sample·images/s", "cores": cores,
                                    "kind": "oracle", "sample": sample}
        print(json.dumps(line), flush=True)
    ctx.close()
    if distributed:
        dist.destroy_process_group()


def conv_layers(model):
    """(k, stride, cin, cout, out_h, out_w) of every layer in execution order (the CNN)."""
    H, W, C = model["in_h"], model["in_w"], model["in_c"]
    bw = model.get("base_width", 64)
    out = []

    def conv(h, w, cin, cout, k, st, p):
        oh, ow = (h + 2 * p - k) // st + 1, (w + 2 * p - k) // st + 1
        out.append((k, st, cin, cout, oh, ow))
        return oh, ow

    H, W = conv(H, W, C, bw, 3, 1, 1)
    width = bw
    for stage in range(4):
        cout = bw << stage
        for blk in range(2):
            st = 2 if (stage > 0 and blk == 0) else 1
            h1, w1 = conv(H, W, width, cout, 3, st, 1)
            conv(h1, w1, cout, cout, 3, 1, 1)
            if st != 1 or width != cout:
                conv(H, W, width, cout, 1, st, 0)
            H, W, width = h1, w1, cout
    out.append((1, 1, width, model["n_classes"], 1, 1))
    return out


def roofline(model, B, S_loc, prof, steps, peaks, peak_src):
    """Dominant kernel class vs its bound.

    MLP: the sampled-GEMM kernels are ALU-bound by ε regeneration; unit =
    ε normals generated, peak = 148 SMs × 128 lanes × f_clk / (instructions per normal).
    CNN: the conv kernels are tensor-bound; unit = dense bf16 FLOP, peak = measured cuBLAS
    bf16 (sustained: the kernels are timed inside a multi-ms step)."""
    dom = max((k for k in prof if k in ("fwd", "dgrad", "wgrad", "wgen")),
              key=lambda k: prof[k]["ms"], default=None)
    if dom is None:
        return None
    ms = prof[dom]["ms"] / steps
    if model["kind"] == "mlp" and n_params(model) < 10000:
        # C1 (161 parameters, 78 KFLOP per step): launch/latency-bound, no roofline
        return {"kernel": dom, "ms_per_step": ms, "bound": "latency", "achieved": None, "peak": None,
                "unit": None, "frac": None, "traffic": None,
                "note": "C1 is latency-bound (tiny MLP); SURVEY.md §8(d) reports µs/step only"}
    if model["kind"] == "mlp":
        w = model["widths"]
        layers = [(w[i + 1], w[i]) for i in range(len(w) - 1)]
        normals = {"fwd": S_loc * sum(n * k + n for n, k in layers),
                   "dgrad": S_loc * sum(n * k for n, k in layers[1:]),
                   "wgrad": S_loc * sum(n * k + n for n, k in layers)}
        flops = {"fwd": 2 * B * S_loc * sum(n * k for n, k in layers),
                 "dgrad": 2 * B * S_loc * sum(n * k for n, k in layers[1:]),
                 "wgrad": 2 * B * S_loc * sum(n * k for n, k in layers)}
        clk_mhz = peaks.get("sm_max_mhz", 1965.0)
        peak = 148 * 128 * clk_mhz * 1e6 / INSTR_PER_NORMAL / 1e9  # Gnormal/s
        ach = normals[dom] / (ms / 1e3) / 1e9
        return {"kernel": dom, "ms_per_step": ms, "bound": "alu", "achieved": ach, "peak": peak,
                "unit": "Gnormal/s", "frac": ach / peak, "traffic": _ncu_traffic("mlp", dom),
                "peak_source": f"derived: 148 SM x 128 lanes x {clk_mhz:.0f} MHz / "
                               f"{INSTR_PER_NORMAL} SASS instr per normal (DESIGN.md §4)",
                "tensor_tflops": flops[dom] / (ms / 1e3) / 1e12,
                "tensor_frac_of_measured": flops[dom] / (ms / 1e3) / 1e12
                / peaks.get("bf16_tflops", 1590.0),
                # context: the standalone generator's measured rate (scripts/eps_rate.py; the
                # fused kernels also load μ/σ, build and store W_s tiles, run the epilogue)
                **_standalone_eps(ach)}
    convs = conv_layers(model)
    f_all = sum(2 * B * oh * ow * co * k * k * ci for k, st, ci, co, oh, ow in convs)
    f_nostem = f_all - 2 * B * convs[0][4] * convs[0][5] * convs[0][3] * 9 * convs[0][2]
    flops = {"fwd": S_loc * f_all, "dgrad": S_loc * f_nostem, "wgrad": S_loc * f_all}
    peak = peaks.get("bf16_tflops_sustained", 1400.0)
    if dom not in flops:
        return {"kernel": dom, "ms_per_step": ms, "bound": "alu", "achieved": None, "peak": None,
                "unit": None, "frac": None, "traffic": None}
    ach = flops[dom] / (ms / 1e3) / 1e12
    return {"kernel": dom, "ms_per_step": ms, "bound": "tensor", "achieved": ach, "peak": peak,
            "unit": "TFLOP/s", "frac": ach / peak, "traffic": _ncu_traffic("cnn", dom),
            "peak_source": f"measured bf16 sustained ({peak_src}, MEASURED_PEAKS.json); "
                           f"burst {peaks.get('bf16_tflops')}"}


def _standalone_eps(achieved):
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01", "session2", "eps_rate.txt")
    try:
        rate = json.loads(open(path).read().strip().splitlines()[-1])["eps_bench_gnormal_per_s"]
    except (OSError, ValueError, KeyError, IndexError):
        return {}
    return {"standalone_generator_gnormal_s": rate, "frac_of_standalone_generator": achieved / rate,
            "standalone_source": "profiles/r01/session2/eps_rate.txt (scripts/eps_rate.py, measured)"}


# SASS instructions issued per ε normal by the fused generator (eps4 + W build), from
# cuobjdump of the gen kernel; see DESIGN.md §4 and profiles/.
INSTR_PER_NORMAL = 40.0


def _ncu_traffic(kind, kernel):
    """DRAM bytes (read + write) per launch of the class, from an ncu capture committed under
    profiles/ (profiles/ncu_traffic.json, written by scripts/traffic_summary.py)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)).get(f"{kind}:{kernel}")
        except Exception:
            return None
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5", "C6"])
    ap.add_argument("--mode", default=None, choices=["sample", "data"])
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--ref-budget", type=float, default=None,
                    help="seconds of oracle CPU work per reference step (default: 150 s / (K+W))")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--agg", default="sample", choices=["sample", "mean", "gnll"],
                    help="mean: exact aggregation, the loss of the mean prediction; gnll: Gaussian "
                         "NLL of the predictive mean and variance (C1, --precision fp32)")
    ap.add_argument("--optimizer", default="none", choices=["none", "adam"],
                    help="adam: each step also applies the fused Adam update (bnn_elbo_step_adam)")
    args = ap.parse_args()
    world, rank, local_rank = _env_world()
    if args.gpus != world and world != 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    if args.ref_budget is None:
        args.ref_budget = min(15.0, max(1.0, 150.0 / (args.steps + args.warmup)))
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local_rank)


if __name__ == "__main__":
    main()
