#!/usr/bin/env python
"""bench.py — ELBO-step throughput (sample·images/s) of the sample-sharded BNN step on B200.

Contract (README/DESIGN.md §7): `python bench.py --gpus N --steps K --warmup W` runs the
BASELINE.json workload; for N>1 it is launched under torchrun (one rank per GPU, NCCL).
Rank 0 prints ONE JSON line. A "step" is one pass of the whole hot path (σ prologue,
sampled forward, loss head, sampled backward with sample-accumulating wgrad, allreduce,
finalize + KL) over one synthetic minibatch.

Default workload: C3 = the ResNet-18-shaped Bayesian CNN on 32×32×3 CIFAR-shaped batches,
B = 128, S = 8 per GPU, per-sample crop+flip (BASELINE.json configs[2], the configuration its
metric is quoted on); N > 1 is weak-scaled (S = 8·N sharded over N ranks, same batch).
`--config C2` is the Bayesian MLP 784-1024-1024-10 (B = 256, S = 64), C4 the strong-scaled
S = 64 run (sample- vs `--mode data`-sharded), C5 the 4×2 hybrid grid, C1/C6 the small MLPs.

`--gpus N` with N > 1 outside torchrun re-executes itself under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU, NCCL) and fails
loudly when fewer than N GPUs are visible.

`--impl reference` times the CPU oracle (oracle/, fp64, all host cores): each of its steps is
a bounded, stated slice of the same workload (the full C3 step is ≈ 1 core-hour), timed as
it runs — the tier's reference arm.
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
    "vit_cifar": "Bayesian ViT (4x4 patches, width 192, 3 heads, 6 layers, MLP 768), 32x32x3, per-sample crop+flip",
}


def run_plan(config, world, mode_arg=None):
    """Samples / batch per rank for a BASELINE config at `world` GPUs."""
    cfg = CONFIGS[config]
    if config in ("C3", "C7"):  # weak: S = 8 per GPU, same batch everywhere
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
    """SM clocks + throttle reasons sampled every 5 ms during the timed region (NVML, the
    library nvidia-smi reads; nvidia-smi -lms as the fallback)."""

    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []  # (sm_mhz, sm_max_mhz, reasons bitmask)
        self.stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[self.idx]) if vis and vis.split(",")[0].isdigit() else self.idx
            h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def poll():
                while not self.stop.is_set():
                    self.rows.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), mx, reasons(h)))
                    time.sleep(0.005)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        if self.t is not None:
            time.sleep(0.01)
            self.stop.set()
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [r[0] for r in self.rows]
        reasons = sorted({k for r in self.rows for k, bit in self.BITS.items() if r[2] & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in self.rows),
                "sm_mhz_min": min(sm), "reasons": reasons, "samples": len(self.rows),
                "source": "NVML every 5 ms inside the timed region"}


# ====================================================================== reference arm
def oracle_slice(model, B, budget_s, aug="none"):
    """Size a bounded slice of one step for the fp64 oracle (as it stands, all host cores):
    all B examples × n samples if one sample of the batch fits the budget, else 1 sample × n
    examples (≥ the core count, the oracle parallelises over examples). Returns a callable
    that runs the slice once, and its (samples, images, description)."""
    import oracle as O
    mu, rho = synth.init_params(model, seed=2)
    x, yc, yr = synth.make_batch(model, B, seed=1)
    cores = os.cpu_count() or 1
    O.lib()
    a = O.AUG_PER_SAMPLE if aug == "per_sample" else O.AUG_NONE

    def run(S_s, B_s):
        if model["kind"] == "vit":
            O.vit_elbo_partial(model, mu, rho, x[:B_s], yc[:B_s], B, 0, 64, 0, S_s, 0x5EED, 0, a)
            return
        O.elbo_partial(model, mu, rho, x[:B_s], None if yc is None else yc[:B_s],
                       None if yr is None else yr[:B_s], B, 0, 64, 0, S_s, 0x5EED, 0, a)

    Bp = min(B, cores)
    t0 = time.perf_counter()
    run(1, Bp)
    t_img = (time.perf_counter() - t0) / Bp  # wall seconds per sample·image with ≥ cores threads busy
    n_img = max(1, int(budget_s / max(t_img, 1e-9)))
    if n_img >= B:
        S_s, B_s = max(1, min(64, n_img // B)), B
    else:
        S_s, B_s = 1, max(1, min(B, n_img))
    desc = (f"{S_s} sample(s) x {B_s} of {B} images of one step (a bounded slice; value = "
            f"sample-images of the slice / its wall time), fp64, {cores} threads")
    return (lambda: run(S_s, B_s)), S_s, B_s, cores, desc


def cpu_oracle_rate(model, B, budget_s, aug="none"):
    fn, S_s, B_s, cores, desc = oracle_slice(model, B, budget_s, aug)
    t0 = time.perf_counter()
    fn()
    dt = time.perf_counter() - t0
    return S_s * B_s / dt, cores, desc


def run_reference(args, world, rank):
    """The tier's reference arm: the oracle as it stands, rank 0 only; each step is the same
    bounded slice of the workload, timed as it runs (ms_per_step is that slice's time)."""
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    model = MODELS[cfg["model"]]
    plan = run_plan(args.config, world, args.mode)
    B, S = plan["B"], plan["S"]
    fn, S_s, B_s, cores, desc = oracle_slice(model, B, args.ref_budget, cfg.get("aug", "none"))
    for _ in range(args.warmup):
        fn()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    ms = sum(ts) / len(ts) * 1e3
    v = S_s * B_s / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "sample·images/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True,
            "scaling": plan["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {WORKLOAD_NAMES[cfg['model']]}",
                       "global_batch": B, "samples": S,
                       "reference_step": desc,
                       "full_step_estimate_s": S * B / v},
            "cpu_baseline": {"value": v, "unit": "sample·images/s", "cores": cores,
                             "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": "sample·images/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ====================================================================== our arm
def _time_steps(step, n, stream, flush, sampler=None):
    """n steps, each bracketed by CUDA events on the library's stream, an L2 flush (a 256 MiB
    memset, > the 126 MB L2) between them outside the events; returns the summed ms."""
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for i in range(n):
        flush.zero_()
        ev[i][0].record(stream)
        step(i)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev)


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
    x_all, yc_all, yr_all = synth.make_batch(MODELS[cfg["model"]], B, seed=1)

    def shard(gi, bl):
        return (x_all[gi * bl:(gi + 1) * bl], None if yc_all is None else yc_all[gi * bl:(gi + 1) * bl],
                None if yr_all is None else yr_all[gi * bl:(gi + 1) * bl])

    x_h, yc_h, yr_h = shard(g_idx, B_loc)
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
                         device=local_rank, stream=stream.cuda_stream, aug=cfg.get("aug", "none"),
                         sample_chunk=args.sample_chunk)
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
    launches0 = ctx.launch_count()
    with ClockSampler(local_rank) as clk:
        total_ms = _time_steps(lambda i: step(args.warmup + i), args.steps, stream, flush)
    launches = ctx.launch_count() - launches0
    if distributed:
        dist.barrier()
    if args.profile_run:  # under ncu: the timed steps only (their numbers are not bench values)
        ctx.close()
        if rank == 0:
            print(json.dumps({"profile_run": True, "launches": int(launches), "steps": args.steps}), flush=True)
        if distributed:
            dist.destroy_process_group()
        return
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
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = S * B / (ms_per_step / 1e3)

    # ---------------- end to end through the public API with host buffers
    x_pin = torch.from_numpy(np.ascontiguousarray(x_h)).pin_memory()
    y_pin = torch.from_numpy(np.ascontiguousarray(yc_h if yc_h is not None else yr_h)).pin_memory()
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
    ctx.close()

    # ---------------- the paper's comparison: the same library, DDP-style data-sharded
    # (K = 1, G = world: every rank draws all S samples for its B/world examples),
    # same global S and B, timed the same way (N > 1 only; at N = 1 the two modes coincide)
    ddp = None
    if world > 1 and args.config in ("C3", "C4") and args.mode != "data" and not args.no_ddp and B % world == 0:
        Bd = B // world
        xd_h, ycd_h, yrd_h = shard(rank, Bd)
        xd = torch.from_numpy(np.ascontiguousarray(xd_h)).to(dev)
        yd = torch.from_numpy(np.ascontiguousarray(ycd_h if ycd_h is not None else yrd_h)).to(dev)
        obj = [native.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        cd = native.Context(model, precision=args.precision, mode="data", K=1, G=world, rank=rank,
                            world=world, uid=obj[0], max_B_loc=Bd, max_S_loc=S, dataset_size=D,
                            device=local_rank, stream=stream.cuda_stream, aug=cfg.get("aug", "none"),
                            sample_chunk=min(S, max(8, args.sample_chunk)))

        def dstep(i):
            cd.elbo_step(mu, rho, xd, yd, B, S, 0x5EED, i, grad_mu=gmu, grad_rho=grho,
                         loss_dev=loss_dev, want_loss=False)
        for i in range(args.warmup):
            dstep(i)
        torch.cuda.synchronize()
        dist.barrier()
        td = torch.tensor([_time_steps(lambda i: dstep(args.warmup + i), args.steps, stream, flush)],
                          dtype=torch.float64, device=dev)
        dist.all_reduce(td, op=dist.ReduceOp.MAX)
        ms_d = float(td.item()) / args.steps
        ddp = {"value": S * B / (ms_d / 1e3), "ms_per_step": ms_d, "unit": "sample·images/s",
               "parallelism": f"data-sharded K1xG{world} (S_loc={S}, B_loc={Bd})",
               "note": "the paper's DDP-style comparison (P:185-193, P:390-394), same library/kernels"}
        cd.close()

    if rank == 0:
        peaks, peak_src = _peaks()
        line = {"metric": METRIC, "value": value, "unit": "sample·images/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": plan["scaling"], "vs_baseline": None,
                "dtype": "bf16" if args.precision == "bf16" else "f32", "data": "synthetic",
                "config": {"workload": f"{args.config}: {WORKLOAD_NAMES[cfg['model']]}",
                           "global_batch": B, "samples": S, "samples_per_gpu": S_loc,
                           "batch_per_gpu": B_loc,
                           "params": P, "parallelism": f"{plan['mode']}-sharded K{K}xG{G}",
                           "loss_aggregation": {"mean": "loss of the mean prediction (exact, PAPER.md:272-281)",
                                                "gnll": "Gaussian NLL of the predictive mean/variance (P:349, P:281)",
                                                "sample": "mean of per-sample losses (Alg. 1 l.9)"}[args.agg],
                           "optimizer": "fused Adam (in the timed step)" if adam else
                                        "none (step returns grad_mu, grad_rho; north_star boundary)",
                           "init": "Kaiming mu, rho = softplus^-1(1/fan_in) (PAPER.md:148; DESIGN.md §5)",
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
        if ddp is not None:
            line["ddp_comparison"] = ddp
        line["roofline"] = roofline(model, B_loc, S_loc, prof, prof_steps, peaks, peak_src, args.precision == "bf16")
        if world == 1 and not args.no_cpu_baseline:
            r, cores, sample = cpu_oracle_rate(MODELS[cfg["model"]], B, args.ref_budget,
                                               aug=cfg.get("aug", "none"))
            line["cpu_baseline"] = {"value": r, "unit": "sample·images/s", "cores": cores,
                                    "kind": "oracle", "sample": sample}
        print(json.dumps(line), flush=True)
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


def roofline(model, B, S_loc, prof, steps, peaks, peak_src, bf16=True):
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
    if model["kind"] == "mlp" and model.get("method") == "mcd":
        # C6 (MC dropout): weights μ, no ε drawn (R25); 96-128-128-24 at B = 256 is a few
        # GFLOP per step, far below every roofline: latency-bound, reported with its tensor rate
        w = model["widths"]
        fl = {"fwd": 2 * B * S_loc * sum(w[i] * w[i + 1] for i in range(len(w) - 1)),
              "dgrad": 2 * B * S_loc * sum(w[i] * w[i + 1] for i in range(1, len(w) - 1)),
              "wgrad": 2 * B * S_loc * sum(w[i] * w[i + 1] for i in range(len(w) - 1))}
        return {"kernel": dom, "ms_per_step": ms, "bound": "latency", "achieved": None, "peak": None,
                "unit": None, "frac": None, "traffic": None,
                "tensor_tflops": fl[dom] / (ms / 1e3) / 1e12,
                "note": "MC dropout draws no eps (weights mu); tiny GEMMs: launch/latency-bound"}
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
    if model["kind"] == "vit":
        return vit_roofline(model, B, S_loc, prof, steps, peaks, peak_src, bf16)
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


def vit_flops(model, B):
    """GEMM-shaped FLOP of one forward per sample (projections + attention products)."""
    D, M, h, L = model["dim"], model["mlp"], model["heads"], model["depth"]
    T = 1 + (model["in_h"] // model["patch"]) * (model["in_w"] // model["patch"])
    pk = model["patch"] ** 2 * model["in_c"]
    proj = 2 * B * T * L * (3 * D * D + D * D + 2 * D * M) + 2 * B * (T - 1) * pk * D + 2 * B * D * model["n_classes"]
    attn = 2 * 2 * B * L * h * T * T * (D // h)
    return proj, attn


def vit_roofline(model, B, S_loc, prof, steps, peaks, peak_src, bf16):
    """The ViT's sampled projections (fwd + dgrad + wgrad classes): BF16 — tcgen05 against the
    measured bf16 peak (W_s is regenerated per 256-row tile, so like C2 the generator's ALU work
    is the co-limiter); FP32 — SIMT against the FP32 FMA peak (148 SM × 128 FMA/clk × 2 × f_max)."""
    proj, attn = vit_flops(model, B)
    ms = sum(prof[k]["ms"] for k in ("fwd", "dgrad", "wgrad") if k in prof) / steps
    fl = 3 * proj * S_loc
    ach = fl / (ms / 1e3) / 1e12
    if bf16:
        peak = peaks.get("bf16_tflops_sustained", 1400.0)
        src = f"measured bf16 sustained ({peak_src}, MEASURED_PEAKS.json)"
        bound = "tensor"
    else:
        clk = peaks.get("sm_max_mhz", 1965.0)
        peak = 148 * 128 * 2 * clk * 1e6 / 1e12
        src = f"derived FP32 FMA peak: 148 SM x 128 lanes x 2 FLOP x {clk:.0f} MHz"
        bound = "alu"
    step_ms = sum(v["ms"] for v in prof.values()) / steps
    return {"kernel": "fwd+dgrad+wgrad (sampled projections)", "ms_per_step": ms, "bound": bound, "achieved": ach,
            "peak": peak, "unit": "TFLOP/s", "frac": ach / peak, "traffic": None, "peak_source": src,
            "attention_ms_per_step": prof.get("attn", {}).get("ms", 0.0) / steps,
            "attention_tflop_per_step": 3 * attn * S_loc / 1e12,
            "projection_share_of_profiled_step": ms / step_ms if step_ms else None}


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


def _spawn(args_list, n):
    """Re-execute this script under torchrun with n ranks (one per GPU) on 127.0.0.1."""
    import socket
    import torch
    if torch.cuda.device_count() < n:
        print(f"bench.py: --gpus {n} but only {torch.cuda.device_count()} GPU(s) visible", file=sys.stderr)
        sys.exit(2)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + args_list
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C4", "C5", "C6", "C7"])
    ap.add_argument("--mode", default=None, choices=["sample", "data"])
    ap.add_argument("--precision", default=None, choices=["bf16", "fp32"],
                    help="default bf16 (C7, the ViT: fp32)")
    ap.add_argument("--sample-chunk", type=int, default=0,
                    help="samples per pass through the network (0: the library default, all local samples)")
    ap.add_argument("--ref-budget", type=float, default=None,
                    help="seconds of oracle CPU work per reference step (default: 150 s / (K+W), ≤ 15 s)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-run", action="store_true",
                    help="for ncu launch lists: warm-up + timed steps only, no e2e / class profiling / "
                         "CPU baseline; prints no bench line")
    ap.add_argument("--no-ddp", action="store_true", help="skip the data-sharded comparison line (N > 1)")
    ap.add_argument("--agg", default="sample", choices=["sample", "mean", "gnll"],
                    help="mean: exact aggregation, the loss of the mean prediction; gnll: Gaussian "
                         "NLL of the predictive mean and variance (C1, --precision fp32)")
    ap.add_argument("--optimizer", default="none", choices=["none", "adam"],
                    help="adam: each step also applies the fused Adam update (bnn_elbo_step_adam)")
    args = ap.parse_args()
    world, rank, local_rank = _env_world()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _spawn(sys.argv[1:], args.gpus)
    if args.gpus != world:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.precision is None:
        args.precision = "fp32" if args.config == "C7" else "bf16"
    if args.warmup < 3 and not args.profile_run:
        print("bench.py: --warmup must be >= 3", file=sys.stderr)
        sys.exit(2)
    if args.ref_budget is None:
        args.ref_budget = min(15.0, max(1.0, 150.0 / (args.steps + args.warmup)))
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local_rank)


if __name__ == "__main__":
    main()
