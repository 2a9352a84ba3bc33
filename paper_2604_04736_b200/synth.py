"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds none of the method's arithmetic: it only draws μ, ρ, x and y with
numpy so that the oracle and the CUDA path see the same numbers. The recipe follows
SURVEY.md §8(d) and is restated in DESIGN.md §5:

* μ ~ N(0, 2/fan_in) (Kaiming), weights and biases alike ("initialized in the
  same fashion as for a non-Bayesian network"; biases are variational).
* ρ = softplus⁻¹(c/fan_in) with c = 1 ("constant value that depends on the layer size",
  PAPER.md:148; "scaled inversely with the layer width"), or, for the
  finite-difference and gradient-checking tests, ρ ~ U(-3, 0) so σ ∈ [0.05, 0.69].
* MLP regression (C1): x ~ N(0,1)^8; y = a fixed random 8-16-1 ReLU teacher + N(0, 0.1²).
* MLP classification (C2): x ~ U[0,1]^784 (MNIST-like intensities); labels uniform.
* CNN (C3-C5): x ~ N(0,1) NHWC 32×32×3 (post-normalisation CIFAR-like); labels uniform.

Two parameter regimes (reading R26):

* ``regime="kaiming"`` — the recipe above; the bench workload. Some ReLU pre-activations of
  every example lie within one bf16 rounding of 0, so the BF16 mode's own definition of the
  sampled weight (w_s = RN_bf16(fma_f32(σ, ε, μ)), reading R14) already moves the exact fp64
  gradient of the 20-layer CNN by ≈ 10 % (measured by the oracle alone,
  tests/test_conditioning.py).
* ``regime="positive"`` — the parity regime of the BF16 path: every ReLU pre-activation is
  bounded away from 0, so the step is a smooth function of its operands and bf16 rounding
  moves it by O(2⁻⁸). Hidden-layer weights have a positive mean and a signed spread,
  μ = (1 + v·N(0,1))/fan_in with v = 0.1·√fan_in (each pre-activation ≈ its input mean ×
  (1 ± 10 %)), σ = v/(2·fan_in) (the sampled noise comparable to the μ spread), biases
  μ = 0.2 + 0.01·U(0,1); the output layer is signed, μ ~ N(0, h²/fan_in) with h = 1 (MLP) or
  1/16 (CNN, whose features grow ×2 per residual block) so the logits are O(1); inputs
  x ~ U(0.5, 1.5). A quarter of the units of every layer whose output goes only through a ReLU
  into the next layer (MLP hidden layers; the CNN stem and the first conv of every BasicBlock)
  have the mirrored sign (weights and bias × −1): their pre-activation is ≈ −(input mean) ×
  (1 ± 10 %), firmly below 0, so the ReLU masks of the forward and of the dgrad epilogues are
  exercised without near-ties (their inputs to the next layer are exact zeros, whose
  pre-activations stay positive). CNN images should be ≥ 16×16: at 8×8 stage 4 is 1×1 and a 3×3 kernel sees
  only its centre tap (1/9 of the mean), which brings a few units back near 0. Every weight is still a distinct signed number,
  so a wrong index, tap, tile or operand changes the result by O(1) of the spread.
"""
from __future__ import annotations

import math

import numpy as np

from .configs import input_shape, layout, n_outputs, n_params


def _softplus_inv(s: np.ndarray) -> np.ndarray:
    # ρ such that log(1 + e^ρ) = s; expm1 keeps small s accurate
    return np.log(np.expm1(s))


def _positive_params(model: dict, seed: int, off_frac: float = 0.25):
    rng = np.random.default_rng(seed)
    lay = layout(model)
    P = n_params(model)
    mu = np.empty(P, np.float64)
    rho = np.empty(P, np.float64)
    # output-layer scale: features grow ×2 per residual block (both block inputs positive)
    head = 1.0 if model["kind"] == "mlp" else 1.0 / 16.0
    off = {}  # layer → boolean row mask of the "off" units (pre-activation firmly < 0)
    for ti in lay:
        n = ti["rows"] * ti["cols"]
        sl = slice(ti["offset"], ti["offset"] + n)
        f = ti["fan_in"]
        layer = ti["t"] // 2
        role = ti["role"]
        if role in ("hidden", "stem", "c1") and layer not in off:
            # a quarter of the units (rows) of every layer whose output feeds only a ReLU and
            # then the next conv / linear (never a residual sum) get the mirrored sign
            off[layer] = rng.uniform(0.0, 1.0, ti["rows"] if ti["t"] % 2 == 0 else ti["cols"]) < off_frac
        sign = np.where(off[layer], -1.0, 1.0) if layer in off else None
        if ti["t"] % 2 == 0:  # weight [rows = units, cols = fan-in]
            if role != "out":
                v = 0.1 * math.sqrt(f)
                w = (1.0 + v * rng.normal(0.0, 1.0, (ti["rows"], ti["cols"]))) / f
                if sign is not None:
                    w *= sign[:, None]
                mu[sl] = w.reshape(-1)
                sig = 0.5 * v / f
            else:
                mu[sl] = rng.normal(0.0, head / math.sqrt(f), n)
                sig = 0.5 * head / math.sqrt(f)
        else:  # bias [units]
            if role != "out":
                b = 0.2 + 0.01 * rng.uniform(0.0, 1.0, n)
                mu[sl] = b * sign if sign is not None else b
            else:
                mu[sl] = 0.0
            sig = 0.005
        rho[sl] = _softplus_inv(np.full(n, sig))
    return mu.astype(np.float32), rho.astype(np.float32)


def _vit_params(model: dict, seed: int, rho_mode: str):
    """ViT: Kaiming μ for every linear weight and bias (as the other models),
    LayerNorm gains μ = 1 and offsets μ = 0, cls / position embeddings μ ~ N(0, 0.02²) (the ViT
    convention); σ = 1/fan_in ("scaled inversely with the layer width") or, for the
    finite-difference tests, ρ ~ U(−3, 0)."""
    rng = np.random.default_rng(seed)
    P = n_params(model)
    mu = np.empty(P, np.float64)
    rho = np.empty(P, np.float64)
    for ti in layout(model):
        n = ti["rows"] * ti["cols"]
        sl = slice(ti["offset"], ti["offset"] + n)
        f, role = ti["fan_in"], ti["role"]
        if role in ("w", "b"):
            mu[sl] = rng.normal(0.0, math.sqrt(2.0 / f), n)
        elif role == "ln_g":
            mu[sl] = 1.0
        elif role == "ln_b":
            mu[sl] = 0.0
        else:  # cls, pos
            mu[sl] = rng.normal(0.0, 0.02, n)
        if rho_mode == "wide":
            rho[sl] = rng.uniform(-3.0, 0.0, n)
        elif rho_mode == "tiny":
            rho[sl] = -40.0
        else:
            rho[sl] = _softplus_inv(np.full(n, 1.0 / f))
    return mu.astype(np.float32), rho.astype(np.float32)


def init_params(model: dict, seed: int = 2, rho_mode: str = "init", sigma_c: float = 1.0,
                regime: str = "kaiming"):
    """Return (mu, rho) as float32 arrays of length n_params(model)."""
    if model["kind"] == "vit":
        return _vit_params(model, seed, rho_mode)
    if regime == "positive":
        assert rho_mode == "init"
        return _positive_params(model, seed)
    assert regime == "kaiming", regime
    rng = np.random.default_rng(seed)
    P = n_params(model)
    mu = np.empty(P, np.float64)
    rho = np.empty(P, np.float64)
    for ti in layout(model):
        n = ti["rows"] * ti["cols"]
        sl = slice(ti["offset"], ti["offset"] + n)
        mu[sl] = rng.normal(0.0, math.sqrt(2.0 / ti["fan_in"]), n)
        if rho_mode == "init":
            rho[sl] = _softplus_inv(np.full(n, sigma_c / ti["fan_in"]))
        elif rho_mode == "wide":
            rho[sl] = rng.uniform(-3.0, 0.0, n)
        elif rho_mode == "tiny":
            rho[sl] = -40.0
        else:
            raise ValueError(rho_mode)
    return mu.astype(np.float32), rho.astype(np.float32)


def make_batch(model: dict, B: int, seed: int = 1, regime: str = "kaiming"):
    """Return (x, y_cls, y_reg): x float32 [B, *input_shape]; exactly one of y_* is set."""
    rng = np.random.default_rng(seed)
    shp = input_shape(model)
    O = n_outputs(model)
    if regime == "positive":
        x = rng.uniform(0.5, 1.5, (B,) + shp)
        if model["loss"].split("_")[0] == "ce":
            return x.astype(np.float32), rng.integers(0, O, B).astype(np.int32), None
        return x.astype(np.float32), None, rng.normal(0.0, 1.0, (B, O)).astype(np.float32)
    assert regime == "kaiming", regime
    if model["kind"] == "mlp" and model["loss"].split("_")[0] in ("mse", "gnll"):
        x = rng.normal(0.0, 1.0, (B,) + shp)
        # fixed teacher network: widths of the model, ReLU hidden layers
        w = model["widths"]
        trng = np.random.default_rng(12345)
        h = x
        for i in range(1, len(w)):
            W = trng.normal(0.0, math.sqrt(2.0 / w[i - 1]), (w[i], w[i - 1]))
            h = h @ W.T
            if i < len(w) - 1:
                h = np.maximum(h, 0.0)
        y = h + rng.normal(0.0, 0.1, h.shape)
        return x.astype(np.float32), None, y.astype(np.float32)
    if model["kind"] == "mlp":
        x = rng.uniform(0.0, 1.0, (B,) + shp)
    else:
        x = rng.normal(0.0, 1.0, (B,) + shp)
    if model["loss"].split("_")[0] == "ce":
        y = rng.integers(0, O, B).astype(np.int32)
        return x.astype(np.float32), y, None
    y = rng.normal(0.0, 1.0, (B, O))
    return x.astype(np.float32), None, y.astype(np.float32)
