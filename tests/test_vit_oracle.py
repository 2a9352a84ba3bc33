"""Pins of the ViT oracle (oracle/vit_oracle.c) against what mathematics and
independent formulations fix — no GPU:

* an independent fp64 torch formulation (F.layer_norm, F.gelu, softmax attention, autograd),
  with and without per-sample augmentation: the whole data term (acc_μ, acc_ρ, L_data);
* central finite differences of the ELBO (the network is smooth — GELU, LayerNorm, softmax —
  so FD holds everywhere), for entries of every kind of tensor, common random numbers;
* σ → 0 (ρ = −40): the data term is the deterministic ViT with weights μ;
* sample averaging: the S-sample partial equals the sum of single-sample partials.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2604_04736_b200 import synth
from paper_2604_04736_b200.configs import layout
from . import torch_ref as R

TINY = dict(kind="vit", in_h=8, in_w=8, in_c=3, patch=4, dim=16, heads=2, depth=2, mlp=32, n_classes=3,
            loss="ce")


def _inputs(model, B, rho_mode="wide", seed=1):
    mu, rho = synth.init_params(model, seed=seed + 1, rho_mode=rho_mode)
    x, y, _ = synth.make_batch(model, B, seed=seed)
    return mu, rho, x, y


@pytest.mark.parametrize("aug", [False, True])
def test_vit_oracle_matches_torch_autograd(aug):
    mu, rho, x, y = _inputs(TINY, 3)
    S = 2
    acc = O.vit_elbo_partial(TINY, mu, rho, x, y, 3, 0, S, 0, S, 0x5EED, 4, O.AUG_PER_SAMPLE if aug else O.AUG_NONE)
    ref = R.vit_acc(TINY, mu, rho, x, y, S, 0x5EED, 4, aug=aug)
    P = (len(acc) - 1) // 2
    for a, b in ((acc[:P], ref[:P]), (acc[P:2 * P], ref[P:2 * P])):
        assert np.abs(a - b).max() <= 1e-10 * np.abs(b).max()
    assert abs(acc[-1] - ref[-1]) <= 1e-12 * abs(ref[-1])
    # every tensor receives gradient (no silently dropped term)
    for ti in layout(TINY):
        sl = slice(ti["offset"], ti["offset"] + ti["rows"] * ti["cols"])
        assert np.abs(acc[:P][sl]).max() > 0, ti


def test_vit_full_size_matches_torch_autograd():
    """The paper's ViT (32×32, 4×4 patches, 192 wide, 3 heads, 6 layers, MLP 768): one sample,
    two examples with augmentation."""
    model = dict(TINY, in_h=32, in_w=32, dim=192, heads=3, depth=6, mlp=768, n_classes=10)
    mu, rho, x, y = _inputs(model, 2, rho_mode="init")
    acc = O.vit_elbo_partial(model, mu, rho, x, y, 2, 0, 1, 0, 1, 7, 1, O.AUG_PER_SAMPLE)
    ref = R.vit_acc(model, mu, rho, x, y, 1, 7, 1, aug=True)
    P = (len(acc) - 1) // 2
    assert np.abs(acc[:P] - ref[:P]).max() <= 1e-9 * np.abs(ref[:P]).max()
    assert np.abs(acc[P:2 * P] - ref[P:2 * P]).max() <= 1e-9 * np.abs(ref[P:2 * P]).max()


def test_vit_finite_differences():
    """∂L/∂μ_i and ∂L/∂ρ_i (full ELBO: data term + KL/|D|) against 4th-order central
    differences with the same (seed, step): ≤ 1e-6 relative, for entries of every tensor kind."""
    mu, rho, x, y = _inputs(TINY, 2)
    S, D, seed, step = 2, 50.0, 11, 3
    ref = O.vit_elbo_step(TINY, mu, rho, x, y, S, seed, step, D)
    rng = np.random.default_rng(3)
    idx = []
    for ti in layout(TINY):
        n = ti["rows"] * ti["cols"]
        idx += list(ti["offset"] + rng.integers(0, n, 2))
    m64, r64 = mu.astype(np.float64), rho.astype(np.float64)

    def L(m, r):
        return O.vit_elbo_step(TINY, m, r, x, y, S, seed, step, D)["loss"]

    h = 1e-4
    for which, base, g in (("mu", m64, ref["grad_mu"]), ("rho", r64, ref["grad_rho"])):
        for i in idx:
            vals = []
            for k in (-2, -1, 1, 2):
                v = base.copy()
                v[i] += k * h
                vals.append(L(v, r64) if which == "mu" else L(m64, v))
            fd = (vals[0] - 8 * vals[1] + 8 * vals[2] - vals[3]) / (12 * h)
            assert abs(fd - g[i]) <= 1e-6 * max(abs(g[i]), 1e-3 * np.abs(g).max()), (which, i, fd, g[i])


def test_vit_sigma_to_zero_is_the_deterministic_network():
    mu, rho, x, y = _inputs(TINY, 3, rho_mode="tiny")
    S = 2
    acc = O.vit_elbo_partial(TINY, mu, rho, x, y, 3, 0, S, 0, S, 1, 0)
    ws = []
    m = torch.tensor(mu.astype(np.float64), requires_grad=True)
    for ti in layout(TINY):
        ws.append(m[ti["offset"]:ti["offset"] + ti["rows"] * ti["cols"]].reshape(ti["rows"], ti["cols"]))
    z = R.vit_forward(TINY, ws, torch.tensor(x.astype(np.float64)))
    loss = torch.nn.functional.cross_entropy(z, torch.tensor(y.astype(np.int64)))
    loss.backward()
    P = (len(acc) - 1) // 2
    assert abs(acc[-1] - float(loss)) <= 1e-12
    assert np.abs(acc[:P] - m.grad.numpy()).max() <= 1e-12 * np.abs(m.grad.numpy()).max() + 1e-14


def test_vit_sample_averaging_is_the_sum_of_single_samples():
    mu, rho, x, y = _inputs(TINY, 4)
    S = 3
    full = O.vit_elbo_partial(TINY, mu, rho, x, y, 4, 0, S, 0, S, 9, 2, O.AUG_PER_SAMPLE)
    parts = sum(O.vit_elbo_partial(TINY, mu, rho, x, y, 4, 0, S, s, s + 1, 9, 2, O.AUG_PER_SAMPLE)
                for s in range(S))
    assert np.abs(full - parts).max() <= 1e-13 * np.abs(full).max()
    # data sharding: examples [0, 2) and [2, 4) as two data groups
    half = [O.vit_elbo_partial(TINY, mu, rho, x[g * 2:(g + 1) * 2], y[g * 2:(g + 1) * 2], 4, 2 * g, S, 0, S, 9, 2,
                               O.AUG_PER_SAMPLE) for g in range(2)]
    assert np.abs(full - (half[0] + half[1])).max() <= 1e-13 * np.abs(full).max()
