"""Pins of the oracle's ELBO step (oracle/bnn_oracle.c) against things other than itself.

* closed forms: KL, loss assembly, uniform CE = ln 10
  (SPEC.md:649), log-softmax [1,2,3], KL vs a Monte-Carlo estimate;
* central finite differences of the whole ELBO (north_star: relative error ≤ 1e-6);
* an independent PyTorch fp64 formulation (library forward + autograd backward),
  including the σ→0 special case (deterministic network with weights μ);
* brute force: the S-sample step equals the sum of single-sample partials, and any
  K×G sharding of samples × examples sums to the single-rank result;
* the Bayesian linear regression closed form (expected data term, its gradients and the
  posterior predictive) against a large-S Monte Carlo run.
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_2604_04736_b200 import synth
from paper_2604_04736_b200.configs import MODELS, layout, n_params

from . import torch_ref

C1 = MODELS["mlp_8_16_1"]
TINY_CNN = dict(kind="resnet18", in_h=8, in_w=8, in_c=3, n_classes=10, base_width=4, loss="ce")


def _softplus_inv(s):
    return math.log(math.expm1(s))


def test_layout_matches_configs():
    for model in (C1, MODELS["mlp_784_1024_1024_10"], MODELS["resnet18_cifar"], TINY_CNN):
        assert O.n_params(model) == n_params(model)
        a = O.tensor_infos(model)
        b = layout(model)
        assert [(t["offset"], t["rows"], t["cols"]) for t in a] == \
               [(t["offset"], t["rows"], t["cols"]) for t in b]
    # |θ| values stated in SURVEY.md §8 (161 / 1,863,690 / 11,169,162)
    assert n_params(C1) == 161
    assert n_params(MODELS["mlp_784_1024_1024_10"]) == 1863690
    assert n_params(MODELS["resnet18_cifar"]) == 11169162


@pytest.mark.parametrize("mu,sigma,kl_each", [(0.0, 1.0, 0.0), (1.0, 1.0, 0.5),
                                              (0.0, 0.5, 0.3181471806)])
def test_kl_closed_form_values(mu, sigma, kl_each):
    model = dict(kind="mlp", widths=[3, 5], loss="mse")  # P = 20
    P = n_params(model)
    r = O.finalize(model, np.full(P, mu), np.full(P, _softplus_inv(sigma)),
                   np.zeros(2 * P + 1), 1000.0)
    assert r["kl"] == pytest.approx(kl_each * P, rel=1e-9, abs=1e-12)


def test_kl_vs_monte_carlo():
    """KL(q‖N(0,1)) closed form vs E_q[log q − log p] over 1e6 draws."""
    rng = np.random.default_rng(3)
    model = dict(kind="mlp", widths=[2, 2], loss="mse")  # P = 6
    P = n_params(model)
    mu = rng.uniform(-1, 1, P)
    sigma = rng.uniform(0.1, 2.0, P)
    rho = np.log(np.expm1(sigma))
    kl = O.finalize(model, mu, rho, np.zeros(2 * P + 1), 1.0)["kl"]
    w = mu + sigma * rng.standard_normal((1_000_000, P))
    logq = -0.5 * ((w - mu) / sigma) ** 2 - np.log(sigma)
    logp = -0.5 * w ** 2
    mc = (logq - logp).sum(axis=1)
    assert abs(mc.mean() - kl) < max(0.01 * P, 5 * mc.std() / 1000.0)


def test_loss_assembly_worked_value():
    """kl = 10, |D| = 1000, L_data = 0.5 → 0.51."""
    model = dict(kind="mlp", widths=[3, 5], loss="mse")  # P = 20; μ=1, σ=1 → KL = 10
    P = n_params(model)
    acc = np.zeros(2 * P + 1)
    acc[2 * P] = 0.5
    r = O.finalize(model, np.ones(P), np.full(P, _softplus_inv(1.0)), acc, 1000.0)
    assert r["kl"] == pytest.approx(10.0, rel=1e-12)
    assert r["loss"] == pytest.approx(0.51, rel=1e-12)


def test_uniform_ce_is_ln10_and_log_softmax_values():
    # μ = 0, σ → 0: all logits are 0 → CE = ln 10 for any label
    model = dict(kind="mlp", widths=[4, 10], loss="ce")
    P = n_params(model)
    x = np.random.default_rng(0).normal(size=(6, 4)).astype(np.float32)
    y = np.arange(6, dtype=np.int32) % 10
    acc = O.elbo_partial(model, np.zeros(P), np.full(P, -40.0), x, y, None, 6, 0, 3, 0, 3, 1, 0)
    assert acc[2 * P] == pytest.approx(math.log(10.0), rel=1e-12)
    # logits [1, 2, 3] via the bias → CE(y=0) = 2.4076, CE(y=2) = 0.4076
    model = dict(kind="mlp", widths=[1, 3], loss="ce")
    P = n_params(model)
    mu = np.array([0, 0, 0, 1, 2, 3], np.float64)
    for yl, val in ((0, 2.40760596), (2, 0.40760596)):
        acc = O.elbo_partial(model, mu, np.full(P, -40.0), np.ones((1, 1), np.float32),
                             np.array([yl], np.int32), None, 1, 0, 1, 0, 1, 1, 0)
        assert acc[2 * P] == pytest.approx(val, abs=1e-8)


def _fd_check(model, mu, rho, x, yc, yr, S, D, act, idx_mu, idx_rho, aug=0, h=1e-4, agg="sample"):
    """Fourth-order central differences: (8[L(+h) − L(−h)] − [L(+2h) − L(−2h)]) / 12h."""
    base = O.elbo_step(model, mu, rho, x, yc, yr, S, 11, 4, D, aug=aug, act=act, agg=agg)
    g_mu, g_rho = base["grad_mu"], base["grad_rho"]
    gmax = max(np.abs(g_mu).max(), np.abs(g_rho).max())

    def L(m, r):
        return O.elbo_step(model, m, r, x, yc, yr, S, 11, 4, D, aug=aug, act=act, agg=agg)["loss"]

    for vec, grad, idxs, which in ((mu, g_mu, idx_mu, "mu"), (rho, g_rho, idx_rho, "rho")):
        for i in idxs:
            def at(delta):
                v = vec.copy()
                v[i] += delta
                return L(v, rho) if which == "mu" else L(mu, v)
            fd = (8 * (at(h) - at(-h)) - (at(2 * h) - at(-2 * h))) / (12 * h)
            tol = 1e-6 * max(abs(grad[i]), 1e-3 * gmax)
            assert abs(fd - grad[i]) <= tol, (which, i, fd, grad[i])


@pytest.mark.parametrize("act", ["tanh", "relu"])
def test_finite_differences_mlp_regression(act):
    mu, rho = synth.init_params(C1, seed=2, rho_mode="wide")
    mu, rho = mu.astype(np.float64), rho.astype(np.float64)
    x, _, yr = synth.make_batch(C1, 32, seed=1)
    P = n_params(C1)
    idx = range(P) if act == "tanh" else range(0, P, 3)
    _fd_check(C1, mu, rho, x, None, yr, 4, 1024.0, act, idx, idx)


def test_finite_differences_mlp_classification():
    model = dict(kind="mlp", widths=[6, 7, 5], loss="ce")
    mu, rho = synth.init_params(model, seed=5, rho_mode="wide")
    x, yc, _ = synth.make_batch(model, 9, seed=4)
    P = n_params(model)
    _fd_check(model, mu.astype(np.float64), rho.astype(np.float64), x, yc, None, 3, 500.0,
              "tanh", range(P), range(P))


def test_finite_differences_cnn_tanh():
    mu, rho = synth.init_params(TINY_CNN, seed=6, rho_mode="wide")
    x, yc, _ = synth.make_batch(TINY_CNN, 2, seed=7)
    P = n_params(TINY_CNN)
    rng = np.random.default_rng(0)
    # include every tensor's first element plus random ones: stem, blocks, projections, FC
    idx = sorted(set([t["offset"] for t in layout(TINY_CNN)] + list(rng.integers(0, P, 30))))
    _fd_check(TINY_CNN, mu.astype(np.float64), rho.astype(np.float64), x, yc, None, 2, 100.0,
              "tanh", idx, idx[::2], aug=O.AUG_PER_SAMPLE)


def _cmp(a, b, rtol):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    assert np.linalg.norm(a - b) <= rtol * max(np.linalg.norm(b), 1e-300), \
        np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("rho_mode", ["wide", "tiny"])
@pytest.mark.parametrize("which", ["mlp_ce", "mlp_mse", "cnn"])
def test_against_torch_autograd(which, rho_mode):
    if which == "mlp_ce":
        model, B, S, aug = dict(kind="mlp", widths=[12, 16, 9, 4], loss="ce"), 7, 3, False
    elif which == "mlp_mse":
        model, B, S, aug = C1, 32, 4, False
    else:
        model = dict(kind="resnet18", in_h=16, in_w=16, in_c=3, n_classes=10, base_width=4,
                     loss="ce")
        B, S, aug = 3, 2, True
    mu, rho = synth.init_params(model, seed=8, rho_mode=rho_mode)
    x, yc, yr = synth.make_batch(model, B, seed=9)
    D = 777.0
    o = O.elbo_step(model, mu, rho, x, yc, yr, S, 0xABCDEF, 2, D,
                    aug=O.AUG_PER_SAMPLE if aug else O.AUG_NONE)
    t = torch_ref.elbo(model, mu, rho, x, yc, yr, S, 0xABCDEF, 2, D, aug=aug)
    assert o["loss"] == pytest.approx(t["loss"], rel=1e-12)
    assert o["kl"] == pytest.approx(t["kl"], rel=1e-12)
    assert o["L_data"] == pytest.approx(t["L_data"], rel=1e-12)
    _cmp(o["grad_mu"], t["grad_mu"], 1e-10)
    _cmp(o["grad_rho"], t["grad_rho"], 1e-10)
    if rho_mode == "tiny":
        # σ → 0 (ρ = −40, σ ≈ 4e-18): the data term and the data part of grad_μ are those of
        # the deterministic network with weights μ
        if not aug:
            l0, g0 = torch_ref.deterministic(model, mu, x, yc, yr)
            assert o["L_data"] == pytest.approx(l0, rel=1e-12)
            _cmp(o["grad_mu"] - mu.astype(np.float64) / D, g0, 1e-10)


def test_sample_and_example_sharding_sum_to_single_rank():
    model = dict(kind="mlp", widths=[10, 12, 5], loss="ce")
    mu, rho = synth.init_params(model, seed=1, rho_mode="wide")
    x, yc, _ = synth.make_batch(model, 8, seed=2)
    S, B = 6, 8
    full = O.elbo_partial(model, mu, rho, x, yc, None, B, 0, S, 0, S, 3, 1)
    # one sample at a time (brute force over samples)
    per_sample = sum(O.elbo_partial(model, mu, rho, x, yc, None, B, 0, S, s, s + 1, 3, 1)
                     for s in range(S))
    _cmp(per_sample, full, 1e-13)
    # K=3 sample groups × G=2 data groups
    tot = np.zeros_like(full)
    for k in range(3):
        for g in range(2):
            xs, ys = x[g * 4:(g + 1) * 4], yc[g * 4:(g + 1) * 4]
            tot += O.elbo_partial(model, mu, rho, xs, ys, None, B, g * 4, S, 2 * k, 2 * k + 2,
                                  3, 1)
    _cmp(tot, full, 1e-13)


def test_sharding_with_augmentation_is_rank_invariant():
    """Per-sample augmentation is keyed by global (s, b), so any sharding gives the same sum."""
    model = dict(kind="resnet18", in_h=8, in_w=8, in_c=3, n_classes=10, base_width=2, loss="ce")
    mu, rho = synth.init_params(model, seed=1)
    x, yc, _ = synth.make_batch(model, 4, seed=2)
    full = O.elbo_partial(model, mu, rho, x, yc, None, 4, 0, 2, 0, 2, 3, 1, O.AUG_PER_SAMPLE)
    tot = np.zeros_like(full)
    for k in range(2):
        for g in range(2):
            tot += O.elbo_partial(model, mu, rho, x[2 * g:2 * g + 2], yc[2 * g:2 * g + 2], None,
                                  4, 2 * g, 2, k, k + 1, 3, 1, O.AUG_PER_SAMPLE)
    _cmp(tot, full, 1e-13)
    none = O.elbo_partial(model, mu, rho, x, yc, None, 4, 0, 2, 0, 2, 3, 1, O.AUG_NONE)
    assert not np.allclose(none, full)


def test_bayesian_linear_regression_closed_form():
    """1-layer linear model with MSE: E_ε[(xᵀw+b−y)²] = (xᵀμ+μ_b−y)² + Σx_k²σ_k² + σ_b²."""
    d, B, S = 5, 4, 20000
    model = dict(kind="mlp", widths=[d, 1], loss="mse")
    rng = np.random.default_rng(4)
    mu = rng.normal(0, 0.5, d + 1)
    sigma = rng.uniform(0.2, 0.8, d + 1)
    rho = np.log(np.expm1(sigma))
    x = rng.normal(0, 1, (B, d)).astype(np.float32)
    y = rng.normal(0, 1, (B, 1)).astype(np.float32)
    xd, yd = x.astype(np.float64), y.astype(np.float64)[:, 0]
    m = xd @ mu[:d] + mu[d]
    v = (xd ** 2) @ sigma[:d] ** 2 + sigma[d] ** 2
    expect_L = np.mean((m - yd) ** 2 + v)
    expect_gmu = np.concatenate([2 * ((m - yd)[:, None] * xd).mean(0), [2 * (m - yd).mean()]])
    expect_gsig = np.concatenate([2 * (xd ** 2).mean(0) * sigma[:d], [2 * sigma[d]]])
    acc = O.elbo_partial(model, mu, rho, x, None, y, B, 0, S, 0, S, 21, 0)
    P = d + 1
    # Monte-Carlo standard errors from the per-sample outputs
    z = O.forward(model, mu, rho, x, 0, S, 21, 0)[:, :, 0]  # [S, B]
    ls = ((z - yd) ** 2).mean(1)
    assert abs(acc[2 * P] - expect_L) < 5 * ls.std() / math.sqrt(S)
    gs = np.concatenate([2 * ((z - yd)[:, :, None] * xd).mean(1), 2 * (z - yd).mean(1)[:, None]], 1)
    se = gs.std(0) / math.sqrt(S)
    assert np.all(np.abs(acc[:P] - expect_gmu) < 5 * se)
    eps = np.stack([np.concatenate([O.eps_fill(21, 0, s, 0, 0, 1, 0, d)[0],
                                    O.eps_fill(21, 0, s, 1, 0, 1, 0, 1)[0]])
                    for s in range(0, S, 40)])
    ge = gs[::40] * eps
    se_r = ge.std(0) / math.sqrt(S) * math.sqrt(40)
    assert np.all(np.abs(acc[P:2 * P] - expect_gsig) < 6 * se_r)
    mean, var = O.predict(model, mu, rho, x, S, 21, 0)
    assert np.all(np.abs(mean[:, 0] - m) < 5 * np.sqrt(v / S))
    assert np.all(np.abs(var[:, 0] - v) < 5 * v * math.sqrt(2.0 / S))


def test_predict_degenerate_and_consistency():
    model = dict(kind="mlp", widths=[6, 8, 3], loss="ce")
    mu, rho = synth.init_params(model, seed=3, rho_mode="wide")
    x, _, _ = synth.make_batch(model, 5, seed=4)
    mean, var = O.predict(model, mu, rho, x, 1, 9, 0)
    assert np.all(var == 0.0)                            # S = 1 → variance 0
    assert np.allclose(mean.sum(1), 1.0)                 # softmax probabilities
    mean, var = O.predict(model, mu, rho, x, 16, 9, 0)
    z = O.forward(model, mu, rho, x, 0, 16, 9, 0)
    p = np.exp(z - z.max(-1, keepdims=True))
    p /= p.sum(-1, keepdims=True)
    assert np.allclose(mean, p.mean(0), rtol=1e-12)
    assert np.allclose(var, p.var(0), rtol=1e-10, atol=1e-15)


# ---------------------------------------------------------------- Adam
def test_adam_matches_torch_optim_adam():
    """oracle.adam (Kingma & Ba Alg. 1, "e.g., Adam") pinned to the library
    routine torch.optim.Adam (fp64, no weight decay / amsgrad) over several steps with
    changing gradients, on a mixture of magnitudes including exact zeros."""
    import torch

    rng = np.random.default_rng(7)
    n = 1000
    theta0 = rng.standard_normal(n)
    lr, b1, b2, eps = 3e-3, 0.85, 0.995, 1e-6
    th = theta0.copy()
    m = np.zeros(n)
    v = np.zeros(n)
    p = torch.nn.Parameter(torch.tensor(theta0, dtype=torch.float64))
    opt = torch.optim.Adam([p], lr=lr, betas=(b1, b2), eps=eps)
    for t in range(1, 6):
        g = rng.standard_normal(n) * np.logspace(-6, 1, n)
        g[::97] = 0.0
        O.adam(th, g, m, v, lr, b1, b2, eps, t)
        p.grad = torch.tensor(g)
        opt.step()
        ref = p.detach().numpy()
        np.testing.assert_allclose(th, ref, rtol=0, atol=1e-14)
        st = opt.state[p]
        np.testing.assert_allclose(m, st["exp_avg"].numpy(), rtol=1e-11, atol=0)
        np.testing.assert_allclose(v, st["exp_avg_sq"].numpy(), rtol=1e-11, atol=0)


def test_adam_first_step_is_signed_lr():
    """Closed form: at t = 1, m̂ = g and v̂ = g², so θ moves by −α·g/(|g| + ε)."""
    g = np.array([2.0, -0.5, 0.0, 1e-3])
    th = np.zeros(4)
    m = np.zeros(4)
    v = np.zeros(4)
    O.adam(th, g, m, v, 0.1, 0.9, 0.999, 1e-8, 1)
    np.testing.assert_allclose(th, -0.1 * g / (np.abs(g) + 1e-8), rtol=1e-15, atol=0)


# ---------------------------------------------------------------- exact aggregation
@pytest.mark.parametrize("loss", ["ce", "mse"])
def test_mean_aggregation_finite_differences(loss):
    """The loss of the mean prediction: whole gradient vs central FD."""
    if loss == "ce":
        model, B, S, D = dict(kind="mlp", widths=[6, 7, 5], loss="ce"), 9, 3, 500.0
    else:
        model, B, S, D = C1, 16, 4, 1024.0
    mu, rho = synth.init_params(model, seed=5, rho_mode="wide")
    x, yc, yr = synth.make_batch(model, B, seed=4)
    P = n_params(model)
    _fd_check(model, mu.astype(np.float64), rho.astype(np.float64), x, yc, yr, S, D, "tanh",
              range(P), range(P), agg="mean")


@pytest.mark.parametrize("loss", ["ce", "mse"])
def test_mean_aggregation_against_torch_autograd(loss):
    """Independent fp64 torch formulation (mean of softmax probabilities / of predictions,
    F.nll_loss / F.mse_loss, autograd) on a ReLU MLP, σ wide."""
    model = dict(kind="mlp", widths=[12, 16, 9, 4], loss=loss)
    mu, rho = synth.init_params(model, seed=8, rho_mode="wide")
    x, yc, yr = synth.make_batch(model, 7, seed=9)
    o = O.elbo_step(model, mu, rho, x, yc, yr, 5, 0xABC, 2, 777.0, agg="mean")
    t = torch_ref.elbo(model, mu, rho, x, yc, yr, 5, 0xABC, 2, 777.0, agg="mean")
    assert o["loss"] == pytest.approx(t["loss"], rel=1e-12)
    assert o["L_data"] == pytest.approx(t["L_data"], rel=1e-11)
    _cmp(o["grad_mu"], t["grad_mu"], 1e-10)
    _cmp(o["grad_rho"], t["grad_rho"], 1e-10)


@pytest.mark.parametrize("loss", ["ce", "mse"])
def test_mean_aggregation_single_sample_equals_per_sample(loss):
    """S = 1: the mean prediction is the prediction, so both aggregations coincide."""
    model = dict(kind="mlp", widths=[10, 12, 5], loss=loss)
    mu, rho = synth.init_params(model, seed=3, rho_mode="wide")
    x, yc, yr = synth.make_batch(model, 6, seed=3)
    a = O.elbo_step(model, mu, rho, x, yc, yr, 1, 9, 0, 100.0)
    b = O.elbo_step(model, mu, rho, x, yc, yr, 1, 9, 0, 100.0, agg="mean")
    assert b["loss"] == pytest.approx(a["loss"], rel=1e-13)
    _cmp(b["grad_mu"], a["grad_mu"], 1e-12)
    _cmp(b["grad_rho"], a["grad_rho"], 1e-12)


def test_geometric_mean_gap_ce():
    """averaging per-sample CE (the sample-sharded approximation with one
    sample per GPU) is CE of the GEOMETRIC mean of the true-class probabilities, the exact loss
    CE of the ARITHMETIC mean; so L_sample = −mean_b ln GM_s(p) ≥ L_mean = −mean_b ln AM_s(p)
    (AM-GM). Statistics recomputed here with numpy from the oracle's per-sample logits."""
    model = dict(kind="mlp", widths=[10, 12, 5], loss="ce")
    mu, rho = synth.init_params(model, seed=4, rho_mode="wide")
    x, yc, _ = synth.make_batch(model, 8, seed=6)
    S, D = 6, 1e9
    z = O.forward(model, mu, rho, x, 0, S, 21, 0)
    p = np.exp(z - z.max(-1, keepdims=True))
    p /= p.sum(-1, keepdims=True)
    py = np.take_along_axis(p, yc[None, :, None].astype(np.int64), -1)[..., 0]  # [S, B]
    gm = np.exp(np.log(py).mean(0))
    am = py.mean(0)
    a = O.elbo_step(model, mu, rho, x, yc, None, S, 21, 0, D)
    b = O.elbo_step(model, mu, rho, x, yc, None, S, 21, 0, D, agg="mean")
    assert a["L_data"] == pytest.approx(float(-np.log(gm).mean()), rel=1e-12)
    assert b["L_data"] == pytest.approx(float(-np.log(am).mean()), rel=1e-12)
    assert a["L_data"] > b["L_data"]


def test_bias_variance_gap_mse():
    """MSE: mean_s (ŷ_s − y)² = (ȳ − y)² + Var_s(ŷ) (population), so the per-sample data term
    exceeds the exact one by the predictive variance of bnn_predict's oracle."""
    model = C1
    mu, rho = synth.init_params(model, seed=2, rho_mode="wide")
    x, _, yr = synth.make_batch(model, 32, seed=1)
    S = 8
    a = O.elbo_step(model, mu, rho, x, None, yr, S, 5, 1, 1e9)
    b = O.elbo_step(model, mu, rho, x, None, yr, S, 5, 1, 1e9, agg="mean")
    _, var = O.predict(model, mu, rho, x, S, 5, 1)
    assert a["L_data"] - b["L_data"] == pytest.approx(float(var.mean()), rel=1e-10)


def test_mean_aggregation_cnn_against_torch_autograd():
    """Exact aggregation on a tiny ResNet-18-shaped net with augmentation: oracle vs the
    independent torch formulation (mean softmax probability, F.nll_loss, autograd)."""
    model = dict(kind="resnet18", in_h=8, in_w=8, in_c=3, n_classes=10, base_width=4, loss="ce")
    # init σ: with σ up to 0.69 this BatchNorm-free net saturates the softmax and the true-class
    # mean probability underflows to 0 (an infinite loss, reading R21)
    mu, rho = synth.init_params(model, seed=8, rho_mode="init")
    x, yc, _ = synth.make_batch(model, 3, seed=9)
    o = O.elbo_step(model, mu, rho, x, yc, None, 2, 0xABC, 2, 777.0, aug=O.AUG_PER_SAMPLE, agg="mean")
    assert np.isfinite(o["loss"])
    t = torch_ref.elbo(model, mu, rho, x, yc, None, 2, 0xABC, 2, 777.0, aug=True, agg="mean")
    assert o["loss"] == pytest.approx(t["loss"], rel=1e-12)
    _cmp(o["grad_mu"], t["grad_mu"], 1e-10)
    _cmp(o["grad_rho"], t["grad_rho"], 1e-10)


# ---------------------------------------------------------------- Gaussian NLL of the predictive (f1)
def test_gnll_mean_aggregation_finite_differences():
    """Gaussian NLL with the samples' predictive mean and variance:
    whole gradient vs central FD (tanh MLP, σ wide so the predictive variance is not tiny)."""
    model = dict(kind="mlp", widths=[6, 7, 3], loss="gnll")
    mu, rho = synth.init_params(model, seed=5, rho_mode="wide")
    x, _, yr = synth.make_batch(model, 9, seed=4)
    P = n_params(model)
    _fd_check(model, mu.astype(np.float64), rho.astype(np.float64), x, None, yr, 4, 500.0, "tanh",
              range(P), range(P), agg="mean")


@pytest.mark.parametrize("rho_mode", ["wide", "init"])
def test_gnll_against_torch_autograd(rho_mode):
    """Oracle vs an independent torch formulation (torch.var, autograd) on a ReLU MLP."""
    model = dict(kind="mlp", widths=[12, 16, 9, 4], loss="gnll")
    mu, rho = synth.init_params(model, seed=8, rho_mode=rho_mode)
    x, _, yr = synth.make_batch(model, 7, seed=9)
    o = O.elbo_step(model, mu, rho, x, None, yr, 5, 0xABC, 2, 777.0, agg="mean")
    t = torch_ref.elbo(model, mu, rho, x, None, yr, 5, 0xABC, 2, 777.0, agg="mean")
    assert o["loss"] == pytest.approx(t["loss"], rel=1e-10)
    _cmp(o["grad_mu"], t["grad_mu"], 1e-8)
    _cmp(o["grad_rho"], t["grad_rho"], 1e-8)


# ---------------------------------------------------------------- MC dropout
MCD = dict(kind="mlp", widths=[12, 16, 9, 4], loss="mse", method="mcd", dropout_p=0.3)


def test_dropout_mask_statistics():
    """Keep rate 1 − p (binomial, 5σ) and independence across layers / samples / examples."""
    p, n = 0.3, 20000
    keep = np.array([O.dropout_keep(7, 3, 0, 1, b, j, p) for b in range(200) for j in range(100)])
    assert abs(keep.mean() - (1 - p)) <= 5 * np.sqrt(p * (1 - p) / n)
    other = np.array([O.dropout_keep(7, 3, 1, 1, b, j, p) for b in range(200) for j in range(100)])
    other_l = np.array([O.dropout_keep(7, 3, 0, 2, b, j, p) for b in range(200) for j in range(100)])
    agree = (1 - p) ** 2 + p ** 2
    for o in (other, other_l):
        assert abs(np.mean(keep == o) - agree) <= 5 * np.sqrt(agree * (1 - agree) / n)
    assert all(O.dropout_keep(7, 3, 0, 1, b, j, 0.0) for b in range(8) for j in range(8))


def test_mcd_p0_is_the_deterministic_network():
    """p = 0: every sample is the network with weights μ (torch, library layers + autograd)."""
    model = dict(MCD, dropout_p=0.0)
    mu, rho = synth.init_params(model, seed=3, rho_mode="wide")
    x, _, yr = synth.make_batch(model, 10, seed=4)
    o = O.elbo_step(model, mu, rho, x, None, yr, 3, 5, 1, 100.0)
    l0, g0 = torch_ref.deterministic(model, mu, x, None, yr)
    assert o["loss"] == pytest.approx(l0, rel=1e-12)
    _cmp(o["grad_mu"], g0, 1e-10)
    assert not np.any(o["grad_rho"]) and o["kl"] == 0.0


@pytest.mark.parametrize("agg", ["sample", "mean"])
def test_mcd_against_torch_autograd(agg):
    """MC-dropout step (per-sample MSE and MSE of the averaged predictions) against the
    independent torch formulation with the same keep masks."""
    mu, rho = synth.init_params(MCD, seed=8, rho_mode="wide")
    x, _, yr = synth.make_batch(MCD, 7, seed=9)
    o = O.elbo_step(MCD, mu, rho, x, None, yr, 4, 0xABC, 2, 777.0, agg=agg)
    t = torch_ref.elbo(MCD, mu, rho, x, None, yr, 4, 0xABC, 2, 777.0, agg=agg)
    assert o["loss"] == pytest.approx(t["loss"], rel=1e-12)
    _cmp(o["grad_mu"], t["grad_mu"], 1e-10)
    assert not np.any(o["grad_rho"])


def test_gnll_bayesian_linear_regression_large_S():
    """Gaussian NLL of the predictive (R24) on a 1-layer Bayesian linear regression: as S grows
    the sample mean and variance of the predictions converge to the closed forms
    m = xᵀμ + μ_b, v = Σ x_k² σ_k² + σ_b², so the data term converges to
    mean_b [½ ln(2π(v + 1e-6)) + (y − m)²/(2(v + 1e-6))]; with S = 20000 the oracle's value
    lies within the delta-method error of the closed form."""
    d, B, S = 5, 4, 20000
    model = dict(kind="mlp", widths=[d, 1], loss="gnll")
    rng = np.random.default_rng(11)
    mu = rng.normal(0, 0.5, d + 1)
    sigma = rng.uniform(0.2, 0.8, d + 1)
    rho = np.log(np.expm1(sigma))
    x = rng.normal(0, 1, (B, d)).astype(np.float32)
    y = rng.normal(0, 1, (B, 1)).astype(np.float32)
    xd, yd = x.astype(np.float64), y.astype(np.float64)[:, 0]
    m = xd @ mu[:d] + mu[d]
    v = (xd ** 2) @ sigma[:d] ** 2 + sigma[d] ** 2 + 1e-6
    expect = np.mean(0.5 * np.log(2 * np.pi * v) + (yd - m) ** 2 / (2 * v))
    o = O.elbo_step(model, mu, rho, x, None, y, S, 21, 0, 1e12, agg="mean")
    # error of the estimate: ∂L/∂m · SE(m) + ∂L/∂v · SE(v) per example, averaged
    dLdm = -(yd - m) / v
    dLdv = 0.5 / v - (yd - m) ** 2 / (2 * v ** 2)
    se = np.sqrt((dLdm ** 2) * v / S + (dLdv ** 2) * 2 * v ** 2 / S) / B  # per example (shared samples: add linearly)
    tol = 5 * np.sum(se)
    assert abs(o["L_data"] - expect) < tol, (o["L_data"], expect, tol)
    assert tol < 0.02 * abs(expect) + 0.02  # the check is informative
