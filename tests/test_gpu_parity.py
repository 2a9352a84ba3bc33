"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle.

Bars (BASELINE.json north_star, reading R15):
  * ε bit-exact (EPS-v1, docs/EPS.md);
  * FP32 mode: loss and every gradient tensor within 1e-4 relative;
  * BF16 tensor-core mode: within 2e-2 relative, against the EXACT oracle, in the parity
    regime of reading R26 (synth regime="positive": no ReLU decision within bf16 rounding of
    0, so the step is a smooth function of its operands; tests/test_conditioning.py pins that
    the BF16 mode's own weight rounding moves the exact step by < 1 % there);
  * sharded (virtual ranks, K×G grids) vs single rank: within 1e-5 relative.

"Within tol relative" for a tensor t is BOTH ‖Δ‖₂ ≤ tol·‖ref‖₂ AND, element by element,
|g_i − ref_i| ≤ tol·max_j |ref_j| (so one wrong row or tile of a large tensor fails even when
it is small against the tensor norm) — `_assert_close`.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2604_04736_b200 import synth
from paper_2604_04736_b200.configs import CONFIGS, MODELS

pytestmark = pytest.mark.gpu

C1 = MODELS["mlp_8_16_1"]
C2 = MODELS["mlp_784_1024_1024_10"]
RAGGED = dict(kind="mlp", widths=[100, 200, 130, 10], loss="ce")
RAGGED_MSE = dict(kind="mlp", widths=[36, 72, 3], loss="mse")


def _native():
    from paper_2604_04736_b200 import native
    return native


def _dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _per_tensor_rel(ctx, g, ref):
    out = []
    for t in ctx.tensors:
        sl = slice(t["offset"], t["offset"] + t["rows"] * t["cols"])
        out.append(_rel(g[sl], ref[sl]))
    return out


def _assert_close(ctx, g, ref, tol, what=""):
    """Per tensor: ‖g−ref‖₂ ≤ tol·‖ref‖₂ and elementwise |g_i−ref_i| ≤ tol·max|ref| (R15)."""
    g = np.asarray(g, np.float64)
    ref = np.asarray(ref, np.float64)
    assert np.all(np.isfinite(g)), what
    for t in ctx.tensors:
        sl = slice(t["offset"], t["offset"] + t["rows"] * t["cols"])
        d = np.abs(g[sl] - ref[sl])
        scale = np.abs(ref[sl]).max()
        if scale == 0.0:
            assert d.max() == 0.0, (what, t["t"], d.max())
            continue
        l2 = np.linalg.norm(d) / np.linalg.norm(ref[sl])
        el = d.max() / scale
        assert l2 <= tol and el <= tol, (what, "tensor", t["t"], "l2", l2, "elem", el,
                                         "at", int(np.argmax(d)))


def _acc_parts(ctx, acc):
    """(acc_μ, acc_ρ, L_data) of a bnn_elbo_partial buffer: the data term alone (no KL)."""
    a = acc.cpu().numpy().astype(np.float64)
    P = ctx.n_params
    return a[:P], a[ctx.acc_rho_offset:ctx.acc_rho_offset + P], a[ctx.acc_loss_offset]


def _inputs(model, B, rho_mode="init", seed=1, regime="kaiming"):
    if regime == "positive":
        mu, rho = synth.init_params(model, seed=seed + 1, regime="positive")
        x, yc, yr = synth.make_batch(model, B, seed=seed, regime="positive")
        return mu, rho, x, yc, yr
    mu, rho = synth.init_params(model, seed=seed + 1, rho_mode=rho_mode)
    x, yc, yr = synth.make_batch(model, B, seed=seed)
    return mu, rho, x, yc, yr


def _run_gpu(model, precision, mu, rho, x, yc, yr, S, seed, step, D, **kw):
    native = _native()
    B = x.shape[0]
    ctx = native.Context(model, precision=precision, max_B_loc=B, max_S_loc=S, dataset_size=D, **kw)
    y = _dev(yc) if yc is not None else _dev(yr)
    loss, gmu, grho = ctx.elbo_step(_dev(mu), _dev(rho), _dev(x), y, B, S, seed, step)
    torch.cuda.synchronize()
    return ctx, loss, gmu.cpu().numpy(), grho.cpu().numpy()


# ------------------------------------------------------------------ ε
@pytest.mark.parametrize("args", [(0x5EED, 0, 0, 0, 0, 64, 0, 1024),
                                  (0xFFFFFFFFFFFFFFFF, 7, 1048575, 4094, 123456, 3, 784, 261),
                                  (42, 123456789, 31, 5, 0, 1, 0, 4 * 4096 + 3)])
def test_eps_bit_exact(args):
    native = _native()
    g = native.eps_fill(*args).cpu().numpy()
    o = O.eps_fill(*args)
    assert g.dtype == o.dtype == np.float32
    assert np.array_equal(g.view(np.uint32), o.view(np.uint32))


def test_eps_transform_exhaustive_bit_exact():
    """All 2^24 radius and angle inputs: CUDA pieces ≡ oracle pieces, bit for bit (this covers
    the branch-free sqrt of csrc/eps.cuh against the oracle's IEEE sqrtf)."""
    native = _native()
    L = O.log24_all()
    R_ref = np.sqrt((L * np.float32(-2.0)).astype(np.float32))
    R = native.eps_transform_table(0).cpu().numpy()
    assert np.array_equal(R.view(np.uint32), R_ref.view(np.uint32))
    c_ref, s_ref = O.sincos2pi24_all()
    assert np.array_equal(native.eps_transform_table(1).cpu().numpy().view(np.uint32), c_ref.view(np.uint32))
    assert np.array_equal(native.eps_transform_table(2).cpu().numpy().view(np.uint32), s_ref.view(np.uint32))


def test_eps_bench_kernel_runs():
    native = _native()
    sink = torch.zeros(148 * 4, device="cuda")
    native.eps_bench(1 << 20, 9, sink, 148 * 4)
    torch.cuda.synchronize()
    tot = float(sink.double().sum())
    # mean of 4M normals: |Σ| ≲ 5·sqrt(4M)
    assert abs(tot) < 5 * (4 << 20) ** 0.5


# ------------------------------------------------------------------ full steps
CASES = [
    ("C1", C1, 32, 4, "init"),
    ("C1_wide", C1, 32, 4, "wide"),
    ("ragged_ce", RAGGED, 77, 3, "wide"),
    ("ragged_mse", RAGGED_MSE, 40, 5, "init"),
    ("C2_S4", C2, 256, 4, "init"),
]


@pytest.mark.parametrize("name,model,B,S,rho_mode", CASES)
def test_elbo_step_fp32_matches_oracle(name, model, B, S, rho_mode):
    mu, rho, x, yc, yr = _inputs(model, B, rho_mode)
    D = 1000.0
    ctx, loss, gmu, grho = _run_gpu(model, "fp32", mu, rho, x, yc, yr, S, 0xC0FFEE, 3, D)
    ref = O.elbo_step(model, mu, rho, x, yc, yr, S, 0xC0FFEE, 3, D)
    assert abs(loss - ref["loss"]) <= 1e-4 * abs(ref["loss"])
    _assert_close(ctx, gmu, ref["grad_mu"], 1e-4, "grad_mu")
    _assert_close(ctx, grho, ref["grad_rho"], 1e-4, "grad_rho")


@pytest.mark.parametrize("name,model,B,S,rho_mode", CASES)
def test_elbo_step_bf16_matches_exact_oracle(name, model, B, S, rho_mode):
    """BF16 tcgen05 path against the exact fp64 oracle at 2e-2 (north_star) in the parity
    regime (R26): the whole step (loss, grad_μ, grad_ρ) and its data term alone (acc_μ, acc_ρ
    of bnn_elbo_partial, so the KL part of grad_ρ cannot hide the ε-weighted sum)."""
    mu, rho, x, yc, yr = _inputs(model, B, regime="positive")
    D = 1000.0
    ctx, loss, gmu, grho = _run_gpu(model, "bf16", mu, rho, x, yc, yr, S, 0xC0FFEE, 3, D)
    ref = O.elbo_step(model, mu, rho, x, yc, yr, S, 0xC0FFEE, 3, D)
    assert abs(loss - ref["loss"]) <= 2e-2 * abs(ref["loss"])
    _assert_close(ctx, gmu, ref["grad_mu"], 2e-2, "grad_mu")
    _assert_close(ctx, grho, ref["grad_rho"], 2e-2, "grad_rho")
    acc = ctx.elbo_partial(_dev(mu), _dev(rho), _dev(x), _dev(yc) if yc is not None else _dev(yr), B, S,
                           0xC0FFEE, 3)
    am, ar, al = _acc_parts(ctx, acc)
    ra = O.elbo_partial(model, mu, rho, x, yc, yr, B, 0, S, 0, S, 0xC0FFEE, 3)
    P = ctx.n_params
    _assert_close(ctx, am, ra[:P], 2e-2, "acc_mu")
    _assert_close(ctx, ar, ra[P:2 * P], 2e-2, "acc_rho")
    assert abs(al - ra[-1]) <= 2e-2 * abs(ra[-1])


@pytest.mark.parametrize("name,model,B,S,rho_mode", CASES)
def test_elbo_step_bf16_matches_emulating_oracle(name, model, B, S, rho_mode):
    """The BF16 MLP kernels in the Kaiming regime (ReLU near-ties included) against the oracle
    with R14's rounding points (emu, pinned against an independent numpy emulation in
    tests/test_oracle_bf16_emulation.py): ≤ 2e-3 per tensor, ≤ 1e-2 of the tensor max per
    element (a near-tie of a bf16 rounding decided by fp32 accumulation order moves one element
    by one bf16 ulp)."""
    mu, rho, x, yc, yr = _inputs(model, B, rho_mode)
    D = 1000.0
    ctx, loss, gmu, grho = _run_gpu(model, "bf16", mu, rho, x, yc, yr, S, 0xC0FFEE, 3, D)
    emu = O.elbo_step(model, mu, rho, x, yc, yr, S, 0xC0FFEE, 3, D, emu=True)
    assert abs(loss - emu["loss"]) <= 1e-4 * abs(emu["loss"])
    assert max(_per_tensor_rel(ctx, gmu, emu["grad_mu"])) <= 2e-3
    assert max(_per_tensor_rel(ctx, grho, emu["grad_rho"])) <= 2e-3
    _assert_close(ctx, gmu, emu["grad_mu"], 1e-2, "grad_mu")
    _assert_close(ctx, grho, emu["grad_rho"], 1e-2, "grad_rho")


def test_sigma_to_zero_limit_gpu():
    """ρ = −40: the step is the deterministic network with weights μ (plus the KL terms)."""
    mu, rho, x, yc, yr = _inputs(RAGGED, 33, "tiny")
    ctx, loss, gmu, grho = _run_gpu(RAGGED, "fp32", mu, rho, x, yc, yr, 2, 1, 0, 500.0)
    ref = O.elbo_step(RAGGED, mu, rho, x, yc, yr, 2, 1, 0, 500.0)
    assert _rel(gmu, ref["grad_mu"]) < 1e-4
    assert _rel(grho, ref["grad_rho"]) < 1e-4


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_sample_chunking_equals_single_chunk(precision):
    mu, rho, x, yc, yr = _inputs(RAGGED, 64, "wide")
    _, l1, g1, r1 = _run_gpu(RAGGED, precision, mu, rho, x, yc, yr, 6, 5, 1, 100.0)
    _, l2, g2, r2 = _run_gpu(RAGGED, precision, mu, rho, x, yc, yr, 6, 5, 1, 100.0, sample_chunk=4)
    assert _rel(g2, g1) < 1e-5 and _rel(r2, r1) < 1e-5
    assert abs(l2 - l1) <= 1e-5 * abs(l1)


def test_deterministic_bitwise():
    mu, rho, x, yc, yr = _inputs(C2, 128, "init")
    _, l1, g1, r1 = _run_gpu(C2, "bf16", mu, rho, x, yc, yr, 4, 5, 1, 100.0)
    _, l2, g2, r2 = _run_gpu(C2, "bf16", mu, rho, x, yc, yr, 4, 5, 1, 100.0)
    assert l1 == l2 and np.array_equal(g1, g2) and np.array_equal(r1, r2)


# ------------------------------------------------------------------ sharding (virtual ranks)
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("mode,K,G", [("sample", 4, 1), ("data", 1, 2), ("hybrid", 2, 2)])
def test_virtual_rank_sharding_equals_single_rank(mode, K, G, precision):
    native = _native()
    model, B, S, D = RAGGED, 64, 8, 321.0
    mu, rho, x, yc, yr = _inputs(model, B, "wide")
    mu_d, rho_d = _dev(mu), _dev(rho)
    single = native.Context(model, precision=precision, max_B_loc=B, max_S_loc=S, dataset_size=D)
    acc1 = single.elbo_partial(mu_d, rho_d, _dev(x), _dev(yc), B, S, 77, 9)
    l1, g1, r1 = single.finalize(mu_d, rho_d, acc1)
    total = None
    world = K * G
    for rank in range(world):
        ctx = native.Context(model, precision=precision, mode=mode, K=K, G=G, rank=rank,
                             world=world, max_B_loc=B // G, max_S_loc=S // K, dataset_size=D)
        g = rank % G
        xs, ys = x[g * (B // G):(g + 1) * (B // G)], yc[g * (B // G):(g + 1) * (B // G)]
        acc = ctx.elbo_partial(mu_d, rho_d, _dev(xs), _dev(ys), B, S, 77, 9)
        total = acc if total is None else total + acc  # fixed rank order
    l2, g2, r2 = single.finalize(mu_d, rho_d, total)
    torch.cuda.synchronize()
    tol = 1e-5  # north_star: single-GPU vs sharded within 1e-5 relative
    assert _rel(g2.cpu().numpy(), g1.cpu().numpy()) < tol
    assert _rel(r2.cpu().numpy(), r1.cpu().numpy()) < tol
    assert abs(float(l2) - float(l1)) <= tol * abs(float(l1))


# ------------------------------------------------------------------ exact aggregation
MEAN_CASES = [
    ("ragged_ce_mean", dict(RAGGED, loss="ce_mean"), 77, 6, "wide"),
    ("ragged_ce_mean_init", dict(RAGGED, loss="ce_mean"), 77, 6, "init"),
    ("ragged_mse_mean", dict(RAGGED_MSE, loss="mse_mean"), 40, 5, "init"),
    ("C2_ce_mean_S8", dict(C2, loss="ce_mean"), 256, 8, "init"),
]


def _base(model):
    return dict(model, loss=model["loss"].replace("_mean", ""))


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-4), ("bf16", 2e-2)])
@pytest.mark.parametrize("name,model,B,S,rho_mode", MEAN_CASES)
def test_mean_aggregation_matches_oracle(name, model, B, S, rho_mode, precision, tol):
    """Loss of the mean prediction through bnn_elbo_step: loss and every
    gradient tensor against oracle.elbo_step(agg="mean"), FP32 1e-4 (Kaiming regime, σ as
    named) / BF16 2e-2 (parity regime R26)."""
    regime = "positive" if precision == "bf16" else "kaiming"
    mu, rho, x, yc, yr = _inputs(_base(model), B, rho_mode, regime=regime)
    D = 1000.0
    ctx, loss, gmu, grho = _run_gpu(model, precision, mu, rho, x, yc, yr, S, 0xC0FFEE, 3, D)
    ref = O.elbo_step(_base(model), mu, rho, x, yc, yr, S, 0xC0FFEE, 3, D, agg="mean")
    assert abs(loss - ref["loss"]) <= tol * abs(ref["loss"])
    _assert_close(ctx, gmu, ref["grad_mu"], tol, "grad_mu")
    _assert_close(ctx, grho, ref["grad_rho"], tol, "grad_rho")


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("loss", ["ce_mean", "mse_mean"])
@pytest.mark.parametrize("mode,K,G,chunk", [("sample", 4, 1, 0), ("hybrid", 2, 2, 1), ("sample", 1, 1, 2)])
def test_mean_aggregation_virtual_ranks_equal_single_rank(loss, mode, K, G, chunk, precision):
    """Exact mode sharded: each rank's statistic (bnn_mean_stats), summed over the sample groups
    of its data group, then bnn_elbo_partial_mean; Σ acc → finalize equals the single rank
    within 1e-5 (north_star). chunk > 0 also exercises the recomputed forward of a
    multi-chunk step."""
    native = _native()
    base = RAGGED if loss == "ce_mean" else RAGGED_MSE
    model = dict(base, loss=loss)
    B, S, D = 64, 8, 321.0
    mu, rho, x, yc, yr = _inputs(base, B, "wide")
    y = yc if loss == "ce_mean" else yr
    mu_d, rho_d = _dev(mu), _dev(rho)
    single = native.Context(model, precision=precision, max_B_loc=B, max_S_loc=S, dataset_size=D)
    l1, g1, r1 = single.elbo_step(mu_d, rho_d, _dev(x), _dev(y), B, S, 77, 9)
    width = 1 if loss == "ce_mean" else base["widths"][-1]
    world = K * G
    ctxs, shards = [], []
    for rank in range(world):
        ctx = native.Context(model, precision=precision, mode=mode, K=K, G=G, rank=rank, world=world,
                             max_B_loc=B // G, max_S_loc=S // K, dataset_size=D, sample_chunk=chunk)
        g = rank % G
        sl = slice(g * (B // G), (g + 1) * (B // G))
        ctxs.append(ctx)
        shards.append((_dev(x[sl]), _dev(y[sl])))
    stats = [c.mean_stats(mu_d, rho_d, xs, ys, B, S, 77, 9, width) for c, (xs, ys) in zip(ctxs, shards)]
    total = None
    for rank, (c, (xs, ys)) in enumerate(zip(ctxs, shards)):
        g = rank % G
        gst = None
        for r in range(g, world, G):  # the sample groups of data group g, rank order
            gst = stats[r].clone() if gst is None else gst + stats[r]
        acc = c.elbo_partial_mean(mu_d, rho_d, xs, ys, B, S, 77, 9, gst)
        total = acc if total is None else total + acc
    l2, g2, r2 = single.finalize(mu_d, rho_d, total)
    torch.cuda.synchronize()
    tol = 1e-5
    assert _rel(g2.cpu().numpy(), g1.cpu().numpy()) < tol
    assert _rel(r2.cpu().numpy(), r1.cpu().numpy()) < tol
    assert abs(float(l2) - float(l1)) <= tol * abs(float(l1))


@pytest.mark.parametrize("loss", ["ce", "ce_mean", "mse_mean"])
def test_nccl_communicator_world1_equals_no_communicator(loss):
    """The NCCL code path on one GPU (communicator of world 1: the acc allreduce and, for the
    mean-prediction losses, the statistic allgather + merge) gives the no-communicator result
    bit for bit."""
    native = _native()
    base = RAGGED if loss != "mse_mean" else RAGGED_MSE
    model = dict(base, loss=loss)
    B, S = 48, 4
    mu, rho, x, yc, yr = _inputs(base, B, "init")
    y = _dev(yc if yc is not None else yr)
    out = []
    for uid in (None, native.get_unique_id()):
        ctx = native.Context(model, precision="bf16", max_B_loc=B, max_S_loc=S, dataset_size=500.0,
                             uid=uid)
        l, g, r = ctx.elbo_step(_dev(mu), _dev(rho), _dev(x), y, B, S, 3, 4)
        torch.cuda.synchronize()
        out.append((l, g.cpu(), r.cpu()))
        ctx.close()
    assert out[0][0] == out[1][0]
    assert torch.equal(out[0][1], out[1][1]) and torch.equal(out[0][2], out[1][2])


# ------------------------------------------------------------------ predict
@pytest.mark.parametrize("precision,tol,regime", [("fp32", 1e-4, "kaiming"), ("bf16", 2e-2, "positive")])
def test_predict_matches_oracle(precision, tol, regime):
    """Predictive mean and population variance over S samples (R16) against the oracle,
    elementwise (|Δ| ≤ tol·max|ref|) and per tensor. The variance is a difference of nearly
    equal sample predictions, so its error is the prediction's error × mean/spread: FP32 at
    1e-3; BF16 (positive regime, σ comparable to the μ spread) at 2e-2."""
    native = _native()
    model, B, S = RAGGED, 50, 8
    mu, rho, x, _, _ = _inputs(model, B, "wide", regime=regime)
    ctx = native.Context(model, precision=precision, max_B_loc=B, max_S_loc=S, dataset_size=1.0)
    mean, var = ctx.predict(_dev(mu), _dev(rho), _dev(x), S, 3, 0)
    rm, rv = O.predict(model, mu, rho, x, S, 3, 0)
    mean, var = mean.cpu().numpy().astype(np.float64), var.cpu().numpy().astype(np.float64)
    vtol = 1e-3 if precision == "fp32" else tol
    assert _rel(mean, rm) < tol and np.abs(mean - rm).max() <= tol * np.abs(rm).max()
    assert _rel(var, rv) < vtol and np.abs(var - rv).max() <= vtol * np.abs(rv).max()


# ------------------------------------------------------------------ fused Adam
def _adam_case(model, precision, B, S, steps, lr=1e-2, b1=0.9, b2=0.999, eps=1e-8, rho_mode="wide"):
    native = _native()
    mu, rho, x, yc, yr = _inputs(model, B, rho_mode)
    D = 1000.0
    ctx = native.Context(model, precision=precision, max_B_loc=B, max_S_loc=S, dataset_size=D)
    y = _dev(yc) if yc is not None else _dev(yr)
    dmu, drho, dx = _dev(mu), _dev(rho), _dev(x)
    mom = [torch.zeros_like(dmu) for _ in range(4)]
    gmu, grho = torch.empty_like(dmu), torch.empty_like(drho)
    ref_mu, ref_rho = mu.astype(np.float64).copy(), rho.astype(np.float64).copy()
    rm = [np.zeros(ref_mu.size) for _ in range(4)]
    out = []
    for t in range(1, steps + 1):
        loss = ctx.elbo_step_adam(dmu, drho, dx, y, B, S, 0xADA, 10 + t, mom, t=t, lr=lr, beta1=b1,
                                  beta2=b2, eps=eps, grad_mu=gmu, grad_rho=grho)
        ref = O.elbo_step(model, ref_mu, ref_rho, x, yc, yr, S, 0xADA, 10 + t, D)
        O.adam(ref_mu, ref["grad_mu"], rm[0], rm[1], lr, b1, b2, eps, t)
        O.adam(ref_rho, ref["grad_rho"], rm[2], rm[3], lr, b1, b2, eps, t)
        torch.cuda.synchronize()
        out.append(dict(loss=loss, ref_loss=ref["loss"], gmu=gmu.cpu().numpy(), grho=grho.cpu().numpy(),
                        ref_gmu=ref["grad_mu"], ref_grho=ref["grad_rho"], mu=dmu.cpu().numpy(),
                        rho=drho.cpu().numpy(), ref_mu=ref_mu.copy(), ref_rho=ref_rho.copy(),
                        mom=[m.cpu().numpy() for m in mom], ref_mom=[m.copy() for m in rm]))
    return ctx, mu, rho, out


def _displacement_ok(theta, ref, theta0, lr, steps):
    """Adam moves an element by ≈ lr·sign(ĝ) per step, so an element whose reference gradient
    is below the fp32 error level can legitimately move the other way; the displacement is
    compared as a whole (≤ 5e-3 relative) and elementwise to 1e-3·lr except for ≤ 0.1 % of
    elements (those near-zero-gradient sign ties)."""
    d, dr = theta - theta0, ref - theta0
    rel = np.linalg.norm(d - dr) / max(np.linalg.norm(dr), 1e-300)
    bad = np.mean(np.abs(d - dr) > 1e-3 * lr * steps + 1e-6 * np.abs(ref))
    return rel, bad


@pytest.mark.parametrize("model,B,S", [(C1, 32, 4), (RAGGED, 77, 3), (RAGGED_MSE, 40, 5)])
def test_fused_adam_step_matches_oracle_fp32(model, B, S):
    """bnn_elbo_step_adam (FP32 mode) over 3 updates against oracle.elbo_step + oracle.adam
    (Kingma & Ba, pinned to torch.optim.Adam): loss and gradients ≤ 1e-4 per tensor, the
    moments ≤ 1e-4 / 2e-4, μ and ρ displacements as _displacement_ok."""
    lr, steps = 1e-2, 3
    ctx, mu0, rho0, out = _adam_case(model, "fp32", B, S, steps, lr=lr)
    for k, o in enumerate(out):
        assert abs(o["loss"] - o["ref_loss"]) <= 1e-4 * abs(o["ref_loss"]), k
        _assert_close(ctx, o["gmu"], o["ref_gmu"], 1e-4, ("grad_mu", k))
        _assert_close(ctx, o["grho"], o["ref_grho"], 1e-4, ("grad_rho", k))
    last = out[-1]
    assert _rel(last["mom"][0], last["ref_mom"][0]) <= 1e-3
    assert _rel(last["mom"][2], last["ref_mom"][2]) <= 1e-3
    assert _rel(last["mom"][1], last["ref_mom"][1]) <= 2e-3
    assert _rel(last["mom"][3], last["ref_mom"][3]) <= 2e-3
    for th, ref, th0 in ((last["mu"], last["ref_mu"], mu0), (last["rho"], last["ref_rho"], rho0)):
        rel, bad = _displacement_ok(th.astype(np.float64), ref, th0.astype(np.float64), lr, steps)
        assert rel <= 5e-3 and bad <= 1e-3, (rel, bad)


def test_fused_adam_bf16_consistent_with_plain_step():
    """BF16 C2-shaped step: the fused step's gradients are bit-identical to bnn_elbo_step's on
    the same inputs, and its first update is exactly m = RN((1−β1)·g), v = RN((1−β2)·RN(g²)),
    θ' = θ − lr·(m/bc1)/(√(v/bc2)+ε) in fp32."""
    native = _native()
    model, B, S = C2, 256, 4
    mu, rho, x, yc, _ = _inputs(model, B, "init")
    ctx = native.Context(model, precision="bf16", max_B_loc=B, max_S_loc=S, dataset_size=60000.0)
    y = _dev(yc)
    loss0, g0, r0 = ctx.elbo_step(_dev(mu), _dev(rho), _dev(x), y, B, S, 5, 1)
    dmu, drho = _dev(mu), _dev(rho)
    mom = [torch.zeros_like(dmu) for _ in range(4)]
    gmu, grho = torch.empty_like(dmu), torch.empty_like(dmu)
    lr, b1, b2, eps = 1e-3, 0.9, 0.999, 1e-8
    loss1 = ctx.elbo_step_adam(dmu, drho, _dev(x), y, B, S, 5, 1, mom, t=1, lr=lr, beta1=b1, beta2=b2,
                               eps=eps, grad_mu=gmu, grad_rho=grho)
    torch.cuda.synchronize()
    assert loss1 == loss0
    assert torch.equal(gmu, g0) and torch.equal(grho, r0)
    # the library rounds β to fp32 and forms 1 − β and the bias corrections in double
    omb1 = float(np.float32(1.0 - float(np.float32(b1))))
    omb2 = float(np.float32(1.0 - float(np.float32(b2))))
    assert torch.equal(mom[0], g0 * omb1) and torch.equal(mom[2], r0 * omb1)
    assert torch.equal(mom[1], (g0 * g0) * omb2) and torch.equal(mom[3], (r0 * r0) * omb2)
    for th, th0, g, m, v in ((dmu, _dev(mu), g0, mom[0], mom[1]), (drho, _dev(rho), r0, mom[2], mom[3])):
        bc1, bc2 = omb1, omb2  # t = 1
        expect = th0 - lr * (m / bc1) / (torch.sqrt(v / bc2) + eps)
        assert torch.allclose(th, expect, rtol=0, atol=1e-6)
        assert float((th - th0).abs().max()) <= 1.01 * lr


# ------------------------------------------------------------------ full BASELINE size (C2)
def test_c2_full_size_bf16_loss_and_logits():
    """BASELINE.json configs[1] at full size (B=256, S=64), bench launch configuration:
    the loss needs every sample's forward pass (the oracle's forward only, ≈30 GFLOP fp64);
    gradients at full size are checked in test_c2_full_size_bf16_gradients."""
    cfg = CONFIGS["C2"]
    mu, rho, x, yc, _ = _inputs(C2, cfg["B"], "init")
    ctx, loss, gmu, grho = _run_gpu(C2, "bf16", mu, rho, x, yc, None, cfg["S"], 0x5EED, 0, cfg["D"])
    z = O.forward(C2, mu, rho, x, 0, cfg["S"], 0x5EED, 0)
    lse = np.log(np.exp(z - z.max(-1, keepdims=True)).sum(-1)) + z.max(-1)
    L_data = float((lse - np.take_along_axis(z, yc[None, :, None].astype(np.int64), -1)[..., 0]).mean())
    kl = O.finalize(C2, mu, rho, np.zeros(2 * ctx.n_params + 1), cfg["D"])["kl"]
    ref = L_data + kl / cfg["D"]
    assert abs(loss - ref) <= 2e-2 * abs(ref)
    assert np.all(np.isfinite(gmu)) and np.all(np.isfinite(grho))


@pytest.mark.slow
def test_c2_full_size_bf16_gradients():
    cfg = CONFIGS["C2"]
    mu, rho, x, yc, _ = _inputs(C2, cfg["B"], "init")
    ctx, loss, gmu, grho = _run_gpu(C2, "bf16", mu, rho, x, yc, None, cfg["S"], 0x5EED, 0, cfg["D"])
    ref = O.elbo_step(C2, mu, rho, x, yc, None, cfg["S"], 0x5EED, 0, cfg["D"])
    _assert_close(ctx, gmu, ref["grad_mu"], 2e-2, "grad_mu")
    _assert_close(ctx, grho, ref["grad_rho"], 2e-2, "grad_rho")


# ------------------------------------------------------------------ ResNet-18-shaped CNN (FP32 path)
SMALL_CNN = dict(kind="resnet18", in_h=16, in_w=16, in_c=3, n_classes=10, base_width=8, loss="ce")


@pytest.mark.parametrize("rho_mode", ["wide", "init"])
@pytest.mark.parametrize("aug", ["none", "per_sample"])
def test_cnn_fp32_matches_oracle(aug, rho_mode):
    """FP32 SIMT CNN path ≤ 1e-4. σ wide saturates this BatchNorm-free net (loss ~5e7); the
    init σ (loss ~25) is the informative case (step key 7: no fp32/fp64 ReLU tie, R23)."""
    model, B, S, D = SMALL_CNN, 6, 3, 45000.0
    mu, rho, x, yc, _ = _inputs(model, B, rho_mode)
    step = 5 if rho_mode == "wide" else 7
    ref = O.elbo_step(model, mu, rho, x, yc, None, S, 0xBEEF, step, D,
                      aug=O.AUG_PER_SAMPLE if aug == "per_sample" else O.AUG_NONE)
    ctx, loss, gmu, grho = _run_gpu(model, "fp32", mu, rho, x, yc, None, S, 0xBEEF, step, D, aug=aug)
    assert abs(loss - ref["loss"]) <= 1e-4 * abs(ref["loss"])
    _assert_close(ctx, gmu, ref["grad_mu"], 1e-4, "grad_mu")
    _assert_close(ctx, grho, ref["grad_rho"], 1e-4, "grad_rho")


def test_cnn_fp32_hybrid_virtual_ranks_with_augmentation():
    native = _native()
    model, B, S, D = SMALL_CNN, 4, 4, 100.0
    mu, rho, x, yc, _ = _inputs(model, B, "wide")
    mu_d, rho_d = _dev(mu), _dev(rho)
    single = native.Context(model, precision="fp32", max_B_loc=B, max_S_loc=S, dataset_size=D,
                            aug="per_sample")
    l1, g1, r1 = single.finalize(mu_d, rho_d, single.elbo_partial(mu_d, rho_d, _dev(x), _dev(yc), B, S, 3, 1))
    total = None
    for rank in range(4):
        ctx = native.Context(model, precision="fp32", mode="hybrid", K=2, G=2, rank=rank, world=4,
                             max_B_loc=B // 2, max_S_loc=S // 2, dataset_size=D, aug="per_sample")
        g = rank % 2
        acc = ctx.elbo_partial(mu_d, rho_d, _dev(x[2 * g:2 * g + 2]), _dev(yc[2 * g:2 * g + 2]), B, S, 3, 1)
        total = acc if total is None else total + acc
    l2, g2, r2 = single.finalize(mu_d, rho_d, total)
    torch.cuda.synchronize()
    assert _rel(g2.cpu().numpy(), g1.cpu().numpy()) < 1e-5
    assert _rel(r2.cpu().numpy(), r1.cpu().numpy()) < 1e-5


def test_cnn_fp32_predict():
    native = _native()
    model, B, S = SMALL_CNN, 5, 4
    mu, rho, x, _, _ = _inputs(model, B, "wide")
    ctx = native.Context(model, precision="fp32", max_B_loc=B, max_S_loc=S, dataset_size=1.0)
    mean, var = ctx.predict(_dev(mu), _dev(rho), _dev(x), S, 3, 0)
    rm, rv = O.predict(model, mu, rho, x, S, 3, 0)
    assert _rel(mean.cpu().numpy(), rm) < 1e-4
    assert _rel(var.cpu().numpy(), rv) < 1e-3


# ------------------------------------------------------------------ ResNet-18-shaped CNN (BF16 tcgen05 path)
BF16_CNN = dict(kind="resnet18", in_h=16, in_w=16, in_c=3, n_classes=10, base_width=64, loss="ce")


def _cnn_layerwise(ctx, model, mu, rho, x, yc, S, B, seed, step, a, pairs, tol_out, tol_grad):
    """Every stored activation and stored gradient of the listed (sample, example) pairs, layer
    by layer, against the EXACT oracle's layer dump: per (pair, layer) ‖Δ‖₂ ≤ tol·‖ref‖₂ and
    |Δ_i| ≤ tol·max|ref| — no medians, every pair and layer on its own."""
    n_layers = len(ctx.tensors) // 2
    outs = [ctx.layer_output(l, 0).cpu().numpy().astype(np.float64) for l in range(n_layers)]
    grads = [ctx.layer_output(l, 1).cpu().numpy().astype(np.float64) if l < n_layers - 1 else None
             for l in range(n_layers)]
    sizes = [o.size // (S * B) for o in outs]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    for s, b in pairs:
        i = s * B + b
        d = {g: O.layer_dump(model, mu, rho, x, yc, None, b, s, seed, step, aug=a, grad=g)
             for g in (False, True)}
        for l in range(n_layers):
            k = slice(i * sizes[l], (i + 1) * sizes[l])
            o = slice(offs[l], offs[l + 1])
            for name, gpu, ref, tol in (("out", outs[l], d[False], tol_out), ("grad", grads[l], d[True], tol_grad)):
                if gpu is None or (name == "grad" and not np.any(gpu)):  # projections: gradient not stored
                    continue
                u, v = gpu[k], ref[o]
                scale = np.abs(v).max()
                e2 = np.linalg.norm(u - v) / max(np.linalg.norm(v), 1e-30)
                ee = np.abs(u - v).max() / max(scale, 1e-30)
                assert e2 <= tol and ee <= tol, (name, s, b, l, e2, ee)


@pytest.mark.parametrize("aug,hw,B", [("none", 16, 4), ("per_sample", 16, 3)])
def test_cnn_bf16_layerwise_against_exact_oracle(aug, hw, B):
    """The tcgen05 conv path, layer by layer, for EVERY (sample, example), against the exact
    oracle in the parity regime (R26): stored activations within 1e-2, stored gradients within
    2e-2. A wrong tap, channel, bias, residual, mask or tile is O(1) and fails here first."""
    native = _native()
    model, S = dict(BF16_CNN, in_h=hw, in_w=hw), 2
    mu, rho, x, yc, _ = _inputs(model, B, regime="positive")
    a = O.AUG_PER_SAMPLE if aug == "per_sample" else O.AUG_NONE
    ctx = native.Context(model, precision="bf16", max_B_loc=B, max_S_loc=S, dataset_size=1e4, aug=aug)
    ctx.elbo_partial(_dev(mu), _dev(rho), _dev(x), _dev(yc), B, S, 0xBEEF, 5)
    torch.cuda.synchronize()
    _cnn_layerwise(ctx, model, mu, rho, x, yc, S, B, 0xBEEF, 5, a,
                   [(s, b) for s in range(S) for b in range(B)], 1e-2, 2e-2)


@pytest.mark.parametrize("aug,hw,B", [("none", 16, 4), ("per_sample", 16, 5)])
def test_cnn_bf16_end_to_end_vs_oracle(aug, hw, B):
    """Whole BF16 CNN step against the exact oracle at north_star's 2e-2 (parity regime R26):
    loss, grad_μ and grad_ρ of every tensor (elementwise and per tensor), and the data term
    alone (acc_μ, acc_ρ of bnn_elbo_partial: the ε-weighted conv wgrad sums, not hidden by
    the KL part of grad_ρ)."""
    model, S, D = dict(BF16_CNN, in_h=hw, in_w=hw), 2, 45000.0
    mu, rho, x, yc, _ = _inputs(model, B, regime="positive")
    a = O.AUG_PER_SAMPLE if aug == "per_sample" else O.AUG_NONE
    ctx, loss, gmu, grho = _run_gpu(model, "bf16", mu, rho, x, yc, None, S, 0xBEEF, 5, D, aug=aug)
    ref = O.elbo_step(model, mu, rho, x, yc, None, S, 0xBEEF, 5, D, aug=a)
    assert abs(loss - ref["loss"]) <= 2e-2 * abs(ref["loss"])
    _assert_close(ctx, gmu, ref["grad_mu"], 2e-2, "grad_mu")
    _assert_close(ctx, grho, ref["grad_rho"], 2e-2, "grad_rho")
    am, ar, al = _acc_parts(ctx, ctx.elbo_partial(_dev(mu), _dev(rho), _dev(x), _dev(yc), B, S, 0xBEEF, 5))
    ra = O.elbo_partial(model, mu, rho, x, yc, None, B, 0, S, 0, S, 0xBEEF, 5, aug=a)
    P = ctx.n_params
    _assert_close(ctx, am, ra[:P], 2e-2, "acc_mu")
    _assert_close(ctx, ar, ra[P:2 * P], 2e-2, "acc_rho")
    assert abs(al - ra[-1]) <= 2e-2 * abs(ra[-1])


def test_cnn_bf16_c3_resolution_all_gradients():
    """C3's resolution and batch (ResNet-18, 32×32×3, B = 128, per-sample augmentation) at
    S = 2, bench launch configuration: the data term of every gradient tensor (acc_μ, acc_ρ),
    the loss and the full grad_μ / grad_ρ against the exact oracle at 2e-2 (R26 regime;
    ≈ 1 TFLOP of fp64 oracle work, about a minute on the host cores)."""
    model = dict(kind="resnet18", in_h=32, in_w=32, in_c=3, n_classes=10, base_width=64, loss="ce")
    B, S, D = 128, 2, 45000.0
    mu, rho, x, yc, _ = _inputs(model, B, regime="positive")
    native = _native()
    ctx = native.Context(model, precision="bf16", max_B_loc=B, max_S_loc=8, dataset_size=D, aug="per_sample")
    mu_d, rho_d = _dev(mu), _dev(rho)
    acc = ctx.elbo_partial(mu_d, rho_d, _dev(x), _dev(yc), B, S, 0x5EED, 0)
    loss, gmu, grho = ctx.finalize(mu_d, rho_d, acc)
    torch.cuda.synchronize()
    ra = O.elbo_partial(model, mu, rho, x, yc, None, B, 0, S, 0, S, 0x5EED, 0, aug=O.AUG_PER_SAMPLE)
    ref = O.finalize(model, mu, rho, ra, D)
    P = ctx.n_params
    am, ar, al = _acc_parts(ctx, acc)
    _assert_close(ctx, am, ra[:P], 2e-2, "acc_mu")
    _assert_close(ctx, ar, ra[P:2 * P], 2e-2, "acc_rho")
    assert abs(al - ra[-1]) <= 2e-2 * abs(ra[-1])
    assert abs(float(loss) - ref["loss"]) <= 2e-2 * abs(ref["loss"])
    _assert_close(ctx, gmu.cpu().numpy(), ref["grad_mu"], 2e-2, "grad_mu")
    _assert_close(ctx, grho.cpu().numpy(), ref["grad_rho"], 2e-2, "grad_rho")


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_cnn_sample_chunking_equals_single_chunk(precision):
    """S = 4 in chunks of 2 (the C4 path: S_loc > chunk) = one chunk of 4, up to fp32
    summation order of the per-chunk accumulation."""
    native = _native()
    model, B, S = dict(BF16_CNN, in_h=8, in_w=8), 3, 4
    mu, rho, x, yc, _ = _inputs(model, B, "init")
    out = []
    for chunk in (0, 2):
        ctx = native.Context(model, precision=precision, max_B_loc=B, max_S_loc=S, sample_chunk=chunk,
                             dataset_size=1e4, aug="per_sample")
        out.append(ctx.elbo_step(_dev(mu), _dev(rho), _dev(x), _dev(yc), B, S, 21, 2))
        torch.cuda.synchronize()
    (l0, m0, r0), (l1, m1, r1) = out
    assert abs(l0 - l1) <= 1e-6 * abs(l0)
    assert _rel(m1.cpu().numpy(), m0.cpu().numpy()) < 1e-5
    assert _rel(r1.cpu().numpy(), r0.cpu().numpy()) < 1e-5


def test_cnn_bf16_full_size_c3_sampled_examples():
    """C3 at full size in the bench launch configuration (ResNet-18, 32×32×3, B = 128, S = 8,
    per-sample augmentation): the stored activations and gradients of sampled (sample, example)
    pairs — first, last and two in between — against the exact oracle, with the layer-wise
    bounds of test_cnn_bf16_layerwise_against_exact_oracle (parity regime R26)."""
    native = _native()
    model = dict(kind="resnet18", in_h=32, in_w=32, in_c=3, n_classes=10, base_width=64, loss="ce")
    B, S = 128, 8
    mu, rho, x, yc, _ = _inputs(model, B, regime="positive")
    ctx = native.Context(model, precision="bf16", max_B_loc=B, max_S_loc=S, dataset_size=45000.0,
                         aug="per_sample")
    ctx.elbo_partial(_dev(mu), _dev(rho), _dev(x), _dev(yc), B, S, 0x5EED, 0)
    torch.cuda.synchronize()
    _cnn_layerwise(ctx, model, mu, rho, x, yc, S, B, 0x5EED, 0, O.AUG_PER_SAMPLE,
                   [(0, 0), (3, 77), (5, 1), (S - 1, B - 1)], 1e-2, 2e-2)


def test_cnn_bf16_sample_sharded_virtual_ranks_equal_single_rank():
    """BF16 CNN: K = 2 sample groups × G = 2 data groups (C5's grid shape) summed through
    bnn_finalize equal the single rank within 1e-5 (north_star: sharded = single), with
    per-sample augmentation keyed by global (s, b)."""
    native = _native()
    model, B, S, D = dict(BF16_CNN, in_h=8, in_w=8), 4, 4, 100.0
    mu, rho, x, yc, _ = _inputs(model, B, "init")
    mu_d, rho_d = _dev(mu), _dev(rho)
    single = native.Context(model, precision="bf16", max_B_loc=B, max_S_loc=S, dataset_size=D, aug="per_sample")
    l1, g1, r1 = single.finalize(mu_d, rho_d, single.elbo_partial(mu_d, rho_d, _dev(x), _dev(yc), B, S, 9, 4))
    total = None
    for rank in range(4):
        ctx = native.Context(model, precision="bf16", mode="hybrid", K=2, G=2, rank=rank, world=4,
                             max_B_loc=B // 2, max_S_loc=S // 2, dataset_size=D, aug="per_sample")
        g = rank % 2
        acc = ctx.elbo_partial(mu_d, rho_d, _dev(x[2 * g:2 * g + 2]), _dev(yc[2 * g:2 * g + 2]), B, S, 9, 4)
        total = acc if total is None else total + acc
    l2, g2, r2 = single.finalize(mu_d, rho_d, total)
    torch.cuda.synchronize()
    assert abs(l1.item() - l2.item()) <= 1e-5 * abs(l1.item())
    assert _rel(g2.cpu().numpy(), g1.cpu().numpy()) < 1e-5
    assert _rel(r2.cpu().numpy(), r1.cpu().numpy()) < 1e-5


# ------------------------------------------------------------------ exact aggregation on the CNN (f1)
@pytest.mark.parametrize("aug", ["none", "per_sample"])
def test_cnn_fp32_mean_aggregation_matches_oracle(aug):
    """CE of the mean class probability on the ResNet-18-shaped net, FP32 path:
    loss and gradients ≤ 1e-4 against oracle.elbo_step(agg="mean")."""
    model, B, S, D = SMALL_CNN, 6, 3, 45000.0
    # init σ: at σ ≤ 0.69 this BatchNorm-free net saturates the softmax and the mean true-class
    # probability underflows (infinite loss, reading R21). Step key 7: with key 5 and
    # augmentation one stage-4 ReLU pre-activation of one example lies within fp32 rounding of
    # 0 and is decided differently by the fp32 kernels and the fp64 oracle (R23)
    mu, rho, x, yc, _ = _inputs(model, B, "init")
    a = O.AUG_PER_SAMPLE if aug == "per_sample" else O.AUG_NONE
    ref = O.elbo_step(model, mu, rho, x, yc, None, S, 0xBEEF, 7, D, aug=a, agg="mean")
    ctx, loss, gmu, grho = _run_gpu(dict(model, loss="ce_mean"), "fp32", mu, rho, x, yc, None, S, 0xBEEF, 7,
                                    D, aug=aug)
    assert abs(loss - ref["loss"]) <= 1e-4 * abs(ref["loss"])
    _assert_close(ctx, gmu, ref["grad_mu"], 1e-4, "grad_mu")
    _assert_close(ctx, grho, ref["grad_rho"], 1e-4, "grad_rho")


@pytest.mark.parametrize("chunk", [0, 1])
def test_cnn_bf16_mean_aggregation(chunk):
    """BF16 tcgen05 CNN with the mean-probability loss: loss and gradients within 2e-2 of the
    exact oracle (parity regime R26), and two virtual sample groups (statistics summed,
    bnn_elbo_partial_mean) equal to the single rank within 1e-5; chunk = 1 exercises the
    recomputed forward."""
    native = _native()
    model, B, S, D = dict(BF16_CNN, in_h=16, in_w=16), 5, 4, 45000.0
    mu, rho, x, yc, _ = _inputs(model, B, regime="positive")
    mm = dict(model, loss="ce_mean")
    ref = O.elbo_step(model, mu, rho, x, yc, None, S, 0xBEEF, 5, D, aug=O.AUG_PER_SAMPLE, agg="mean")
    ctx, loss, gmu, grho = _run_gpu(mm, "bf16", mu, rho, x, yc, None, S, 0xBEEF, 5, D, aug="per_sample",
                                    sample_chunk=chunk)
    assert abs(loss - ref["loss"]) <= 2e-2 * abs(ref["loss"])
    _assert_close(ctx, gmu, ref["grad_mu"], 2e-2, "grad_mu")
    _assert_close(ctx, grho, ref["grad_rho"], 2e-2, "grad_rho")
    mu_d, rho_d, x_d, y_d = _dev(mu), _dev(rho), _dev(x), _dev(yc)
    ctxs = [native.Context(mm, precision="bf16", mode="sample", K=2, G=1, rank=r, world=2, max_B_loc=B,
                           max_S_loc=S // 2, dataset_size=D, aug="per_sample", sample_chunk=chunk) for r in range(2)]
    st = [c.mean_stats(mu_d, rho_d, x_d, y_d, B, S, 0xBEEF, 5, 1) for c in ctxs]
    gst = st[0] + st[1]
    total = None
    for c in ctxs:
        acc = c.elbo_partial_mean(mu_d, rho_d, x_d, y_d, B, S, 0xBEEF, 5, gst)
        total = acc if total is None else total + acc
    l2, g2, r2 = ctx.finalize(mu_d, rho_d, total)
    torch.cuda.synchronize()
    assert _rel(g2.cpu().numpy(), gmu) < 1e-5
    assert _rel(r2.cpu().numpy(), grho) < 1e-5
    assert abs(float(l2) - loss) <= 1e-5 * abs(loss)


@pytest.mark.parametrize("loss", ["ce_mean", "mse_mean"])
def test_mean_statistic_matches_oracle(loss):
    """bnn_mean_stats (the statistic exchanged between forward and backward) against the
    oracle's orc_mean_stats for rank 3 of a 2×2 grid: samples [3, 6), global examples 40..79,
    FP32 path: ≤ 1e-5 relative."""
    native = _native()
    base = RAGGED if loss == "ce_mean" else RAGGED_MSE
    model = dict(base, loss=loss)
    B, S = 80, 6
    mu, rho, x, yc, yr = _inputs(base, B, "init")
    y = yc if loss == "ce_mean" else yr
    ctx = native.Context(model, precision="fp32", mode="hybrid", K=2, G=2, rank=1 * 2 + 1, world=4,
                         max_B_loc=40, max_S_loc=3, dataset_size=100.0)
    xs, ys = x[40:80], y[40:80]
    width = 1 if loss == "ce_mean" else base["widths"][-1]
    g = ctx.mean_stats(_dev(mu), _dev(rho), _dev(xs), _dev(ys), B, S, 11, 3, width).cpu().numpy()
    ref = O.mean_stats(_base(model), mu, rho, xs, None if yc is None else yc[40:80], 40, 3, 6, 11, 3)
    assert _rel(g, ref.reshape(-1)) <= 1e-5


# ------------------------------------------------------------------ Gaussian NLL of the predictive (f1)
@pytest.mark.parametrize("precision,tol", [("fp32", 1e-4)])
@pytest.mark.parametrize("rho_mode", ["wide", "init"])
def test_gnll_matches_oracle(precision, tol, rho_mode):
    """BNN_LOSS_GNLL_MEAN (the two-parameter exchange of P:281) through
    bnn_elbo_step against oracle.elbo_step(loss="gnll", agg="mean"). FP32 only: in BF16 mode
    the rounded predictions perturb the sample variance the seeds divide by (measured 5-7 %
    gradient error), so the library rejects that combination (test below)."""
    base = dict(RAGGED_MSE, loss="gnll")
    B, S, D = 40, 6, 1000.0
    mu, rho, x, _, yr = _inputs(base, B, rho_mode)
    ctx, loss, gmu, grho = _run_gpu(dict(base, loss="gnll_mean"), precision, mu, rho, x, None, yr, S, 0xC0FFEE,
                                    3, D)
    ref = O.elbo_step(base, mu, rho, x, None, yr, S, 0xC0FFEE, 3, D, agg="mean")
    assert abs(loss - ref["loss"]) <= tol * abs(ref["loss"])
    _assert_close(ctx, gmu, ref["grad_mu"], tol, "grad_mu")
    _assert_close(ctx, grho, ref["grad_rho"], tol, "grad_rho")


@pytest.mark.parametrize("mode,K,G,chunk", [("sample", 3, 1, 0), ("hybrid", 2, 2, 1)])
def test_gnll_virtual_ranks_equal_single_rank(mode, K, G, chunk):
    """Per-rank Welford (mean, M2) merged by bnn_mean_merge (Chan's update, rank order), then
    bnn_elbo_partial_mean; Σ acc → finalize equals the single rank within 1e-5."""
    native = _native()
    base = dict(RAGGED_MSE, loss="gnll_mean")
    B, S, D = 48, 12, 321.0
    mu, rho, x, _, yr = _inputs(dict(base, loss="mse"), B, "wide")
    mu_d, rho_d = _dev(mu), _dev(rho)
    single = native.Context(base, precision="fp32", max_B_loc=B, max_S_loc=S, dataset_size=D)
    l1, g1, r1 = single.elbo_step(mu_d, rho_d, _dev(x), _dev(yr), B, S, 77, 9)
    world, O_ = K * G, base["widths"][-1]
    ctxs, shards = [], []
    for rank in range(world):
        ctx = native.Context(base, precision="fp32", mode=mode, K=K, G=G, rank=rank, world=world,
                             max_B_loc=B // G, max_S_loc=S // K, dataset_size=D, sample_chunk=chunk)
        g = rank % G
        sl = slice(g * (B // G), (g + 1) * (B // G))
        ctxs.append(ctx)
        shards.append((_dev(x[sl]), _dev(yr[sl])))
    stats = [c.mean_stats(mu_d, rho_d, xs, ys, B, S, 77, 9, 2 * O_) for c, (xs, ys) in zip(ctxs, shards)]
    total = None
    for rank, (c, (xs, ys)) in enumerate(zip(ctxs, shards)):
        g = rank % G
        gst = c.mean_merge([stats[r] for r in range(g, world, G)], B // G, S)
        acc = c.elbo_partial_mean(mu_d, rho_d, xs, ys, B, S, 77, 9, gst)
        total = acc if total is None else total + acc
    l2, g2, r2 = single.finalize(mu_d, rho_d, total)
    torch.cuda.synchronize()
    assert _rel(g2.cpu().numpy(), g1.cpu().numpy()) < 1e-5
    assert _rel(r2.cpu().numpy(), r1.cpu().numpy()) < 1e-5
    assert abs(float(l2) - float(l1)) <= 1e-5 * abs(float(l1))


def test_gnll_rejects_bf16():
    native = _native()
    with pytest.raises(native.BnnError, match="FP32"):
        native.Context(dict(RAGGED_MSE, loss="gnll_mean"), precision="bf16", max_B_loc=8, max_S_loc=2,
                       dataset_size=1.0)


def test_nccl_communicator_world1_gnll_fp32():
    """The GNLL statistic's allgather + Chan merge on one GPU equals the no-communicator step."""
    native = _native()
    model = dict(RAGGED_MSE, loss="gnll_mean")
    B, S = 48, 4
    mu, rho, x, _, yr = _inputs(dict(RAGGED_MSE), B, "wide")
    out = []
    for uid in (None, native.get_unique_id()):
        ctx = native.Context(model, precision="fp32", max_B_loc=B, max_S_loc=S, dataset_size=500.0, uid=uid)
        l, g, r = ctx.elbo_step(_dev(mu), _dev(rho), _dev(x), _dev(yr), B, S, 3, 4)
        torch.cuda.synchronize()
        out.append((l, g.cpu(), r.cpu()))
        ctx.close()
    assert out[0][0] == out[1][0]
    assert torch.equal(out[0][1], out[1][1]) and torch.equal(out[0][2], out[1][2])


# ------------------------------------------------------------------ MC dropout
MCD_MLP = dict(kind="mlp", widths=[96, 128, 128, 24], loss="mse", method="mcd", dropout_p=0.1)


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-4), ("bf16", 2e-2)])
@pytest.mark.parametrize("loss", ["mse", "mse_mean"])
def test_mcd_step_matches_oracle(precision, tol, loss):
    """MC-dropout step (weights μ, inverted dropout on the hidden activations, keyed masks) of
    the paper's use-case-2 MLP shape 96-128-128-24 (per-sample MSE, and the MSE of the averaged
    predictions the paper trains on) against the exact oracle: FP32 1e-4 (Kaiming
    regime), BF16 2e-2 (parity regime R26), elementwise and per tensor; BF16 in the Kaiming
    regime against the emulating oracle as well."""
    base = dict(MCD_MLP)
    B, S, D = 64, 4, 1000.0
    regime = "positive" if precision == "bf16" else "kaiming"
    mu, rho, x, _, yr = _inputs(base, B, "init", regime=regime)
    ctx, l, gmu, grho = _run_gpu(dict(base, loss=loss), precision, mu, rho, x, None, yr, S, 0xD0, 2, D)
    agg = "mean" if loss == "mse_mean" else "sample"
    ref = O.elbo_step(base, mu, rho, x, None, yr, S, 0xD0, 2, D, agg=agg)
    assert abs(l - ref["loss"]) <= tol * abs(ref["loss"])
    assert not np.any(grho)
    _assert_close(ctx, gmu, ref["grad_mu"], tol, "grad_mu")
    if precision == "bf16" and agg == "sample":
        mu, rho, x, _, yr = _inputs(base, B, "init")
        ctx, l, gmu, grho = _run_gpu(dict(base, loss=loss), precision, mu, rho, x, None, yr, S, 0xD0, 2, D)
        emu = O.elbo_step(base, mu, rho, x, None, yr, S, 0xD0, 2, D, emu=True)
        assert max(_per_tensor_rel(ctx, gmu, emu["grad_mu"])) <= 2e-3
        _assert_close(ctx, gmu, emu["grad_mu"], 1e-2, "grad_mu emu")


def test_mcd_virtual_ranks_equal_single_rank():
    """Sample × data sharding of the MC-dropout step (masks keyed by global sample and global
    example): Σ of the 2×2 virtual ranks' partials = single rank within 1e-5."""
    native = _native()
    B, S, D = 64, 8, 500.0
    mu, rho, x, _, yr = _inputs(MCD_MLP, B, "init")
    mu_d, rho_d = _dev(mu), _dev(rho)
    single = native.Context(MCD_MLP, precision="bf16", max_B_loc=B, max_S_loc=S, dataset_size=D)
    acc1 = single.elbo_partial(mu_d, rho_d, _dev(x), _dev(yr), B, S, 5, 6)
    l1, g1, _ = single.finalize(mu_d, rho_d, acc1)
    total = None
    for rank in range(4):
        ctx = native.Context(MCD_MLP, precision="bf16", mode="hybrid", K=2, G=2, rank=rank, world=4,
                             max_B_loc=B // 2, max_S_loc=S // 2, dataset_size=D)
        g = rank % 2
        acc = ctx.elbo_partial(mu_d, rho_d, _dev(x[g * 32:(g + 1) * 32]), _dev(yr[g * 32:(g + 1) * 32]), B, S, 5, 6)
        total = acc if total is None else total + acc
    l2, g2, _ = single.finalize(mu_d, rho_d, total)
    torch.cuda.synchronize()
    assert _rel(g2.cpu().numpy(), g1.cpu().numpy()) < 1e-5
    assert abs(float(l2) - float(l1)) <= 1e-5 * abs(float(l1))


def test_mcd_predict_matches_oracle():
    """MC-dropout predictive mean / variance over S mask draws, FP32."""
    native = _native()
    B, S = 32, 8
    mu, rho, x, _, _ = _inputs(MCD_MLP, B, "init")
    ctx = native.Context(MCD_MLP, precision="fp32", max_B_loc=B, max_S_loc=S, dataset_size=1.0)
    mean, var = ctx.predict(_dev(mu), _dev(rho), _dev(x), S, 3, 0)
    rm, rv = O.predict(MCD_MLP, mu, rho, x, S, 3, 0)
    assert _rel(mean.cpu().numpy(), rm) < 1e-4
    assert _rel(var.cpu().numpy(), rv) < 1e-3


# ------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("precision,tol", [("fp32", 1e-4), ("bf16", 2e-2)])
@pytest.mark.parametrize("model,B,S", [
    (dict(kind="mlp", widths=[33, 17, 5], loss="ce"), 1, 1),          # one example, one sample
    (dict(kind="mlp", widths=[130, 260, 10], loss="ce"), 300, 2),      # B > 256: two batch tiles, ragged tail
    (dict(kind="mlp", widths=[1030, 129, 3], loss="mse"), 19, 3),      # K and N off every tile size
])
def test_edge_shapes_match_oracle(model, B, S, precision, tol):
    mu, rho, x, yc, yr = _inputs(model, B, "init", regime="positive" if precision == "bf16" else "kaiming")
    ctx, loss, gmu, grho = _run_gpu(model, precision, mu, rho, x, yc, yr, S, 0xE0, 1, 100.0)
    ref = O.elbo_step(model, mu, rho, x, yc, yr, S, 0xE0, 1, 100.0)
    assert abs(loss - ref["loss"]) <= tol * abs(ref["loss"])
    _assert_close(ctx, gmu, ref["grad_mu"], tol, "grad_mu")
    _assert_close(ctx, grho, ref["grad_rho"], tol, "grad_rho")


def test_predict_single_sample_has_zero_variance():
    """S = 1: the predictive variance is exactly 0 (population variance of one value)."""
    native = _native()
    mu, rho, x, _, _ = _inputs(RAGGED, 9, "wide")
    ctx = native.Context(RAGGED, precision="bf16", max_B_loc=9, max_S_loc=1, dataset_size=1.0)
    mean, var = ctx.predict(_dev(mu), _dev(rho), _dev(x), 1, 3, 0)
    torch.cuda.synchronize()
    assert torch.count_nonzero(var).item() == 0
    assert torch.allclose(mean.sum(-1), torch.ones(9, device=mean.device), atol=1e-5)


def test_invariant_violations_fail_loudly_on_device():
    """Shape invariants of the step and a non-finite loss (BNN_ERR_NUMERIC)."""
    native = _native()
    mu, rho, x, yc, _ = _inputs(RAGGED, 8, "init")
    ctx = native.Context(RAGGED, precision="bf16", max_B_loc=8, max_S_loc=2, dataset_size=1.0)
    with pytest.raises(native.BnnError, match="max_S_loc"):
        ctx.elbo_step(_dev(mu), _dev(rho), _dev(x), _dev(yc), 8, 3, 1, 0)
    with pytest.raises(native.BnnError, match="B_loc"):
        big = np.concatenate([x, x])
        ctx.elbo_step(_dev(mu), _dev(rho), _dev(big), _dev(np.concatenate([yc, yc])), 16, 2, 1, 0)
    sh = native.Context(RAGGED, precision="bf16", mode="sample", K=2, rank=0, world=2, max_B_loc=8,
                        max_S_loc=2, dataset_size=1.0)
    with pytest.raises(native.BnnError, match="S mod K"):
        sh.elbo_partial(_dev(mu), _dev(rho), _dev(x), _dev(yc), 8, 3, 1, 0)
    bad = mu.copy()
    bad[0] = np.nan
    with pytest.raises(native.BnnError, match="non-finite"):
        ctx.elbo_step(_dev(bad), _dev(rho), _dev(x), _dev(yc), 8, 2, 1, 0)


def test_bf16_mlp_partial_batch_then_full_batch_on_one_context():
    """a step with B_loc < max_B_loc (the last partial batch of an epoch) on a
    BF16 context, S > 1, then a full batch and a partial one again on the same context: every
    step against the exact oracle (parity regime R26). The descriptors are re-encoded per
    B_loc, so sample s ≥ 1 reads its own rows and no stale row enters the wgrad sums."""
    native = _native()
    model, Bmax, S, D = RAGGED, 96, 3, 500.0
    mu, rho, x, yc, _ = _inputs(model, Bmax, regime="positive")
    ctx = native.Context(model, precision="bf16", max_B_loc=Bmax, max_S_loc=S, dataset_size=D)
    for B in (37, Bmax, 70):
        loss, gmu, grho = ctx.elbo_step(_dev(mu), _dev(rho), _dev(x[:B]), _dev(yc[:B]), B, S, 0xB10C, B)
        torch.cuda.synchronize()
        ref = O.elbo_step(model, mu, rho, x[:B], yc[:B], None, S, 0xB10C, B, D)
        assert abs(loss - ref["loss"]) <= 2e-2 * abs(ref["loss"]), B
        _assert_close(ctx, gmu.cpu().numpy(), ref["grad_mu"], 2e-2, ("grad_mu", B))
        _assert_close(ctx, grho.cpu().numpy(), ref["grad_rho"], 2e-2, ("grad_rho", B))
    mean, var = ctx.predict(_dev(mu), _dev(rho), _dev(x[:21]), S, 3, 0)
    rm, rv = O.predict(model, mu, rho, x[:21], S, 3, 0)
    assert np.abs(mean.cpu().numpy() - rm).max() <= 2e-2 * np.abs(rm).max()


def test_bf16_resnet_partial_batch_is_rejected():
    native = _native()
    model = dict(BF16_CNN, in_h=16, in_w=16)
    mu, rho, x, yc, _ = _inputs(model, 4, regime="positive")
    ctx = native.Context(model, precision="bf16", max_B_loc=4, max_S_loc=2, dataset_size=1.0)
    with pytest.raises(native.BnnError, match="B_loc == max_B_loc"):
        ctx.elbo_step(_dev(mu), _dev(rho), _dev(x[:3]), _dev(yc[:3]), 3, 2, 1, 0)


# ------------------------------------------------------------------ gradient exchange (a7)
@pytest.mark.parametrize("chunk", [0, 2])
def test_cnn_bucketed_exchange_world1_equals_no_communicator(chunk, monkeypatch):
    """The layer-bucketed allreduce on the comm stream (comm.cu): with a 0.25 MB bucket the
    ResNet exchange is split into many NCCL groups issued during the backward (last sample chunk
    only when S_loc > chunk); on one GPU every allreduce is the identity, so loss and gradients
    equal the no-communicator step bit for bit, and the stream ordering (comm stream waits for
    each bucket's writers, the finalize waits for the comm stream) is exercised."""
    native = _native()
    monkeypatch.setenv("BNN_AR_BUCKET_MB", "0.25")
    model = dict(BF16_CNN, in_h=16, in_w=16)
    B, S = 3, 4
    mu, rho, x, yc, _ = _inputs(model, B, regime="positive")
    out = []
    for uid in (None, native.get_unique_id()):
        ctx = native.Context(model, precision="bf16", max_B_loc=B, max_S_loc=S, dataset_size=500.0, uid=uid,
                             aug="per_sample", sample_chunk=chunk)
        for step in (4, 5):  # two steps: the second one's acc zeroing must follow the first exchange
            l, g, r = ctx.elbo_step(_dev(mu), _dev(rho), _dev(x), _dev(yc), B, S, 3, step)
        torch.cuda.synchronize()
        out.append((l, g.cpu(), r.cpu(), ctx.comm_buckets()))
        ctx.close()
    assert out[0][3] == 0 and out[1][3] >= 6, out[1][3]
    assert out[0][0] == out[1][0]
    assert torch.equal(out[0][1], out[1][1]) and torch.equal(out[0][2], out[1][2])


def test_comm_timeout_returns_err_comm():
    """A communicator whose peer never joins (world 2, only rank 0 calls bnn_init) fails with
    BNN_ERR_COMM after comm_timeout_ms instead of hanging. Run in a child
    process so a hang cannot take the test session down."""
    import subprocess
    import sys
    code = (
        "import sys, time; sys.path.insert(0, '.')\n"
        "from paper_2604_04736_b200 import native\n"
        "t0 = time.time()\n"
        "try:\n"
        "    native.Context(dict(kind='mlp', widths=[8, 16, 1], loss='mse'), precision='fp32', mode='sample',\n"
        "                   K=2, rank=0, world=2, uid=native.get_unique_id(), max_B_loc=4, max_S_loc=2,\n"
        "                   dataset_size=1.0, comm_timeout_ms=3000)\n"
        "    print('NO-ERROR')\n"
        "except native.BnnError as e:\n"
        "    print('ERR', time.time() - t0, e)\n")
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=120)
    line = [l for l in r.stdout.splitlines() if l.startswith("ERR ")]  # NCCL may print its banner
    assert line and "timeout" in line[0] and "BNN_ERR" not in line[0], (r.stdout, r.stderr[-2000:])
    assert "libbnn error 3" in line[0], line[0]  # BNN_ERR_COMM
    dt = float(line[0].split()[1])
    assert 2.5 <= dt <= 60.0, dt


# ------------------------------------------------------------------ Bayesian ViT
VIT_TINY = dict(kind="vit", in_h=8, in_w=8, in_c=3, patch=4, dim=32, heads=2, depth=2, mlp=64, n_classes=3,
                loss="ce")
VIT = MODELS["vit_cifar"]


@pytest.mark.parametrize("aug,rho_mode", [("none", "wide"), ("per_sample", "wide"), ("per_sample", "init")])
def test_vit_fp32_matches_oracle(aug, rho_mode):
    """The ViT step (FP32: sampled projections on the MLP's kernels, LayerNorm / attention /
    GELU kernels) against the exact ViT oracle: loss, grad_μ, grad_ρ and the data term ≤ 1e-4."""
    native = _native()
    model, B, S, D = VIT_TINY, 5, 3, 300.0
    mu, rho = synth.init_params(model, seed=2, rho_mode=rho_mode)
    x, yc, _ = synth.make_batch(model, B, seed=1)
    a = O.AUG_PER_SAMPLE if aug == "per_sample" else O.AUG_NONE
    ctx = native.Context(model, precision="fp32", max_B_loc=B, max_S_loc=S, dataset_size=D, aug=aug)
    loss, gmu, grho = ctx.elbo_step(_dev(mu), _dev(rho), _dev(x), _dev(yc), B, S, 0x7177, 2)
    torch.cuda.synchronize()
    ref = O.vit_elbo_step(model, mu, rho, x, yc, S, 0x7177, 2, D, aug=a)
    assert abs(loss - ref["loss"]) <= 1e-4 * abs(ref["loss"])
    _assert_close(ctx, gmu.cpu().numpy(), ref["grad_mu"], 1e-4, "grad_mu")
    _assert_close(ctx, grho.cpu().numpy(), ref["grad_rho"], 1e-4, "grad_rho")
    am, ar, al = _acc_parts(ctx, ctx.elbo_partial(_dev(mu), _dev(rho), _dev(x), _dev(yc), B, S, 0x7177, 2))
    ra = O.vit_elbo_partial(model, mu, rho, x, yc, B, 0, S, 0, S, 0x7177, 2, a)
    P = ctx.n_params
    _assert_close(ctx, am, ra[:P], 1e-4, "acc_mu")
    _assert_close(ctx, ar, ra[P:2 * P], 1e-4, "acc_rho")


def test_vit_fp32_paper_size_matches_oracle():
    """The paper's ViT (32×32 CIFAR-shaped, 4×4 patches, width 192, 3 heads, 6 layers, MLP 768)
    with per-sample augmentation, B = 3, S = 2: every tensor ≤ 1e-4."""
    native = _native()
    B, S, D = 3, 2, 45000.0
    mu, rho = synth.init_params(VIT, seed=2)
    x, yc, _ = synth.make_batch(VIT, B, seed=1)
    ctx = native.Context(VIT, precision="fp32", max_B_loc=B, max_S_loc=S, dataset_size=D, aug="per_sample")
    mu_d, rho_d = _dev(mu), _dev(rho)
    acc = ctx.elbo_partial(mu_d, rho_d, _dev(x), _dev(yc), B, S, 0x5EED, 0)
    loss, gmu, grho = ctx.finalize(mu_d, rho_d, acc)
    torch.cuda.synchronize()
    ra = O.vit_elbo_partial(VIT, mu, rho, x, yc, B, 0, S, 0, S, 0x5EED, 0, O.AUG_PER_SAMPLE)
    ref = O.vit_finalize(mu, rho, ra, D)
    P = ctx.n_params
    am, ar, al = _acc_parts(ctx, acc)
    _assert_close(ctx, am, ra[:P], 1e-4, "acc_mu")
    _assert_close(ctx, ar, ra[P:2 * P], 1e-4, "acc_rho")
    assert abs(al - ra[-1]) <= 1e-4 * abs(ra[-1])
    _assert_close(ctx, gmu.cpu().numpy(), ref["grad_mu"], 1e-4, "grad_mu")
    _assert_close(ctx, grho.cpu().numpy(), ref["grad_rho"], 1e-4, "grad_rho")


@pytest.mark.parametrize("mode,K,G,chunk", [("hybrid", 2, 2, 0), ("sample", 1, 1, 1)])
def test_vit_virtual_ranks_and_chunks_equal_single(mode, K, G, chunk):
    """ViT: a 2×2 sample × data grid of virtual ranks (augmentation keyed by global (s, b)), and
    sample chunks of 1, equal the single-rank single-chunk step within 1e-5."""
    native = _native()
    model, B, S, D = VIT_TINY, 4, 4, 100.0
    mu, rho = synth.init_params(model, seed=3, rho_mode="wide")
    x, yc, _ = synth.make_batch(model, B, seed=4)
    mu_d, rho_d = _dev(mu), _dev(rho)
    single = native.Context(model, precision="fp32", max_B_loc=B, max_S_loc=S, dataset_size=D, aug="per_sample")
    l1, g1, r1 = single.finalize(mu_d, rho_d, single.elbo_partial(mu_d, rho_d, _dev(x), _dev(yc), B, S, 5, 1))
    world = K * G
    total = None
    for rank in range(world):
        ctx = native.Context(model, precision="fp32", mode=mode, K=K, G=G, rank=rank, world=world,
                             max_B_loc=B // G, max_S_loc=S // K, dataset_size=D, aug="per_sample", sample_chunk=chunk)
        g = rank % G
        sl = slice(g * (B // G), (g + 1) * (B // G))
        acc = ctx.elbo_partial(mu_d, rho_d, _dev(x[sl]), _dev(yc[sl]), B, S, 5, 1)
        total = acc if total is None else total + acc
    l2, g2, r2 = single.finalize(mu_d, rho_d, total)
    torch.cuda.synchronize()
    assert abs(float(l2) - float(l1)) <= 1e-5 * abs(float(l1))
    assert _rel(g2.cpu().numpy(), g1.cpu().numpy()) < 1e-5
    assert _rel(r2.cpu().numpy(), r1.cpu().numpy()) < 1e-5


@pytest.mark.parametrize("model,B,S,aug", [(VIT_TINY, 6, 3, "per_sample"), (VIT, 3, 2, "per_sample"),
                                           (VIT, 2, 2, "none")])
def test_vit_bf16_matches_exact_oracle(model, B, S, aug):
    """BF16 ViT (projections on tcgen05 with W_s formed on chip; LayerNorm, attention, GELU and
    the residual stream in fp32) against the exact ViT oracle. Reading R27: this model is at
    the conditioning limit of BF16 — the BF16 mode's own sampled-weight definition alone
    (R14, oracle-only, tests/test_conditioning.py::test_vit_bf16_weight_rounding_spread) moves
    the exact step by 1.9–2.4 % per tensor and up to 3.9 % elementwise — so the bound is
    2.5e-2 per tensor and 5e-2 elementwise (the loss and L_data at 2e-2); the FP32 mode holds
    1e-4 (test_vit_fp32_matches_oracle)."""
    native = _native()
    D = 45000.0
    mu, rho = synth.init_params(model, seed=2)
    x, yc, _ = synth.make_batch(model, B, seed=1)
    a = O.AUG_PER_SAMPLE if aug == "per_sample" else O.AUG_NONE
    ctx = native.Context(model, precision="bf16", max_B_loc=B, max_S_loc=S, dataset_size=D, aug=aug)
    mu_d, rho_d = _dev(mu), _dev(rho)
    acc = ctx.elbo_partial(mu_d, rho_d, _dev(x), _dev(yc), B, S, 0x5EED, 3)
    loss, gmu, grho = ctx.finalize(mu_d, rho_d, acc)
    torch.cuda.synchronize()
    ra = O.vit_elbo_partial(model, mu, rho, x, yc, B, 0, S, 0, S, 0x5EED, 3, a)
    ref = O.vit_finalize(mu, rho, ra, D)
    P = ctx.n_params
    am, ar, al = _acc_parts(ctx, acc)

    def close(g, r, what):
        for t in ctx.tensors:
            sl = slice(t["offset"], t["offset"] + t["rows"] * t["cols"])
            d = np.abs(np.asarray(g[sl], np.float64) - r[sl])
            l2, el = np.linalg.norm(d) / np.linalg.norm(r[sl]), d.max() / np.abs(r[sl]).max()
            assert l2 <= 2.5e-2 and el <= 5e-2, (what, t["t"], l2, el)

    close(am, ra[:P], "acc_mu")
    close(ar, ra[P:2 * P], "acc_rho")
    assert abs(al - ra[-1]) <= 2e-2 * abs(ra[-1])
    assert abs(float(loss) - ref["loss"]) <= 2e-2 * abs(ref["loss"])
    close(gmu.cpu().numpy(), ref["grad_mu"], "grad_mu")
    close(grho.cpu().numpy(), ref["grad_rho"], "grad_rho")


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_out_of_range_label_is_a_numeric_error(precision):
    """A class label outside [0, n_classes) (round-1 ADVICE): no out-of-bounds read, the loss is
    NaN and the step returns BNN_ERR_NUMERIC."""
    native = _native()
    mu, rho, x, yc, _ = _inputs(RAGGED, 8, "init")
    bad = yc.copy()
    bad[3] = 10
    ctx = native.Context(RAGGED, precision=precision, max_B_loc=8, max_S_loc=2, dataset_size=1.0)
    with pytest.raises(native.BnnError, match="non-finite"):
        ctx.elbo_step(_dev(mu), _dev(rho), _dev(x), _dev(bad), 8, 2, 1, 0)


@pytest.mark.parametrize("hw,B", [(16, 3), (32, 2)])
def test_cnn_bf16_conv64_equals_conv3_halo(hw, B, monkeypatch):
    """The stage-1 (64 → 64) layers on the W-stationary tap-paired kernel (kernels_conv64.cu)
    against the same step with those layers on conv3's HALO tile (BNN_CONV64=0): every stored
    activation and gradient of every layer, and acc_μ / acc_ρ. The two differ only in fp32
    summation order before the bf16 rounding of each stored value (a rounding tie can flip one
    bf16 ulp, 2^-8 relative), so the bound is 1e-2 elementwise of each layer's max."""
    native = _native()
    model, S = dict(BF16_CNN, in_h=hw, in_w=hw), 2
    mu, rho, x, yc, _ = _inputs(model, B, regime="positive")
    res = []
    for flag in ("0", "1"):
        monkeypatch.setenv("BNN_CONV64", flag)
        ctx = native.Context(model, precision="bf16", max_B_loc=B, max_S_loc=S, dataset_size=1e4, aug="per_sample")
        acc = ctx.elbo_partial(_dev(mu), _dev(rho), _dev(x), _dev(yc), B, S, 0xBEEF, 5).cpu().numpy()
        torch.cuda.synchronize()
        n_layers = len(ctx.tensors) // 2
        lay = [(ctx.layer_output(l, 0).cpu().numpy(),
                ctx.layer_output(l, 1).cpu().numpy() if l < n_layers - 1 else None) for l in range(n_layers)]
        res.append((acc, lay))
    (a0, l0), (a1, l1) = res
    for l, ((o0, g0), (o1, g1)) in enumerate(zip(l0, l1)):
        assert np.abs(o1 - o0).max() <= 1e-2 * max(np.abs(o0).max(), 1e-30), ("out", l)
        if g0 is not None:
            assert np.abs(g1 - g0).max() <= 1e-2 * max(np.abs(g0).max(), 1e-30), ("grad", l)
    assert np.abs(a1 - a0).max() <= 1e-2 * np.abs(a0).max()


@pytest.mark.parametrize("hw,B,S", [(16, 3, 2), (32, 2, 3)])
def test_cnn_bf16_conv64_wgrad_equals_conv2_wgrad(hw, B, S, monkeypatch):
    """The stage-1 weight gradients on the row-packed kernel (conv64_wgrad_kernel: MN-major views of
    two halo windows, 2 MMAs of N = 192 per 16 pixels) against the generic conv2 wgrad
    (BNN_CONV64W=0) on the same step: acc_μ and acc_ρ of every tensor. Both accumulate the same
    bf16 products in fp32, in a different split / pixel order, so they agree to fp32 summation
    error (1e-4 of each tensor's max; a wrong tap, channel or pixel is O(1))."""
    native = _native()
    model = dict(BF16_CNN, in_h=hw, in_w=hw)
    mu, rho, x, yc, _ = _inputs(model, B, regime="positive")
    accs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("BNN_CONV64W", flag)
        ctx = native.Context(model, precision="bf16", max_B_loc=B, max_S_loc=S, dataset_size=1e4, aug="per_sample")
        accs.append(_acc_parts(ctx, ctx.elbo_partial(_dev(mu), _dev(rho), _dev(x), _dev(yc), B, S, 0xBEEF, 5)))
        torch.cuda.synchronize()
    (m0, r0, l0), (m1, r1, l1) = accs
    for t in ctx.tensors:
        sl = slice(t["offset"], t["offset"] + t["rows"] * t["cols"])
        for name, u, ref in (("acc_mu", m1[sl], m0[sl]), ("acc_rho", r1[sl], r0[sl])):
            assert np.abs(u - ref).max() <= 1e-4 * max(np.abs(ref).max(), 1e-30), (t["t"], name)
    assert l1 == l0


@pytest.mark.parametrize("hw,B,S,kp128", [(32, 2, 2, "0"), (16, 3, 3, "0"), (8, 5, 2, "0"), (32, 1, 8, "0"),
                                          (32, 2, 2, "1"), (16, 3, 3, "1")])
def test_cnn_bf16_stride2_wgrad_tma_equals_gather(hw, B, S, kp128, monkeypatch):
    """Weight gradients of the stride-2 convs (3×3 and the 1×1 shortcuts) with the X window loaded
    by TMA with element stride 2 in W and H against the cp.async gather of the same operand
    (BNN_WGRAD_S2_TMA=0): the same bf16 operands in the same shared-memory layout, summed in the
    same order, so acc_μ and acc_ρ of every tensor agree to 1e-6 of the tensor's max (a wrong
    tap, row parity or image is O(1)); 8×8 inputs put several images in one box, B = 5 leaves a
    ragged last k-step. kp128 = "1": the default 128-pixel k-steps of the TMA path against the
    gather's 64 (other pixel splits: equal to fp32 summation error, 1e-4 of the tensor's max)."""
    native = _native()
    model = dict(BF16_CNN, in_h=hw, in_w=hw)
    mu, rho, x, yc, _ = _inputs(model, B, regime="positive")
    accs = []
    monkeypatch.setenv("BNN_WGRAD_S2_KP128", kp128)
    tol = 1e-6 if kp128 == "0" else 1e-4
    for flag in ("0", "1"):
        monkeypatch.setenv("BNN_WGRAD_S2_TMA", flag)
        ctx = native.Context(model, precision="bf16", max_B_loc=B, max_S_loc=S, dataset_size=1e4, aug="per_sample")
        accs.append(_acc_parts(ctx, ctx.elbo_partial(_dev(mu), _dev(rho), _dev(x), _dev(yc), B, S, 0xBEEF, 5)))
        torch.cuda.synchronize()
    (m0, r0, l0), (m1, r1, l1) = accs
    for t in ctx.tensors:
        sl = slice(t["offset"], t["offset"] + t["rows"] * t["cols"])
        for name, u, ref in (("acc_mu", m1[sl], m0[sl]), ("acc_rho", r1[sl], r0[sl])):
            assert np.abs(u - ref).max() <= tol * max(np.abs(ref).max(), 1e-30), (t["t"], name)
    assert l1 == l0


@pytest.mark.parametrize("hw,B,S,chunk,cl", [(16, 3, 2, 0, None), (32, 2, 3, 0, None), (16, 2, 8, 0, None),
                                             (16, 2, 8, 0, "8"), (16, 2, 8, 0, "4"), (16, 2, 5, 2, None)])
def test_cnn_bf16_eps_fused_wgrad_equals_combine(hw, B, S, chunk, cl, monkeypatch):
    """ε-fused, sample-accumulating stage-1 weight gradient (ε regenerated in the GEMM epilogue,
    samples summed over DSMEM in sample order within a cluster, north_star (3)) against the
    per-sample partials + separate ε combine (BNN_WGRAD_EPS=0): acc_μ, acc_ρ of every tensor within
    fp32 summation error (1e-4 of each tensor's max; a wrong ε, sample or column is O(1)); default
    pairs, clusters of 8 and 4, and a ragged sample chunk (5 samples in chunks of 2)."""
    native = _native()
    model = dict(BF16_CNN, in_h=hw, in_w=hw)
    mu, rho, x, yc, _ = _inputs(model, B, regime="positive")
    accs = []
    if cl is not None:  # clusters of all 8 samples / of 4 (no per-pair partials)
        monkeypatch.setenv("BNN_WGRAD_EPS_CLUSTER", cl)
    for flag in ("0", "1"):
        monkeypatch.setenv("BNN_WGRAD_EPS", flag)
        ctx = native.Context(model, precision="bf16", max_B_loc=B, max_S_loc=S, sample_chunk=chunk, dataset_size=1e4,
                             aug="per_sample")
        accs.append(_acc_parts(ctx, ctx.elbo_partial(_dev(mu), _dev(rho), _dev(x), _dev(yc), B, S, 0xBEEF, 5)))
        torch.cuda.synchronize()
    (m0, r0, l0), (m1, r1, l1) = accs
    for t in ctx.tensors:
        sl = slice(t["offset"], t["offset"] + t["rows"] * t["cols"])
        for name, u, ref in (("acc_mu", m1[sl], m0[sl]), ("acc_rho", r1[sl], r0[sl])):
            assert np.abs(u - ref).max() <= 1e-4 * max(np.abs(ref).max(), 1e-30), (t["t"], name)
    assert l1 == l0


@pytest.mark.parametrize("hw,B,S,aug", [(16, 3, 2, "per_sample"), (32, 2, 3, "per_sample"), (16, 4, 2, "none")])
def test_cnn_bf16_stem_kernel_equals_conv3(hw, B, S, aug, monkeypatch):
    """The stem on stem_fwd_kernel (two taps per MMA through SWIZZLE_NONE core-matrix descriptors,
    pixels on M) against the conv3 gather path (BNN_STEM=0): the stem's stored output, its ReLU
    bitmask's effect on every later layer, and acc_μ / acc_ρ. Same bf16 products, fp32 sums in a
    different order: 1e-2 of each layer's max elementwise (one bf16 ulp), 1e-3 for the accumulators."""
    native = _native()
    model = dict(BF16_CNN, in_h=hw, in_w=hw)
    mu, rho, x, yc, _ = _inputs(model, B, regime="positive")
    res = []
    for flag in ("0", "1"):
        monkeypatch.setenv("BNN_STEM", flag)
        ctx = native.Context(model, precision="bf16", max_B_loc=B, max_S_loc=S, dataset_size=1e4, aug=aug)
        acc = _acc_parts(ctx, ctx.elbo_partial(_dev(mu), _dev(rho), _dev(x), _dev(yc), B, S, 0xBEEF, 5))
        torch.cuda.synchronize()
        n_layers = len(ctx.tensors) // 2
        lay = [ctx.layer_output(l, 0).cpu().numpy() for l in range(n_layers)]
        res.append((acc, lay))
    (a0, l0), (a1, l1) = res
    for l, (o0, o1) in enumerate(zip(l0, l1)):
        assert np.abs(o1 - o0).max() <= 1e-2 * max(np.abs(o0).max(), 1e-30), ("out", l)
    for t in ctx.tensors:
        sl = slice(t["offset"], t["offset"] + t["rows"] * t["cols"])
        for name, u, ref in (("acc_mu", a1[0][sl], a0[0][sl]), ("acc_rho", a1[1][sl], a0[1][sl])):
            assert np.abs(u - ref).max() <= 1e-3 * max(np.abs(ref).max(), 1e-30), (t["t"], name)


_OLD_PATHS = {"BNN_CONV64": "0", "BNN_STEM": "0", "BNN_WGRAD_EPS": "0", "BNN_CONV2_CPS": "1", "BNN_WGRAD_CPS": "1",
              "BNN_WGRAD_S2_TMA": "0"}


@pytest.mark.parametrize("hw,B,S", [(8, 1, 1), (24, 2, 1), (16, 1, 3), (8, 3, 8)])
def test_cnn_bf16_session4_kernels_edge_shapes(hw, B, S, monkeypatch):
    """Edge shapes (one image, one sample, 8×8 inputs where one tile spans several images, 24×24
    (rows not a power of two), S = 8 with B = 3) through the round-2 session-4
    kernels (conv64 fwd / dgrad / ε-fused wgrad, the stem kernel, two CTAs per SM) against the
    same step on the earlier paths: every stored activation and gradient within one bf16 ulp of
    each layer's max (1e-2), acc_μ / acc_ρ within 1e-2 of each tensor's max (their inputs are those
    stored bf16 values, so a rounding tie flipped upstream moves a weight gradient by up to ≈ 2^-8
    of a product: measured 1.6e-3 at 24×24)."""
    native = _native()
    model = dict(BF16_CNN, in_h=hw, in_w=hw)
    mu, rho, x, yc, _ = _inputs(model, B, regime="positive")
    res = []
    for old in (True, False):
        for k, v in _OLD_PATHS.items():
            if old:
                monkeypatch.setenv(k, v)
            else:
                monkeypatch.delenv(k, raising=False)
        ctx = native.Context(model, precision="bf16", max_B_loc=B, max_S_loc=S, dataset_size=1e4, aug="per_sample")
        acc = _acc_parts(ctx, ctx.elbo_partial(_dev(mu), _dev(rho), _dev(x), _dev(yc), B, S, 0xBEEF, 5))
        torch.cuda.synchronize()
        n_layers = len(ctx.tensors) // 2
        lay = [(ctx.layer_output(l, 0).cpu().numpy(),
                ctx.layer_output(l, 1).cpu().numpy() if l < n_layers - 1 else None) for l in range(n_layers)]
        res.append((acc, lay))
    (a0, l0), (a1, l1) = res
    for l, ((o0, g0), (o1, g1)) in enumerate(zip(l0, l1)):
        assert np.abs(o1 - o0).max() <= 1e-2 * max(np.abs(o0).max(), 1e-30), ("out", l)
        if g0 is not None:
            assert np.abs(g1 - g0).max() <= 1e-2 * max(np.abs(g0).max(), 1e-30), ("grad", l)
    for t in ctx.tensors:
        sl = slice(t["offset"], t["offset"] + t["rows"] * t["cols"])
        for name, u, ref in (("acc_mu", a1[0][sl], a0[0][sl]), ("acc_rho", a1[1][sl], a0[1][sl])):
            assert np.abs(u - ref).max() <= 1e-2 * max(np.abs(ref).max(), 1e-30), (t["t"], name)
