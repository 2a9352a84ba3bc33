"""ctypes binding of the CPU oracle (oracle/bnn_oracle.c).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py. The product package never imports it.
The oracle shares no code with the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

MLP, RESNET18 = 0, 1
CE, MSE, GNLL = 0, 1, 2
RELU, TANH = 0, 1
AUG_NONE, AUG_PER_SAMPLE = 0, 1


class OrcModel(C.Structure):
    _fields_ = [("kind", C.c_int), ("n_widths", C.c_int), ("widths", C.c_int * 16),
                ("in_h", C.c_int), ("in_w", C.c_int), ("in_c", C.c_int),
                ("n_classes", C.c_int), ("base_width", C.c_int), ("loss", C.c_int),
                ("act", C.c_int), ("mcd", C.c_int), ("dropout_p", C.c_double)]


def build():
    subprocess.check_call([os.path.join(_HERE, "build.sh")])


def lib():
    global _lib
    if _lib is None:
        srcs = [os.path.join(_HERE, f) for f in ("bnn_oracle.c", "vit_oracle.c")]
        if not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(f) for f in srcs):
            build()
        _lib = C.CDLL(_LIB)
        _lib.orc_log24.restype = C.c_float
        _lib.orc_log24.argtypes = [C.c_float]
        _lib.orc_eps.restype = C.c_float
        _lib.orc_eps.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                 C.c_uint32]
        _lib.orc_n_params.restype = C.c_long
        _lib.orc_eps_fill.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                      C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p]
        _lib.orc_aug_params.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                        C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_philox_fill.argtypes = [C.c_void_p, C.c_void_p, C.c_long, C.c_void_p]
        _lib.orc_elbo_partial.argtypes = [C.c_void_p] + [C.c_void_p] * 5 + [C.c_int] * 6 + [
            C.c_uint64, C.c_uint32, C.c_int, C.c_void_p, C.c_int]
        _lib.orc_elbo_partial_ex.argtypes = [C.c_void_p] + [C.c_void_p] * 5 + [C.c_int] * 6 + [
            C.c_uint64, C.c_uint32, C.c_int, C.c_void_p, C.c_int, C.c_int]
        _lib.orc_finalize.argtypes = [C.c_void_p] * 4 + [C.c_double] + [C.c_void_p] * 4
        _lib.orc_forward.argtypes = [C.c_void_p] * 4 + [C.c_int] * 3 + [C.c_uint64, C.c_uint32,
                                                                         C.c_int, C.c_void_p]
        _lib.orc_forward_ex.argtypes = [C.c_void_p] * 4 + [C.c_int] * 3 + [C.c_uint64, C.c_uint32,
                                                                            C.c_int, C.c_void_p, C.c_int]
        _lib.orc_elbo_step_mean.argtypes = [C.c_void_p] * 6 + [C.c_int] * 2 + [
            C.c_uint64, C.c_uint32, C.c_int, C.c_double] + [C.c_void_p] * 4 + [C.c_int]
        _lib.orc_mean_stats.argtypes = [C.c_void_p] * 5 + [C.c_int] * 4 + [C.c_uint64, C.c_uint32,
                                                                           C.c_int, C.c_void_p]
        _lib.orc_elbo_partial_mean.argtypes = [C.c_void_p] * 6 + [C.c_int] * 6 + [
            C.c_uint64, C.c_uint32, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int]
        _lib.orc_dropout_keep.argtypes = [C.c_uint64] + [C.c_uint32] * 6
        _lib.orc_adam.argtypes = [C.c_long] + [C.c_void_p] * 4 + [C.c_double] * 4 + [C.c_int]
        _lib.orc_predict.argtypes = [C.c_void_p] * 4 + [C.c_int] * 2 + [C.c_uint64, C.c_uint32,
                                                                         C.c_void_p, C.c_void_p]
        # ViT (vit_oracle.c)
        _lib.orc_vit_n_params.restype = C.c_long
        _lib.orc_vit_n_params.argtypes = [C.c_void_p]
        _lib.orc_vit_n_tensors.argtypes = [C.c_void_p]
        _lib.orc_vit_tensor_info.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        _lib.orc_vit_elbo_partial.argtypes = [C.c_void_p] * 5 + [C.c_int] * 6 + [
            C.c_uint64, C.c_uint32, C.c_int, C.c_void_p, C.c_int]
        _lib.orc_vit_forward.argtypes = [C.c_void_p] * 4 + [C.c_int] * 3 + [C.c_uint64, C.c_uint32, C.c_int,
                                                                             C.c_void_p]
        _lib.orc_vit_set_emu_weights.argtypes = [C.c_int]
        _lib.orc_finalize_p.argtypes = [C.c_long] + [C.c_void_p] * 3 + [C.c_double] + [C.c_void_p] * 4
    return _lib


# ---------------------------------------------------------------- Bayesian ViT (f3)
class OrcVit(C.Structure):
    _fields_ = [("in_h", C.c_int), ("in_w", C.c_int), ("in_c", C.c_int), ("patch", C.c_int),
                ("dim", C.c_int), ("heads", C.c_int), ("depth", C.c_int), ("mlp", C.c_int),
                ("n_classes", C.c_int)]


def vit_struct(model: dict) -> OrcVit:
    v = OrcVit()
    for f, _ in OrcVit._fields_:
        setattr(v, f, int(model[f]))
    return v


def vit_n_params(model) -> int:
    return int(lib().orc_vit_n_params(C.byref(vit_struct(model))))


def vit_tensor_infos(model):
    v = vit_struct(model)
    n = lib().orc_vit_n_tensors(C.byref(v))
    out = []
    for t in range(n):
        info = np.zeros(3, np.int64)
        assert lib().orc_vit_tensor_info(C.byref(v), t, info.ctypes.data) == 0
        out.append(dict(t=t, offset=int(info[0]), rows=int(info[1]), cols=int(info[2])))
    return out


def vit_elbo_partial(model, mu, rho, x, y_cls, B_glob, b_offset, S_glob, s0, s1, seed, step, aug=AUG_NONE,
                     nthreads=0, emu=False):
    """[acc_μ (P) | acc_ρ (P) | L_data] of samples [s0, s1) (vit_oracle.c). emu="weights": only the
    BF16 mode's sampled weights RN_bf16(fma_f32(σ, ε, μ)) (R14), the rest exact (conditioning probe)."""
    lib().orc_vit_set_emu_weights(1 if emu == "weights" else 0)
    v = vit_struct(model)
    P = vit_n_params(model)
    mu, rho, x = _d(mu), _d(rho), _d(x)
    yc = np.ascontiguousarray(y_cls, np.int32)
    acc = np.zeros(2 * P + 1, np.float64)
    rc = lib().orc_vit_elbo_partial(C.byref(v), _p(mu), _p(rho), _p(x), _p(yc), x.shape[0], b_offset, B_glob,
                                    S_glob, s0, s1, seed, step, aug, _p(acc), nthreads)
    lib().orc_vit_set_emu_weights(0)
    assert rc == 0, rc
    return acc


def vit_finalize(mu, rho, acc, D):
    P = (len(acc) - 1) // 2
    mu, rho, acc = _d(mu), _d(rho), _d(acc)
    gmu, grho = np.zeros(P), np.zeros(P)
    loss, kl = C.c_double(), C.c_double()
    assert lib().orc_finalize_p(P, _p(mu), _p(rho), _p(acc), D, C.byref(loss), C.byref(kl), _p(gmu),
                                _p(grho)) == 0
    return dict(loss=loss.value, kl=kl.value, grad_mu=gmu, grad_rho=grho, L_data=acc[2 * P])


def vit_elbo_step(model, mu, rho, x, y_cls, S, seed, step, D, aug=AUG_NONE, nthreads=0):
    B = np.asarray(x).shape[0]
    acc = vit_elbo_partial(model, mu, rho, x, y_cls, B, 0, S, 0, S, seed, step, aug, nthreads)
    return vit_finalize(mu, rho, acc, D)


def vit_forward(model, mu, rho, x, s0, s1, seed, step, aug=AUG_NONE):
    """logits [s1 − s0, B, classes]"""
    v = vit_struct(model)
    mu, rho, x = _d(mu), _d(rho), _d(x)
    B = x.shape[0]
    out = np.zeros((s1 - s0, B, int(model["n_classes"])), np.float64)
    assert lib().orc_vit_forward(C.byref(v), _p(mu), _p(rho), _p(x), B, s0, s1, seed, step, aug, _p(out)) == 0
    return out


def model_struct(model: dict, act: str = "relu") -> OrcModel:
    m = OrcModel()
    m.kind = MLP if model["kind"] == "mlp" else RESNET18
    if model["kind"] == "mlp":
        w = model["widths"]
        m.n_widths = len(w)
        for i, v in enumerate(w):
            m.widths[i] = v
    else:
        m.in_h, m.in_w, m.in_c = model["in_h"], model["in_w"], model["in_c"]
        m.n_classes = model["n_classes"]
        m.base_width = model.get("base_width", 64)
    # the loss family; "*_mean" (exact aggregation) is selected by elbo_step(agg="mean")
    m.loss = {"ce": CE, "mse": MSE, "gnll": GNLL, "ce_mean": CE, "mse_mean": MSE,
              "gnll_mean": GNLL}[model["loss"]]
    m.act = RELU if act == "relu" else TANH
    if model.get("method", "vi") == "mcd":  # MC dropout (R25)
        m.mcd = 1
        m.dropout_p = float(model.get("dropout_p", 0.1))
    return m


def _p(a):
    return None if a is None else a.ctypes.data


def _d(a):
    return None if a is None else np.ascontiguousarray(a, np.float64)


# ---------------------------------------------------------------- EPS-v1 (docs/EPS.md)
def philox(ctr, key):
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox_fill(c.ctypes.data, k.ctypes.data, 1, out.ctypes.data)
    return out


def philox_fill(ctr, key, n):
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    out = np.zeros((n, 4), np.uint32)
    lib().orc_philox_fill(c.ctypes.data, k.ctypes.data, n, out.ctypes.data)
    return out


def log24_all():
    out = np.empty(1 << 24, np.float32)
    lib().orc_log24_all(out.ctypes.data_as(C.c_void_p))
    return out


def sincos2pi24_all():
    c = np.empty(1 << 24, np.float32)
    s = np.empty(1 << 24, np.float32)
    lib().orc_sincos2pi24_all(c.ctypes.data_as(C.c_void_p), s.ctypes.data_as(C.c_void_p))
    return c, s


def eps(seed, step, s, t, r, c) -> float:
    return lib().orc_eps(seed, step, s, t, r, c)


def eps_fill(seed, step, s, t, r0, nr, c0, nc) -> np.ndarray:
    out = np.empty((nr, nc), np.float32)
    lib().orc_eps_fill(seed, step, s, t, r0, nr, c0, nc, out.ctypes.data)
    return out


def aug_params(seed, step, s, b):
    dx, dy, fl = C.c_int(), C.c_int(), C.c_int()
    lib().orc_aug_params(seed, step, s, b, C.byref(dx), C.byref(dy), C.byref(fl))
    return dx.value, dy.value, fl.value


# ---------------------------------------------------------------- exact aggregation, sharded
def mean_stats(model, mu, rho, x, y_cls, b_offset, s0, s1, seed, step, aug=AUG_NONE):
    """This shard's statistic of the mean prediction (orc_mean_stats): [B_loc, 1] (CE) or
    [B_loc, outputs] (MSE)."""
    m = model_struct(model)
    mu, rho, x = _d(mu), _d(rho), _d(x)
    yc = None if y_cls is None else np.ascontiguousarray(y_cls, np.int32)
    B = x.shape[0]
    O = model["widths"][-1] if model["kind"] == "mlp" else model["n_classes"]
    w = {"ce": 1, "mse": O, "gnll": 2 * O}[model["loss"]]
    out = np.zeros((B, w))
    assert lib().orc_mean_stats(C.byref(m), _p(mu), _p(rho), _p(x), _p(yc), B, b_offset, s0, s1, seed,
                                step, aug, _p(out)) == 0
    return out


def elbo_partial_mean(model, mu, rho, x, y_cls, y_reg, B_glob, b_offset, S_glob, s0, s1, seed, step,
                      gstats, add_loss, aug=AUG_NONE, nthreads=0):
    """This shard's acc partial of the exact step given the merged statistic
    (orc_elbo_partial_mean)."""
    m = model_struct(model)
    P = lib().orc_n_params(C.byref(m))
    mu, rho, x, yr, g = _d(mu), _d(rho), _d(x), _d(y_reg), _d(gstats)
    yc = None if y_cls is None else np.ascontiguousarray(y_cls, np.int32)
    acc = np.zeros(2 * P + 1)
    assert lib().orc_elbo_partial_mean(C.byref(m), _p(mu), _p(rho), _p(x), _p(yc), _p(yr), x.shape[0],
                                       b_offset, B_glob, S_glob, s0, s1, seed, step, aug, _p(g),
                                       1 if add_loss else 0, _p(acc), nthreads) == 0
    return acc


# ---------------------------------------------------------------- MC dropout mask (f4)
def dropout_keep(seed, step, s, layer, b, j, p):
    """Keep decision of unit j of hidden layer `layer`, global example b, sample s (R25)."""
    p24 = int(round(p * 16777216.0))
    return bool(lib().orc_dropout_keep(seed, step, s, layer, b, j, p24))


# ---------------------------------------------------------------- Adam
def adam(theta, g, m, v, lr, beta1, beta2, eps, t):
    """In-place Adam update of fp64 arrays theta, m, v with gradient g (oracle/bnn_oracle.c
    orc_adam: Kingma & Ba Algorithm 1, the optimizer PAPER.md:166 names)."""
    for a in (theta, g, m, v):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    lib().orc_adam(theta.size, _p(theta), _p(g), _p(m), _p(v), lr, beta1, beta2, eps, t)


# ---------------------------------------------------------------- model
def n_params(model, act="relu"):
    m = model_struct(model, act)
    return lib().orc_n_params(C.byref(m))


def tensor_infos(model):
    m = model_struct(model)
    n = lib().orc_n_tensors(C.byref(m))
    out = []
    info = (C.c_long * 7)()
    for t in range(n):
        assert lib().orc_tensor_info(C.byref(m), t, info) == 0
        out.append(dict(t=t, offset=info[0], rows=info[1], cols=info[2]))
    return out


def elbo_partial(model, mu, rho, x, y_cls, y_reg, B_glob, b_offset, S_glob, s0, s1, seed, step,
                 aug=AUG_NONE, nthreads=0, act="relu", emu=False):
    """emu=True: the BF16 tensor-core mode's rounding points (reading R14);
    emu="weights": only the BF16 mode's sampled weight w_s = RN_bf16(fma_f32(σ, ε, μ)) (R14),
    everything else exact fp64 (the conditioning probe of DESIGN.md R26)."""
    m = model_struct(model, act)
    P = lib().orc_n_params(C.byref(m))
    mu, rho, x, yr = _d(mu), _d(rho), _d(x), _d(y_reg)
    yc = None if y_cls is None else np.ascontiguousarray(y_cls, np.int32)
    B_loc = x.shape[0]
    acc = np.zeros(2 * P + 1, np.float64)
    rc = lib().orc_elbo_partial_ex(C.byref(m), _p(mu), _p(rho), _p(x), _p(yc), _p(yr), B_loc,
                                   b_offset, B_glob, S_glob, s0, s1, seed, step, aug, _p(acc),
                                   nthreads, 2 if emu == "weights" else (1 if emu else 0))
    assert rc == 0, rc
    return acc


def finalize(model, mu, rho, acc, D, act="relu"):
    m = model_struct(model, act)
    P = lib().orc_n_params(C.byref(m))
    mu, rho, acc = _d(mu), _d(rho), _d(acc)
    gmu = np.zeros(P)
    grho = np.zeros(P)
    loss, kl = C.c_double(), C.c_double()
    rc = lib().orc_finalize(C.byref(m), _p(mu), _p(rho), _p(acc), D, C.byref(loss), C.byref(kl),
                            _p(gmu), _p(grho))
    assert rc == 0
    return dict(loss=loss.value, kl=kl.value, grad_mu=gmu, grad_rho=grho, L_data=acc[2 * P])


def elbo_step(model, mu, rho, x, y_cls, y_reg, S, seed, step, D, aug=AUG_NONE, nthreads=0,
              act="relu", emu=False, agg="sample"):
    """agg="sample": L_data = mean over samples of the per-sample loss (Alg. 1 l.9, the path's
    default); agg="mean": the loss of the mean prediction (exact aggregation, PAPER.md:272-281,
    orc_elbo_step_mean)."""
    B = np.asarray(x).shape[0]
    if agg == "mean":
        assert not emu
        m = model_struct(model, act)
        P = lib().orc_n_params(C.byref(m))
        mu, rho, x, yr = _d(mu), _d(rho), _d(x), _d(y_reg)
        yc = None if y_cls is None else np.ascontiguousarray(y_cls, np.int32)
        gmu, grho = np.zeros(P), np.zeros(P)
        loss, kl = C.c_double(), C.c_double()
        rc = lib().orc_elbo_step_mean(C.byref(m), _p(mu), _p(rho), _p(x), _p(yc), _p(yr), B, S,
                                      seed, step, aug, D, C.byref(loss), C.byref(kl), _p(gmu),
                                      _p(grho), nthreads)
        assert rc == 0, rc
        return dict(loss=loss.value, kl=kl.value, grad_mu=gmu, grad_rho=grho,
                    L_data=loss.value - kl.value / D)
    assert agg == "sample"
    assert model["loss"] != "gnll", "the Gaussian NLL of the predictive distribution needs agg='mean'"
    acc = elbo_partial(model, mu, rho, x, y_cls, y_reg, B, 0, S, 0, S, seed, step, aug, nthreads,
                       act, emu)
    return finalize(model, mu, rho, acc, D, act)


def forward(model, mu, rho, x, s0, s1, seed, step, aug=AUG_NONE, act="relu", emu=False):
    m = model_struct(model, act)
    mu, rho, x = _d(mu), _d(rho), _d(x)
    B = x.shape[0]
    O = model["widths"][-1] if model["kind"] == "mlp" else model["n_classes"]
    z = np.zeros((s1 - s0, B, O))
    assert lib().orc_forward_ex(C.byref(m), _p(mu), _p(rho), _p(x), B, s0, s1, seed, step, aug,
                                _p(z), 1 if emu else 0) == 0
    return z


def predict(model, mu, rho, x, S, seed, step):
    m = model_struct(model)
    mu, rho, x = _d(mu), _d(rho), _d(x)
    B = x.shape[0]
    O = model["widths"][-1] if model["kind"] == "mlp" else model["n_classes"]
    mean = np.zeros((B, O))
    var = np.zeros((B, O))
    assert lib().orc_predict(C.byref(m), _p(mu), _p(rho), _p(x), B, S, seed, step, _p(mean),
                             _p(var)) == 0
    return mean, var


def layer_output(model, mu, rho, x, b, s, seed, step, layer, aug=AUG_NONE, emu=False):
    """Stored output of `layer` for example b, sample s (test hook)."""
    m = model_struct(model)
    L = lib()
    L.orc_layer_output.restype = C.c_long
    L.orc_layer_output.argtypes = [C.c_void_p] * 4 + [C.c_int] * 2 + [C.c_uint64, C.c_uint32] + \
        [C.c_int] * 3 + [C.c_void_p]
    mu, rho, x = _d(mu), _d(rho), _d(x)
    out = np.zeros(1 << 22)
    n = L.orc_layer_output(C.byref(m), _p(mu), _p(rho), _p(x), b, s, seed, step, aug,
                           1 if emu else 0, layer, _p(out))
    assert n > 0, n
    return out[:n]


def layer_grad(model, mu, rho, x, y_cls, y_reg, b, s, seed, step, layer, aug=AUG_NONE, emu=False):
    """Unscaled dℓ/d(stored output of `layer`) for example b, sample s (test hook)."""
    m = model_struct(model)
    L = lib()
    L.orc_layer_grad.restype = C.c_long
    L.orc_layer_grad.argtypes = [C.c_void_p] * 6 + [C.c_int] * 2 + [C.c_uint64, C.c_uint32] + \
        [C.c_int] * 3 + [C.c_void_p]
    mu, rho, x, yr = _d(mu), _d(rho), _d(x), _d(y_reg)
    yc = None if y_cls is None else np.ascontiguousarray(y_cls, np.int32)
    out = np.zeros(1 << 22)
    n = L.orc_layer_grad(C.byref(m), _p(mu), _p(rho), _p(x), _p(yc), _p(yr), b, s, seed, step, aug,
                         1 if emu else 0, layer, _p(out))
    assert n > 0, n
    return out[:n]


def layer_dump(model, mu, rho, x, y_cls, y_reg, b, s, seed, step, aug=AUG_NONE, emu=False, grad=False):
    """All layers' stored outputs (grad=False) or unscaled dℓ/d(stored output) (grad=True) for
    example b, sample s, concatenated in layer order (test hook; one pass for all layers)."""
    m = model_struct(model)
    L = lib()
    L.orc_layer_dump.restype = C.c_long
    L.orc_layer_dump.argtypes = [C.c_void_p] * 6 + [C.c_int] * 2 + [C.c_uint64, C.c_uint32] + \
        [C.c_int] * 3 + [C.c_void_p]
    mu, rho, x, yr = _d(mu), _d(rho), _d(x), _d(y_reg)
    yc = None if y_cls is None else np.ascontiguousarray(y_cls, np.int32)
    out = np.zeros(1 << 23)
    n = L.orc_layer_dump(C.byref(m), _p(mu), _p(rho), _p(x), _p(yc), _p(yr), b, s, seed, step, aug,
                         1 if emu else 0, 1 if grad else 0, _p(out))
    assert n > 0, n
    return out[:n]
