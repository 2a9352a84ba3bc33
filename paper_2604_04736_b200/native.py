"""Thin ctypes binding of libbnn.so (include/bnn.h): argument marshalling only.

Every step of the ELBO path runs inside the CUDA library; this module converts torch
tensors to device pointers and Python values to the C structs. There is no fallback: if
libbnn.so is missing or fails to load, lib() raises.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from .configs import n_outputs

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libbnn.so")
_lib = None

MODEL_MLP, MODEL_RESNET18, MODEL_VIT = 0, 1, 2
LOSS = {"ce": 0, "mse": 1, "ce_mean": 2, "mse_mean": 3, "gnll_mean": 4}  # *_mean: exact aggregation
PREC = {"fp32": 0, "bf16": 1}
MODE = {"sample": 0, "data": 1, "hybrid": 2}
AUG = {"none": 0, "per_sample": 1}


class BnnModelDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_widths", C.c_int32), ("widths", C.c_int32 * 16),
                ("in_h", C.c_int32), ("in_w", C.c_int32), ("in_c", C.c_int32),
                ("n_classes", C.c_int32), ("base_width", C.c_int32), ("loss", C.c_int32),
                ("method", C.c_int32), ("dropout_p", C.c_float), ("patch", C.c_int32), ("dim", C.c_int32),
                ("heads", C.c_int32), ("depth", C.c_int32), ("mlp", C.c_int32)]


class BnnConfig(C.Structure):
    _fields_ = [("precision", C.c_int32), ("mode", C.c_int32), ("K", C.c_int32),
                ("G", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
                ("nccl_uid", C.c_void_p), ("max_B_loc", C.c_int32), ("max_S_loc", C.c_int32),
                ("sample_chunk", C.c_int32), ("aug", C.c_int32), ("dataset_size", C.c_double),
                ("device", C.c_int32), ("stream", C.c_void_p), ("comm_timeout_ms", C.c_int32)]


class BnnTensorInfo(C.Structure):
    _fields_ = [("offset", C.c_int64), ("rows", C.c_int32), ("cols", C.c_int32),
                ("t", C.c_int32), ("is_bias", C.c_int32)]


class BnnAdam(C.Structure):
    """bnn_adam (include/bnn.h): hyper-parameters of the fused Adam step."""
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
                ("eps", C.c_float), ("t", C.c_int32)]


class BnnError(RuntimeError):
    pass


def lib():
    """Load libbnn.so (build it first with paper_2604_04736_b200.build if stale)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_SO):
        from . import build
        build.build()
    L = C.CDLL(_SO)
    vp, i32, u32, u64, i64 = C.c_void_p, C.c_int32, C.c_uint32, C.c_uint64, C.c_int64
    L.bnn_get_unique_id.argtypes = [vp]
    L.bnn_init.argtypes = [vp, vp, vp]
    L.bnn_param_layout.argtypes = [vp, vp, vp, vp, i32]
    L.bnn_acc_layout.argtypes = [vp, vp, vp, vp]
    step_args = [vp, vp, vp, vp, vp, vp, i32, i32, i32, u64, u32]
    L.bnn_elbo_step.argtypes = step_args + [vp, vp, vp, vp]
    L.bnn_elbo_step_host.argtypes = step_args + [vp, vp, vp]
    L.bnn_elbo_partial.argtypes = step_args + [vp]
    L.bnn_finalize.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.bnn_sync.argtypes = [vp]
    L.bnn_comm_buckets.argtypes = [vp]
    L.bnn_mean_stats.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, u64, u32, vp]
    L.bnn_elbo_partial_mean.argtypes = step_args + [vp, vp]
    L.bnn_mean_merge.argtypes = [vp, vp, i32, i32, i32, vp]
    L.bnn_finalize_adam.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.bnn_elbo_step_adam.argtypes = step_args + [vp] * 9
    L.bnn_predict.argtypes = [vp, vp, vp, vp, i32, i32, u64, u32, vp, vp]
    L.bnn_eps_fill.argtypes = [u64, u32, u32, u32, u32, u32, u32, u32, vp, vp]
    L.bnn_eps_bench.argtypes = [u64, u64, vp, i32, vp]
    L.bnn_eps_transform_table.argtypes = [i32, vp, vp]
    L.bnn_profile_enable.argtypes = [vp, i32]
    L.bnn_profile_read.argtypes = [vp, vp, i32, vp, vp, i32, vp]
    L.bnn_debug_layer_output.argtypes = [vp, i32, i32, vp, i64, vp]
    L.bnn_launch_count.argtypes = [vp]
    L.bnn_launch_count.restype = i64
    L.bnn_last_error.argtypes = [vp]
    L.bnn_last_error.restype = C.c_char_p
    L.bnn_destroy.argtypes = [vp]
    _lib = L
    return L


def _check(rc, ctx=None):
    if rc != 0:
        msg = lib().bnn_last_error(ctx).decode()
        raise BnnError(f"libbnn error {rc}: {msg}")


def _p(t):
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "tensors must be contiguous CUDA tensors"
    return t.data_ptr()


def _hp(t):
    if t is None:
        return None
    assert not t.is_cuda and t.is_contiguous()
    return t.data_ptr()


def get_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().bnn_get_unique_id(buf))
    return bytes(buf)


def model_desc(model: dict) -> BnnModelDesc:
    d = BnnModelDesc()
    if model["kind"] == "mlp":
        d.kind = MODEL_MLP
        d.n_widths = len(model["widths"])
        for i, w in enumerate(model["widths"]):
            d.widths[i] = w
    elif model["kind"] == "vit":
        d.kind = MODEL_VIT
        d.in_h, d.in_w, d.in_c = model["in_h"], model["in_w"], model["in_c"]
        d.n_classes = model["n_classes"]
        d.patch, d.dim, d.heads, d.depth, d.mlp = (model[k] for k in ("patch", "dim", "heads", "depth", "mlp"))
    else:
        d.kind = MODEL_RESNET18
        d.in_h, d.in_w, d.in_c = model["in_h"], model["in_w"], model["in_c"]
        d.n_classes = model["n_classes"]
        d.base_width = model.get("base_width", 64)
    d.loss = LOSS[model["loss"]]
    if model.get("method", "vi") == "mcd":  # MC dropout
        d.method = 1
        d.dropout_p = float(model.get("dropout_p", 0.1))
    return d


class Context:
    """One rank's bnn_ctx (bnn_init … bnn_destroy)."""

    def __init__(self, model: dict, *, precision="bf16", mode="sample", K=1, G=1, rank=0,
                 world=1, uid: bytes | None = None, max_B_loc=256, max_S_loc=64,
                 sample_chunk=0, aug="none", dataset_size=60000.0, device=0, stream=None,
                 comm_timeout_ms=0):
        self.model = model
        self._L = lib()
        self._desc = model_desc(model)
        cfg = BnnConfig()
        cfg.precision, cfg.mode = PREC[precision], MODE[mode]
        cfg.K, cfg.G, cfg.rank, cfg.world = K, G, rank, world
        self._uid = None
        if uid is not None:
            self._uid = (C.c_uint8 * 128).from_buffer_copy(uid)
            cfg.nccl_uid = C.addressof(self._uid)
        cfg.max_B_loc, cfg.max_S_loc, cfg.sample_chunk = max_B_loc, max_S_loc, sample_chunk
        cfg.aug, cfg.dataset_size, cfg.device = AUG[aug], float(dataset_size), device
        cfg.comm_timeout_ms = comm_timeout_ms
        if stream is None:
            stream = torch.cuda.current_stream(device).cuda_stream
        cfg.stream = stream
        self.device = torch.device("cuda", device)
        self._cfg = cfg
        h = C.c_void_p()
        _check(self._L.bnn_init(C.byref(self._desc), C.byref(cfg), C.byref(h)))
        self._h = h
        n = C.c_int64()
        nt = C.c_int32()
        _check(self._L.bnn_param_layout(h, C.byref(n), C.byref(nt), None, 0), h)
        self.n_params = n.value
        infos = (BnnTensorInfo * nt.value)()
        _check(self._L.bnn_param_layout(h, None, None, infos, nt.value), h)
        self.tensors = [dict(offset=i.offset, rows=i.rows, cols=i.cols, t=i.t, is_bias=i.is_bias)
                        for i in infos]
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        _check(self._L.bnn_acc_layout(h, C.byref(a), C.byref(b), C.byref(c)), h)
        self.acc_rho_offset, self.acc_loss_offset, self.acc_total = a.value, b.value, c.value
        self.n_out = n_outputs(model)

    # -------------------------------------------------------------------------------- steps
    def _y(self, y):
        if y is None:
            return None, None
        if y.dtype == torch.int32:
            return _p(y), None
        return None, _p(y)

    def elbo_step(self, mu, rho, x, y, B_global, S_global, seed, step, *, grad_mu=None,
                  grad_rho=None, loss_dev=None, want_loss=True):
        if grad_mu is None:
            grad_mu = torch.empty_like(mu)
        if grad_rho is None:
            grad_rho = torch.empty_like(rho)
        yc, yr = self._y(y)
        lh = C.c_double()
        _check(self._L.bnn_elbo_step(self._h, _p(mu), _p(rho), _p(x), yc, yr, x.shape[0],
                                     B_global, S_global, seed, step, _p(loss_dev),
                                     C.byref(lh) if want_loss else None, _p(grad_mu),
                                     _p(grad_rho)), self._h)
        return (lh.value if want_loss else None), grad_mu, grad_rho

    def elbo_step_adam(self, mu, rho, x, y, B_global, S_global, seed, step, moments, *, t,
                       lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, grad_mu=None, grad_rho=None,
                       want_loss=True):
        """One training step with the fused Adam update (bnn_elbo_step_adam): mu, rho and
        moments = (m_mu, v_mu, m_rho, v_rho) are updated in place; returns the loss of the
        parameters before the update. grad_mu/grad_rho are written only when given."""
        h = BnnAdam(lr, beta1, beta2, eps, t)
        yc, yr = self._y(y)
        lh = C.c_double()
        m_mu, v_mu, m_rho, v_rho = moments
        _check(self._L.bnn_elbo_step_adam(self._h, _p(mu), _p(rho), _p(x), yc, yr, x.shape[0],
                                          B_global, S_global, seed, step, C.byref(h), _p(m_mu),
                                          _p(v_mu), _p(m_rho), _p(v_rho), None,
                                          C.byref(lh) if want_loss else None, _p(grad_mu),
                                          _p(grad_rho)), self._h)
        return lh.value if want_loss else None

    def finalize_adam(self, mu, rho, acc, moments, *, t, lr=1e-3, beta1=0.9, beta2=0.999,
                      eps=1e-8, grad_mu=None, grad_rho=None):
        h = BnnAdam(lr, beta1, beta2, eps, t)
        loss = torch.zeros(1, dtype=torch.float32, device=self.device)
        m_mu, v_mu, m_rho, v_rho = moments
        _check(self._L.bnn_finalize_adam(self._h, _p(mu), _p(rho), _p(acc), C.byref(h), _p(m_mu),
                                         _p(v_mu), _p(m_rho), _p(v_rho), _p(loss), _p(grad_mu),
                                         _p(grad_rho)), self._h)
        return loss

    def elbo_step_host(self, mu, rho, x_host, y_host, B_global, S_global, seed, step, *,
                       grad_mu, grad_rho):
        yc = _hp(y_host) if y_host is not None and y_host.dtype == torch.int32 else None
        yr = _hp(y_host) if y_host is not None and y_host.dtype != torch.int32 else None
        lh = C.c_double()
        _check(self._L.bnn_elbo_step_host(self._h, _p(mu), _p(rho), _hp(x_host), yc, yr,
                                          x_host.shape[0], B_global, S_global, seed, step,
                                          C.byref(lh), _p(grad_mu), _p(grad_rho)), self._h)
        return lh.value

    def elbo_partial(self, mu, rho, x, y, B_global, S_global, seed, step, acc=None):
        if acc is None:
            acc = torch.zeros(self.acc_total, dtype=torch.float32, device=self.device)
        yc, yr = self._y(y)
        _check(self._L.bnn_elbo_partial(self._h, _p(mu), _p(rho), _p(x), yc, yr, x.shape[0],
                                        B_global, S_global, seed, step, _p(acc)), self._h)
        return acc

    def mean_stats(self, mu, rho, x, y, B_global, S_global, seed, step, width):
        """This rank's exact-aggregation statistic [B_loc, width] (bnn_mean_stats)."""
        out = torch.zeros(x.shape[0] * width, dtype=torch.float32, device=self.device)
        yc, _ = self._y(y)
        _check(self._L.bnn_mean_stats(self._h, _p(mu), _p(rho), _p(x), yc, x.shape[0], B_global,
                                      S_global, seed, step, _p(out)), self._h)
        return out

    def mean_merge(self, stats_list, B_loc, S_global):
        """Merge per-sample-group statistics in list order (bnn_mean_merge)."""
        allst = torch.stack([t.reshape(-1) for t in stats_list]).contiguous()
        out = torch.empty_like(allst[0])
        _check(self._L.bnn_mean_merge(self._h, _p(allst), len(stats_list), B_loc, S_global, _p(out)), self._h)
        return out

    def elbo_partial_mean(self, mu, rho, x, y, B_global, S_global, seed, step, stats, acc=None):
        if acc is None:
            acc = torch.zeros(self.acc_total, dtype=torch.float32, device=self.device)
        yc, yr = self._y(y)
        _check(self._L.bnn_elbo_partial_mean(self._h, _p(mu), _p(rho), _p(x), yc, yr, x.shape[0],
                                             B_global, S_global, seed, step, _p(stats), _p(acc)),
               self._h)
        return acc

    def finalize(self, mu, rho, acc):
        gmu, grho = torch.empty_like(mu), torch.empty_like(rho)
        loss = torch.zeros(1, dtype=torch.float32, device=self.device)
        _check(self._L.bnn_finalize(self._h, _p(mu), _p(rho), _p(acc), _p(loss), _p(gmu),
                                    _p(grho)), self._h)
        return loss, gmu, grho

    def predict(self, mu, rho, x, S_global, seed, step):
        B = x.shape[0]
        mean = torch.empty(B, self.n_out, dtype=torch.float32, device=self.device)
        var = torch.empty_like(mean)
        _check(self._L.bnn_predict(self._h, _p(mu), _p(rho), _p(x), B, S_global, seed, step,
                                   _p(mean), _p(var)), self._h)
        return mean, var

    # -------------------------------------------------------------------------------- misc
    def profile(self, on: bool):
        _check(self._L.bnn_profile_enable(self._h, 1 if on else 0), self._h)

    def profile_read(self) -> dict:
        names = C.create_string_buffer(1024)
        ms = (C.c_double * 32)()
        n = (C.c_int64 * 32)()
        cnt = C.c_int32()
        _check(self._L.bnn_profile_read(self._h, names, 1024, ms, n, 32, C.byref(cnt)), self._h)
        keys = names.value.decode().split(",") if cnt.value else []
        return {k: dict(ms=ms[i], launches=n[i]) for i, k in enumerate(keys)}

    def layer_output(self, layer: int, which: int = 0) -> torch.Tensor:
        """Test hook: stored output (0) or its gradient (1) of `layer` from the last step."""
        cap = 1 << 27
        out = torch.empty(cap, dtype=torch.float32, device=self.device)
        n = C.c_int64()
        _check(self._L.bnn_debug_layer_output(self._h, layer, which, _p(out), cap, C.byref(n)), self._h)
        return out[:n.value].clone()

    def sync(self):
        """bnn_sync: host wait for the context's streams, polling the communicator."""
        _check(self._L.bnn_sync(self._h), self._h)

    def comm_buckets(self) -> int:
        return int(self._L.bnn_comm_buckets(self._h))

    def launch_count(self) -> int:
        return int(self._L.bnn_launch_count(self._h))

    def close(self):
        if getattr(self, "_h", None):
            self._L.bnn_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def eps_fill(seed, step, s, t, r0, nr, c0, nc, device=0) -> torch.Tensor:
    out = torch.empty(nr, nc, dtype=torch.float32, device=torch.device("cuda", device))
    _check(lib().bnn_eps_fill(seed, step, s, t, r0, nr, c0, nc, _p(out),
                              torch.cuda.current_stream(device).cuda_stream))
    return out


def eps_transform_table(which: int, device=0) -> torch.Tensor:
    out = torch.empty(1 << 24, dtype=torch.float32, device=torch.device("cuda", device))
    _check(lib().bnn_eps_transform_table(which, _p(out),
                                         torch.cuda.current_stream(device).cuda_stream))
    return out


def eps_bench(n4: int, seed: int, sink: torch.Tensor, grid: int):
    _check(lib().bnn_eps_bench(n4, seed, _p(sink), grid,
                               torch.cuda.current_stream(sink.device).cuda_stream))
