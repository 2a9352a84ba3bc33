"""Model and workload descriptions (plain data; no arithmetic of the method).

The five workloads C1-C5 are BASELINE.json's ``configs``:

* C1 — Bayesian MLP 8-16-1 regression (MSE), B=32, S=4: the small case the oracle
  finishes in seconds.
* C2 — Bayesian MLP 784-1024-1024-10 (CE), B=256, S=64 on one B200: the bench workload
  at N=1 (BASELINE.json ``configs[1]``).
* C3 — ResNet-18-shaped Bayesian CNN on 32×32×3, B=128, S=8 per GPU (weak scaling).
* C4 — the same CNN, fixed S=64 (strong scaling), sample-sharded vs data-sharded.
* C5 — 4 sample groups × 2 data groups, S=32, global batch 256.
* C6 — not a BASELINE config: the MC-dropout use case shape (MLP
  96-128-128-24 trained on the MSE of the averaged predictions), dropout
  p = 0.1 (reading R25), B=256, S=64 (the paper's batch and sample counts for this use case
  are not stated; C2's are used).

|D| values follow SURVEY.md §8(d): 1024 (C1), 60000 (C2), 45000 (C3-C5).
"""
from __future__ import annotations

MODELS = {
    "mlp_8_16_1": dict(kind="mlp", widths=[8, 16, 1], loss="mse"),
    "mlp_784_1024_1024_10": dict(kind="mlp", widths=[784, 1024, 1024, 10], loss="ce"),
    "resnet18_cifar": dict(kind="resnet18", in_h=32, in_w=32, in_c=3, n_classes=10,
                           base_width=64, loss="ce"),
    "mcd_mlp_96_128_128_24": dict(kind="mlp", widths=[96, 128, 128, 24], loss="mse_mean",
                                  method="mcd", dropout_p=0.1),
    # use case 1: 4×4 patches, width 192, 3 heads, 6 layers, MLP 768
    "vit_cifar": dict(kind="vit", in_h=32, in_w=32, in_c=3, patch=4, dim=192, heads=3, depth=6,
                      mlp=768, n_classes=10, loss="ce"),
}

CONFIGS = {
    "C1": dict(model="mlp_8_16_1", B=32, S=4, D=1024.0, aug="none", K=1, G=1),
    "C2": dict(model="mlp_784_1024_1024_10", B=256, S=64, D=60000.0, aug="none", K=1, G=1),
    "C3": dict(model="resnet18_cifar", B=128, S_per_gpu=8, D=45000.0, aug="per_sample"),
    "C4": dict(model="resnet18_cifar", B=128, S=64, D=45000.0, aug="per_sample"),
    "C5": dict(model="resnet18_cifar", B=256, S=32, D=45000.0, aug="per_sample", K=4, G=2),
    "C6": dict(model="mcd_mlp_96_128_128_24", B=256, S=64, D=1.0, aug="none", K=1, G=1),
    # not a BASELINE config: SURVEY §8(f) f3, the paper's primary use case (ViT on CIFAR-10)
    "C7": dict(model="vit_cifar", B=128, S_per_gpu=8, D=45000.0, aug="per_sample"),
}


def layout(model: dict) -> list[dict]:
    """Parameter tensors in model order.

    Each layer contributes a weight tensor t=2l viewed as [rows=c_out, cols=k·k·c_in]
    (OHWI, c_in fastest) and a bias tensor t=2l+1 viewed as [1, c_out]. Returned dicts
    carry t, offset, rows, cols, the layer's fan-in and its role ("hidden"/"out" for the MLP;
    "stem", "c1"/"c2" (first/second conv of a BasicBlock), "proj", "out" for the ResNet) — the
    last two are used only by the initialiser.
    """
    if model["kind"] == "vit":
        return _vit_layout(model)
    layers = []  # (cin, cout, k, role)
    if model["kind"] == "mlp":
        w = model["widths"]
        for i in range(1, len(w)):
            layers.append((w[i - 1], w[i], 1, "hidden" if i < len(w) - 1 else "out"))
    elif model["kind"] == "resnet18":
        b = model.get("base_width", 64)
        layers.append((model["in_c"], b, 3, "stem"))
        width = b
        for stage in range(4):
            cout = b << stage
            for blk in range(2):
                stride = 2 if (stage > 0 and blk == 0) else 1
                layers.append((width, cout, 3, "c1"))
                layers.append((cout, cout, 3, "c2"))
                if stride != 1 or width != cout:
                    layers.append((width, cout, 1, "proj"))
                width = cout
        layers.append((width, model["n_classes"], 1, "out"))
    else:
        raise ValueError(model["kind"])
    out, off = [], 0
    for l, (cin, cout, k, role) in enumerate(layers):
        cols = k * k * cin
        out.append(dict(t=2 * l, offset=off, rows=cout, cols=cols, fan_in=cols, role=role))
        off += cout * cols
        out.append(dict(t=2 * l + 1, offset=off, rows=1, cols=cout, fan_in=cols, role=role))
        off += cout
    return out


def _vit_layout(model: dict) -> list[dict]:
    """ViT tensors in the order of oracle/vit_oracle.c and the library: each
    [rows, cols] (1-D tensors [1, n]; pos [1, T·D]); role and fan-in for the initialiser."""
    D, M, O = model["dim"], model["mlp"], model["n_classes"]
    T = 1 + (model["in_h"] // model["patch"]) * (model["in_w"] // model["patch"])
    pk = model["patch"] * model["patch"] * model["in_c"]
    spec = [(D, pk, "w", pk), (1, D, "b", pk), (1, D, "cls", D), (1, T * D, "pos", D)]
    for _ in range(model["depth"]):
        spec += [(1, D, "ln_g", D), (1, D, "ln_b", D), (3 * D, D, "w", D), (1, 3 * D, "b", D),
                 (D, D, "w", D), (1, D, "b", D), (1, D, "ln_g", D), (1, D, "ln_b", D),
                 (M, D, "w", D), (1, M, "b", D), (D, M, "w", M), (1, D, "b", M)]
    spec += [(1, D, "ln_g", D), (1, D, "ln_b", D), (O, D, "w", D), (1, O, "b", D)]
    out, off = [], 0
    for t, (r, c, role, fan) in enumerate(spec):
        out.append(dict(t=t, offset=off, rows=r, cols=c, fan_in=fan, role=role))
        off += r * c
    return out


def n_params(model: dict) -> int:
    last = layout(model)[-1]
    return last["offset"] + last["rows"] * last["cols"]


def n_outputs(model: dict) -> int:
    return model["widths"][-1] if model["kind"] == "mlp" else model["n_classes"]  # CNN, ViT


def input_shape(model: dict) -> tuple:
    """Per-example input shape: (features,) for the MLP, (H, W, C) NHWC for the CNN."""
    if model["kind"] == "mlp":
        return (model["widths"][0],)
    return (model["in_h"], model["in_w"], model["in_c"])
