"""An independent fp64 PyTorch-CPU formulation of the ELBO step, used only to pin the oracle.

Forward uses library routines (F.linear, F.conv2d, F.cross_entropy, F.softplus); the
backward is torch autograd. It shares no code with oracle/bnn_oracle.c: only the ε values
(oracle.eps_fill, itself pinned in test_eps_oracle.py) and the augmentation offsets
(oracle.aug_params) are taken from the oracle, so that both evaluate the same draw.
"""
import numpy as np
import torch
import torch.nn.functional as F

import oracle as O
from paper_2604_04736_b200.configs import layout


def _augment(x, seed, step, s, b_global):
    """docs/EPS.md §4: zero-pad by 4, crop at (dy, dx), then optional horizontal flip."""
    dx, dy, fl = O.aug_params(seed, step, s, b_global)
    H, W, C = x.shape
    p = torch.zeros(H + 8, W + 8, C, dtype=x.dtype)
    p[4:4 + H, 4:4 + W] = x
    out = p[dy:dy + H, dx:dx + W]
    if fl:
        out = torch.flip(out, dims=[1])
    return out


def _forward(model, ws, x, act, masks=None):
    """x: [B, features] (MLP) or [B, H, W, C] (CNN); ws: list of tensors in layout order;
    masks[l]: MC-dropout keep mask of hidden layer l ([B, width], already scaled by 1/(1−p))."""
    a = torch.relu if act == "relu" else torch.tanh
    if model["kind"] == "mlp":
        h = x
        n = len(ws) // 2
        for l in range(n):
            W, b = ws[2 * l], ws[2 * l + 1].reshape(-1)
            h = F.linear(h, W, b)
            if l < n - 1:
                h = a(h)
                if masks is not None:
                    h = h * masks[l]
        return h
    # ResNet-18 (reading R12), NCHW for torch
    cin = model["in_c"]
    it = iter(range(len(ws) // 2))

    def conv(h, stride, pad, k):
        l = next(it)
        W = ws[2 * l]
        cout = W.shape[0]
        W4 = W.reshape(cout, k, k, -1).permute(0, 3, 1, 2)
        return F.conv2d(h, W4, ws[2 * l + 1].reshape(-1), stride=stride, padding=pad)

    h = x.permute(0, 3, 1, 2)
    h = a(conv(h, 1, 1, 3))
    bw = model.get("base_width", 64)
    width = bw
    for stage in range(4):
        cout = bw << stage
        for blk in range(2):
            stride = 2 if (stage > 0 and blk == 0) else 1
            y = a(conv(h, stride, 1, 3))
            y = conv(y, 1, 1, 3)
            if stride != 1 or width != cout:
                sc = conv(h, stride, 0, 1)
            else:
                sc = h
            h = a(y + sc)
            width = cout
    h = h.mean(dim=(2, 3))
    l = next(it)
    return F.linear(h, ws[2 * l], ws[2 * l + 1].reshape(-1))


def elbo(model, mu, rho, x, y_cls, y_reg, S, seed, step, D, aug=False, act="relu", agg="sample"):
    """Return loss, L_data, KL, grad_mu, grad_rho (numpy fp64) via autograd. agg="mean": the
    loss of the mean prediction (mean softmax probability for CE, mean output for MSE)."""
    lay = layout(model)
    mu_t = torch.tensor(np.asarray(mu, np.float64), requires_grad=True)
    rho_t = torch.tensor(np.asarray(rho, np.float64), requires_grad=True)
    sigma = F.softplus(rho_t)
    X = torch.tensor(np.asarray(x, np.float64))
    B = X.shape[0]
    L_data = 0.0
    zs = []
    mcd = model.get("method", "vi") == "mcd"
    for s in range(S):
        ws = []
        for ti in lay:
            n = ti["rows"] * ti["cols"]
            sl = slice(ti["offset"], ti["offset"] + n)
            if mcd:  # MC dropout: deterministic weights μ
                ws.append(mu_t[sl].reshape(ti["rows"], ti["cols"]))
                continue
            e = torch.tensor(O.eps_fill(seed, step, s, ti["t"], 0, ti["rows"], 0, ti["cols"])
                             .astype(np.float64)).reshape(-1)
            ws.append((mu_t[sl] + sigma[sl] * e).reshape(ti["rows"], ti["cols"]))
        Xs = X
        if aug:
            Xs = torch.stack([_augment(X[b], seed, step, s, b) for b in range(B)])
        masks = None
        if mcd:  # keep decisions from the oracle's mask function (pinned separately)
            p = model.get("dropout_p", 0.1)
            widths = model["widths"]
            masks = [torch.tensor([[O.dropout_keep(seed, step, s, l, b, j, p) / (1.0 - p)
                                    for j in range(widths[l + 1])] for b in range(B)], dtype=torch.float64)
                     for l in range(len(widths) - 2)]
        z = _forward(model, ws, Xs, act, masks)
        if agg == "mean":
            zs.append(z)
            continue
        if model["loss"] == "ce":
            l = F.cross_entropy(z, torch.tensor(np.asarray(y_cls, np.int64)), reduction="mean")
        else:
            l = F.mse_loss(z, torch.tensor(np.asarray(y_reg, np.float64)), reduction="mean")
        L_data = L_data + l / S
    if agg == "mean":
        Z = torch.stack(zs)
        if model["loss"] == "ce":
            pbar = torch.softmax(Z, dim=-1).mean(0)
            yt = torch.tensor(np.asarray(y_cls, np.int64))
            # log of the true-class column only (another class's P̄ may underflow to 0)
            L_data = -torch.log(pbar.gather(1, yt[:, None])).mean()
        elif model["loss"] == "gnll":
            # Gaussian NLL of the predictive distribution: mean and population variance over
            # samples, variance floor 1e-6 (reading R24); torch's own moments + autograd
            yt = torch.tensor(np.asarray(y_reg, np.float64))
            m = Z.mean(0)
            v = Z.var(0, unbiased=False) + 1e-6
            L_data = (0.5 * torch.log(2.0 * torch.pi * v) + (yt - m) ** 2 / (2.0 * v)).mean()
        else:
            L_data = F.mse_loss(Z.mean(0), torch.tensor(np.asarray(y_reg, np.float64)))
    kl = 0.5 * torch.sum(sigma ** 2 + mu_t ** 2 - 1.0 - torch.log(sigma ** 2))
    if mcd:  # no variational distribution, no prior term
        kl = torch.zeros((), dtype=torch.float64)
    loss = L_data + kl / D
    loss.backward()
    return dict(loss=loss.item(), L_data=float(L_data.detach()), kl=kl.item(),
                grad_mu=mu_t.grad.numpy().copy(),
                grad_rho=(rho_t.grad.numpy().copy() if rho_t.grad is not None else np.zeros(rho_t.shape)))


def deterministic(model, mu, x, y_cls, y_reg):
    """σ = 0 exactly: the plain network with weights μ; returns (data loss, d loss / d μ)."""
    lay = layout(model)
    mu_t = torch.tensor(np.asarray(mu, np.float64), requires_grad=True)
    ws = [mu_t[t["offset"]:t["offset"] + t["rows"] * t["cols"]].reshape(t["rows"], t["cols"])
          for t in lay]
    z = _forward(model, ws, torch.tensor(np.asarray(x, np.float64)), "relu")
    if model["loss"] == "ce":
        l = F.cross_entropy(z, torch.tensor(np.asarray(y_cls, np.int64)))
    else:
        l = F.mse_loss(z, torch.tensor(np.asarray(y_reg, np.float64)))
    l.backward()
    return l.item(), mu_t.grad.numpy().copy()


# ---------------------------------------------------------------- Bayesian ViT
def vit_forward(model, ws, x):
    """Library-routine formulation of the ViT of oracle/vit_oracle.c (pre-norm encoder,
    F.layer_norm eps 1e-6, exact-erf F.gelu, softmax attention); x: [B, H, W, C]."""
    p, D, nh = model["patch"], model["dim"], model["heads"]
    B, H, W, C = x.shape
    dh = D // nh
    pt = x.reshape(B, H // p, p, W // p, p, C).permute(0, 1, 3, 2, 4, 5).reshape(B, -1, p * p * C)
    T = pt.shape[1] + 1
    it = iter(ws)
    Wp, bp, cls, pos = next(it), next(it), next(it), next(it)
    X = torch.cat([cls.reshape(1, 1, D).expand(B, 1, D), F.linear(pt, Wp, bp.reshape(-1))], 1)
    X = X + pos.reshape(1, T, D)
    for _ in range(model["depth"]):
        g1, b1, Wq, bq, Wo, bo, g2, b2, W1, c1, W2, c2 = [next(it) for _ in range(12)]
        h = F.layer_norm(X, (D,), g1.reshape(-1), b1.reshape(-1), eps=1e-6)
        q, k, v = F.linear(h, Wq, bq.reshape(-1)).split(D, dim=-1)
        q, k, v = (t.reshape(B, T, nh, dh).transpose(1, 2) for t in (q, k, v))
        att = torch.softmax(q @ k.transpose(-1, -2) / dh ** 0.5, dim=-1)
        o = (att @ v).transpose(1, 2).reshape(B, T, D)
        X = X + F.linear(o, Wo, bo.reshape(-1))
        h2 = F.layer_norm(X, (D,), g2.reshape(-1), b2.reshape(-1), eps=1e-6)
        X = X + F.linear(F.gelu(F.linear(h2, W1, c1.reshape(-1))), W2, c2.reshape(-1))
    gf, bf, Wh, bh = next(it), next(it), next(it), next(it)
    hf = F.layer_norm(X, (D,), gf.reshape(-1), bf.reshape(-1), eps=1e-6)
    return F.linear(hf[:, 0], Wh, bh.reshape(-1))


def vit_acc(model, mu, rho, x, y, S, seed, step, aug=False, s0=0):
    """[acc_μ | acc_ρ | L_data] of the ViT data term over global samples s0 … s0+S−1 (scale
    1/(S·B) as in the oracle) by torch autograd with the oracle's ε and crop/flip draws."""
    lay = layout(model)
    B = x.shape[0]
    mu = torch.tensor(np.asarray(mu, np.float64))
    sig = F.softplus(torch.tensor(np.asarray(rho, np.float64)))
    xt = torch.tensor(np.asarray(x, np.float64))
    P = mu.numel()
    am, ar, ld = torch.zeros(P, dtype=torch.float64), torch.zeros(P, dtype=torch.float64), 0.0
    for s in range(s0, s0 + S):
        eps = torch.cat([torch.tensor(O.eps_fill(seed, step, s, ti["t"], 0, ti["rows"], 0, ti["cols"]).astype(np.float64))
                         .reshape(-1) for ti in lay])
        w = (mu + sig * eps).clone().requires_grad_(True)
        ws = [w[ti["offset"]:ti["offset"] + ti["rows"] * ti["cols"]].reshape(ti["rows"], ti["cols"]) for ti in lay]
        xs = torch.stack([_augment(xt[b], seed, step, s, b) for b in range(B)]) if aug else xt
        z = vit_forward(model, ws, xs)
        loss = F.cross_entropy(z, torch.tensor(np.asarray(y, np.int64)), reduction="sum") / (S * B)
        loss.backward()
        am += w.grad
        ar += eps * w.grad
        ld += float(loss.detach())
    return np.concatenate([am.numpy(), ar.numpy(), [ld]])
