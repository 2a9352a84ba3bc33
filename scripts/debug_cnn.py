"""Per-tensor comparison of the BF16 CNN path against the emulating and the exact oracle."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
from paper_2604_04736_b200 import native, synth

hw = int(sys.argv[1]) if len(sys.argv) > 1 else 8
model = dict(kind="resnet18", in_h=hw, in_w=hw, in_c=3, n_classes=10, base_width=64, loss="ce")
B, S, D = 4, 2, 100.0
mu, rho = synth.init_params(model, seed=2)
x, yc, _ = synth.make_batch(model, B, seed=1)
ctx = native.Context(model, precision="bf16", max_B_loc=B, max_S_loc=S, dataset_size=D, aug="none")
loss, gm, gr = ctx.elbo_step(torch.from_numpy(mu).cuda(), torch.from_numpy(rho).cuda(),
                             torch.from_numpy(x).cuda(), torch.from_numpy(yc).cuda(), B, S, 7, 1)
torch.cuda.synchronize()
gm = gm.cpu().numpy().astype(np.float64); gr = gr.cpu().numpy().astype(np.float64)
emu = O.elbo_step(model, mu, rho, x, yc, None, S, 7, 1, D, emu=True)
ref = O.elbo_step(model, mu, rho, x, yc, None, S, 7, 1, D)
print("loss gpu", loss, "emu", emu["loss"], "exact", ref["loss"])
for t in ctx.tensors:
    sl = slice(t["offset"], t["offset"] + t["rows"] * t["cols"])
    def rel(a, b):
        return np.linalg.norm(a[sl] - b[sl]) / max(np.linalg.norm(b[sl]), 1e-30)
    print(f"t={t['t']:3d} {t['rows']:4d}x{t['cols']:5d}  mu: vs-emu {rel(gm, emu['grad_mu']):.2e} "
          f"vs-exact {rel(gm, ref['grad_mu']):.2e} emu-vs-exact {rel(emu['grad_mu'], ref['grad_mu']):.2e} | "
          f"rho: vs-emu {rel(gr, emu['grad_rho']):.2e} vs-exact {rel(gr, ref['grad_rho']):.2e}")

# forward only: softmax of the GPU forward (predict, S=1) vs the emulated / exact forward
mean, var = ctx.predict(torch.from_numpy(mu).cuda(), torch.from_numpy(rho).cuda(), torch.from_numpy(x).cuda(), 1, 7, 1)
pg = mean.cpu().numpy()
for emu_flag in (True, False):
    z = O.forward(model, mu, rho, x, 0, 1, 7, 1, emu=emu_flag)[0]
    p = np.exp(z - z.max(-1, keepdims=True)); p /= p.sum(-1, keepdims=True)
    print("forward probs rel err", "emu" if emu_flag else "exact", np.linalg.norm(pg - p) / np.linalg.norm(p))
    print("  logits", z[0][:5])

# per-layer stored activations: GPU vs emulated oracle vs exact oracle (sample 0, example 0)
for t in ctx.tensors[::2]:
    l = t["t"] // 2
    g = ctx.layer_output(l, 0).cpu().numpy().astype(np.float64)
    e = O.layer_output(model, mu, rho, x, 0, 0, 7, 1, l, emu=True)
    r = O.layer_output(model, mu, rho, x, 0, 0, 7, 1, l, emu=False)
    g0 = g[:e.size]
    print(f"layer {l:2d} out {e.size:6d}: gpu-vs-emu {np.linalg.norm(g0-e)/np.linalg.norm(e):.2e} "
          f"gpu-vs-exact {np.linalg.norm(g0-r)/np.linalg.norm(r):.2e} emu-vs-exact {np.linalg.norm(e-r)/np.linalg.norm(r):.2e} "
          f"max|gpu-emu| {np.abs(g0-e).max():.3e} frac!= {(g0 != e).mean():.3f}")

# per-layer gradients (unscaled dl/d out) and sample 1 activations
for t in ctx.tensors[::2]:
    l = t["t"] // 2
    e = O.layer_output(model, mu, rho, x, 0, 1, 7, 1, l, emu=True)
    g = ctx.layer_output(l, 0).cpu().numpy().astype(np.float64)
    n = e.size
    g1 = g[B * n:B * n + n]  # sample 1, example 0
    ge = O.layer_grad(model, mu, rho, x, yc, None, 0, 0, 7, 1, l, emu=True)
    gg = ctx.layer_output(l, 1).cpu().numpy().astype(np.float64)[:n] if l < 20 else None
    msg = f"layer {l:2d}: s1 act gpu-vs-emu {np.linalg.norm(g1-e)/np.linalg.norm(e):.2e}"
    if gg is not None:
        msg += f"  grad gpu-vs-emu {np.linalg.norm(gg-ge)/max(np.linalg.norm(ge),1e-30):.2e} |ge| {np.linalg.norm(ge):.3e} |gg| {np.linalg.norm(gg):.3e}"
    print(msg)
