"""All (sample, example) gradient buffers + acc partials of the BF16 CNN vs the emulating oracle."""
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
mu_d, rho_d = torch.from_numpy(mu).cuda(), torch.from_numpy(rho).cuda()
acc = ctx.elbo_partial(mu_d, rho_d, torch.from_numpy(x).cuda(), torch.from_numpy(yc).cuda(), B, S, 7, 1)
torch.cuda.synchronize()
acc = acc.cpu().numpy().astype(np.float64)
P = ctx.n_params
a_mu, a_rho, a_L = acc[:P], acc[ctx.acc_rho_offset:ctx.acc_rho_offset + P], acc[ctx.acc_loss_offset]
e = O.elbo_partial(model, mu, rho, x, yc, None, B, 0, S, 0, S, 7, 1, emu=True)
e_mu, e_rho, e_L = e[:P], e[P:2 * P], e[2 * P]
print("L_data gpu", a_L, "emu", e_L)
for t in ctx.tensors:
    sl = slice(t["offset"], t["offset"] + t["rows"] * t["cols"])
    r = lambda a, b: np.linalg.norm(a[sl] - b[sl]) / max(np.linalg.norm(b[sl]), 1e-30)
    print(f"t={t['t']:2d} {t['rows']:4d}x{t['cols']:5d} acc_mu {r(a_mu, e_mu):.2e} acc_rho {r(a_rho, e_rho):.2e} "
          f"|mu| {np.linalg.norm(e_mu[sl]):.3e}")
for l in []:
    gg = ctx.layer_output(l, 1).cpu().numpy().astype(np.float64)
    errs = []
    for s in range(S):
        for b in range(B):
            ge = O.layer_grad(model, mu, rho, x, yc, None, b, s, 7, 1, l, emu=True)
            n = ge.size
            g = gg[(s * B + b) * n:(s * B + b + 1) * n]
            errs.append(np.linalg.norm(g - ge) / max(np.linalg.norm(ge), 1e-30))
    print(f"layer {l:2d} grad per (s,b):", " ".join(f"{v:.1e}" for v in errs))
for l in range(21):
    ga = ctx.layer_output(l, 0).cpu().numpy().astype(np.float64)
    errs = []
    for s in range(S):
        for b in range(B):
            ee = O.layer_output(model, mu, rho, x, b, s, 7, 1, l, emu=True)
            n = ee.size
            g = ga[(s * B + b) * n:(s * B + b + 1) * n]
            errs.append(np.linalg.norm(g - ee) / max(np.linalg.norm(ee), 1e-30))
    print(f"layer {l:2d} act per (s,b):", " ".join(f"{v:.1e}" for v in errs))
