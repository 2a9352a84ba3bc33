import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import oracle as O
from paper_2604_04736_b200 import native, synth
M = dict(kind="mlp", widths=[96, 128, 128, 24], loss="mse", method="mcd", dropout_p=0.1)
B, S, D = 64, 4, 1000.0
mu, rho = synth.init_params(M, seed=2, rho_mode="init"); x, _, yr = synth.make_batch(M, B, seed=1)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
for prec in ("bf16",):
    ctx = native.Context(M, precision=prec, max_B_loc=B, max_S_loc=S, dataset_size=D)
    l, g, r = ctx.elbo_step(d(mu), d(rho), d(x), d(yr), B, S, 0xD0, 2)
    g = g.cpu().numpy()
    for emu in (False, True):
        ref = O.elbo_step(M, mu, rho, x, None, yr, S, 0xD0, 2, D, emu=emu)
        errs = []
        for t in ctx.tensors:
            sl = slice(t["offset"], t["offset"] + t["rows"] * t["cols"])
            errs.append(round(float(np.linalg.norm(g[sl] - ref["grad_mu"][sl]) / np.linalg.norm(ref["grad_mu"][sl])), 5))
        print(prec, "emu" if emu else "exact", l, ref["loss"], errs)
# VI (same net, no dropout) for comparison
V = dict(M); V.pop("method"); V.pop("dropout_p")
ctx = native.Context(V, precision="bf16", max_B_loc=B, max_S_loc=S, dataset_size=D)
l, g, r = ctx.elbo_step(d(mu), d(rho), d(x), d(yr), B, S, 0xD0, 2)
g = g.cpu().numpy()
ref = O.elbo_step(V, mu, rho, x, None, yr, S, 0xD0, 2, D)
print("VI bf16 exact", [round(float(np.linalg.norm(g[t["offset"]:t["offset"]+t["rows"]*t["cols"]] - ref["grad_mu"][t["offset"]:t["offset"]+t["rows"]*t["cols"]]) / np.linalg.norm(ref["grad_mu"][t["offset"]:t["offset"]+t["rows"]*t["cols"]])), 5) for t in ctx.tensors])
