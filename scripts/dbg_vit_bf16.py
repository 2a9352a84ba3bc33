"""Per-tensor error profile of the BF16 ViT against the exact oracle (tiny and paper size)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
from paper_2604_04736_b200 import native, synth
from paper_2604_04736_b200.configs import MODELS

for name, model, B, S in (("tiny", dict(kind="vit", in_h=8, in_w=8, in_c=3, patch=4, dim=32, heads=2, depth=2, mlp=64,
                                         n_classes=3, loss="ce"), 6, 3), ("paper", MODELS["vit_cifar"], 3, 2)):
    mu, rho = synth.init_params(model, seed=2)
    x, yc, _ = synth.make_batch(model, B, seed=1)
    ra = O.vit_elbo_partial(model, mu, rho, x, yc, B, 0, S, 0, S, 0x5EED, 3, O.AUG_PER_SAMPLE,
                            emu="weights" if "--emu" in sys.argv else False)
    for prec in ("fp32", "bf16"):
        ctx = native.Context(model, precision=prec, max_B_loc=B, max_S_loc=S, dataset_size=45000.0, aug="per_sample")
        acc = ctx.elbo_partial(torch.from_numpy(mu).cuda(), torch.from_numpy(rho).cuda(), torch.from_numpy(x).cuda(),
                               torch.from_numpy(yc).cuda(), B, S, 0x5EED, 3).cpu().numpy().astype(np.float64)
        P = ctx.n_params
        rows = []
        for t in ctx.tensors:
            sl = slice(t["offset"], t["offset"] + t["rows"] * t["cols"])
            for k, (g, r) in enumerate(((acc[:P][sl], ra[:P][sl]), (acc[ctx.acc_rho_offset:ctx.acc_rho_offset + P][sl], ra[P:2 * P][sl]))):
                d = np.abs(g - r)
                rows.append((d.max() / np.abs(r).max(), np.linalg.norm(d) / np.linalg.norm(r), t["t"], "mu" if k == 0 else "rho"))
        rows.sort(reverse=True)
        print(name, prec, "L_data", acc[ctx.acc_loss_offset], ra[-1])
        for r in rows[:8]:
            print(f"   t={r[2]:3d} {r[3]:3s} elem {r[0]:.4f} l2 {r[1]:.4f}")
