"""Per-tensor comparison of the BF16 CNN path against the FP32 path and the oracle."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
from paper_2604_04736_b200 import native, synth

model = dict(kind="resnet18", in_h=8, in_w=8, in_c=3, n_classes=10, base_width=64, loss="ce")
B, S, D = 4, 2, 100.0
mu, rho = synth.init_params(model, seed=2)
x, yc, _ = synth.make_batch(model, B, seed=1)
res = {}
for prec in ("fp32", "bf16"):
    ctx = native.Context(model, precision=prec, max_B_loc=B, max_S_loc=S, dataset_size=D, aug="none")
    loss, gm, gr = ctx.elbo_step(torch.from_numpy(mu).cuda(), torch.from_numpy(rho).cuda(),
                                 torch.from_numpy(x).cuda(), torch.from_numpy(yc).cuda(), B, S, 7, 1)
    torch.cuda.synchronize()
    res[prec] = (loss, gm.cpu().numpy().astype(np.float64) - mu / D, gr.cpu().numpy().astype(np.float64))
    tensors = ctx.tensors
ref = O.elbo_step(model, mu, rho, x, yc, None, S, 7, 1, D)
print("loss", res["fp32"][0], res["bf16"][0], ref["loss"])
rm = ref["grad_mu"] - mu / D
for t in tensors:
    sl = slice(t["offset"], t["offset"] + t["rows"] * t["cols"])
    def rel(a, b):
        return np.linalg.norm(a[sl] - b[sl]) / max(np.linalg.norm(b[sl]), 1e-30)
    print(f"t={t['t']:3d} {t['rows']:4d}x{t['cols']:5d}  fp32-vs-oracle {rel(res['fp32'][1], rm):.2e}  "
          f"bf16-vs-oracle {rel(res['bf16'][1], rm):.2e}  |ref| {np.linalg.norm(rm[sl]):.3e} "
          f"|bf16| {np.linalg.norm(res['bf16'][1][sl]):.3e}  ratio_sample {res['bf16'][1][sl][:3]} {rm[sl][:3]}")
