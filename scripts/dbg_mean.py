import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle as O
from paper_2604_04736_b200 import native, synth
m = dict(kind='resnet18', in_h=16, in_w=16, in_c=3, n_classes=10, base_width=8, loss='ce')
D, S, B = 45000.0, 1, 3
mu, rho = synth.init_params(m, seed=2, rho_mode="init"); x, yc, _ = synth.make_batch(m, B, seed=1)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
b = 2
c = native.Context(m, precision="fp32", mode="data", K=1, G=3, rank=b, world=3, max_B_loc=1, max_S_loc=S, dataset_size=D, aug="per_sample")
acc = c.elbo_partial(d(mu), d(rho), d(x[b:b+1]), d(yc[b:b+1]), B, S, 0xBEEF, 5)
for layer in range(20, 10, -1):
    gv = c.layer_output(layer, 0).cpu().numpy().astype(np.float64)
    gg = c.layer_output(layer, 1).cpu().numpy().astype(np.float64)
    ov = O.layer_output(m, mu, rho, x, b, 0, 0xBEEF, 5, layer, aug=O.AUG_PER_SAMPLE)
    og = O.layer_grad(m, mu, rho, x, yc, None, b, 0, 0xBEEF, 5, layer, aug=O.AUG_PER_SAMPLE)
    ev = np.linalg.norm(gv - ov) / np.linalg.norm(ov)
    eg = np.linalg.norm(gg - og) / max(np.linalg.norm(og), 1e-30)
    flips = np.sum((gv > 0) != (ov > 0))
    print(layer, "val rel", ev, "grad rel", eg, "mask flips", flips, "n", gv.size, "tiny", np.sort(np.abs(ov[ov != 0]))[:3] / np.abs(ov).max())
