"""One small step of each BF16 / FP32 path for compute-sanitizer (scripts/gpu_sanitize.sh):
the MLP (gen_gemm fwd/dgrad, wgrad_tc, loss/bias/finalize kernels), the ResNet (conv2/conv3
tcgen05 kernels, W_s generation, wgrad + ε combine, GAP), predict and MC dropout."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_04736_b200 import native, synth  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"


def run(model, precision, B, S, aug="none", **kw):
    mu, rho = synth.init_params(model, seed=2)
    x, yc, yr = synth.make_batch(model, B, seed=1)
    ctx = native.Context(model, precision=precision, max_B_loc=B, max_S_loc=S, dataset_size=100.0, aug=aug, **kw)
    y = torch.from_numpy(yc if yc is not None else yr).cuda()
    loss, g, r = ctx.elbo_step(torch.from_numpy(mu).cuda(), torch.from_numpy(rho).cuda(),
                               torch.from_numpy(x).cuda(), y, B, S, 7, 1)
    m, v = ctx.predict(torch.from_numpy(mu).cuda(), torch.from_numpy(rho).cuda(), torch.from_numpy(x).cuda(),
                       S, 7, 1)
    torch.cuda.synchronize()
    print(model.get("kind"), precision, "loss", loss, "finite", bool(np.isfinite(g.cpu().numpy()).all()), flush=True)
    ctx.close()


if which in ("mlp", "all"):
    run(dict(kind="mlp", widths=[784, 1024, 1024, 10], loss="ce"), "bf16", 64, 4)
    run(dict(kind="mlp", widths=[100, 200, 130, 10], loss="ce"), "fp32", 33, 3)
    run(dict(kind="mlp", widths=[96, 128, 128, 24], loss="mse", method="mcd", dropout_p=0.1), "bf16", 32, 2)
if which in ("cnn", "all"):
    run(dict(kind="resnet18", in_h=16, in_w=16, in_c=3, n_classes=10, base_width=64, loss="ce"), "bf16", 2, 2,
        aug="per_sample")
