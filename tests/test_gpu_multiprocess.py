"""Real processes, one GPU: the N > 1 composition of libbnn itself.

Each of `world` OS processes owns one rank of a K×G grid (sample group k = r / G, data group
g = r % G), runs its shard through the library (`bnn_elbo_partial`, the shard computation
without a communicator), and the ranks exchange their acc buffers with a torch.distributed
SUM-allreduce (gloo, on host copies) before `bnn_finalize`. The result must equal the
single-process step within 1e-5 relative (north_star), for the MLP, the CNN and the ViT.
The tests of tests/test_multiprocess_gloo.py compose the oracle; these compose the CUDA
library across processes (the NCCL communicator itself needs one GPU per rank and is
covered at world 1 by test_gpu_parity.py).
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_04736_b200 import synth

pytestmark = pytest.mark.gpu

RAGGED = dict(kind="mlp", widths=[100, 200, 130, 10], loss="ce")
SMALL_CNN = dict(kind="resnet18", in_h=16, in_w=16, in_c=3, n_classes=10, base_width=64, loss="ce")
VIT_TINY = dict(kind="vit", in_h=8, in_w=8, in_c=3, patch=4, dim=32, heads=2, depth=2, mlp=64, n_classes=3,
                loss="ce")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(model, B, S, precision):
    mu, rho = synth.init_params(model, seed=3, rho_mode="wide")
    x, yc, _ = synth.make_batch(model, B, seed=4)
    return mu, rho, x, yc


def _worker(rank, world, K, G, port, model, B, S, precision, aug, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_04736_b200 import native
    mu, rho, x, yc = _case(model, B, S, precision)
    g = rank % G
    sl = slice(g * (B // G), (g + 1) * (B // G))
    mode = "sample" if G == 1 else ("data" if K == 1 else "hybrid")
    ctx = native.Context(model, precision=precision, mode=mode, K=K, G=G, rank=rank,
                         world=world, max_B_loc=B // G, max_S_loc=S // K, dataset_size=500.0, aug=aug)
    mu_d, rho_d = torch.from_numpy(mu).cuda(), torch.from_numpy(rho).cuda()
    acc = ctx.elbo_partial(mu_d, rho_d, torch.from_numpy(np.ascontiguousarray(x[sl])).cuda(),
                           torch.from_numpy(np.ascontiguousarray(yc[sl])).cuda(), B, S, 77, 9)
    host = acc.cpu()
    dist.all_reduce(host, op=dist.ReduceOp.SUM)
    loss, gm, gr = ctx.finalize(mu_d, rho_d, host.cuda())
    torch.cuda.synchronize()
    if rank == 0:
        np.savez(out, loss=np.float64(loss), gm=gm.cpu().numpy(), gr=gr.cpu().numpy())
    ctx.close()
    dist.destroy_process_group()


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name,model,B,S,precision,K,G,aug", [
    ("mlp_fp32_K2", RAGGED, 64, 8, "fp32", 2, 1, "none"),
    ("mlp_bf16_G2", RAGGED, 64, 8, "bf16", 1, 2, "none"),
    ("cnn_bf16_K2_aug", SMALL_CNN, 16, 4, "bf16", 2, 1, "per_sample"),
    ("cnn_bf16_2x2", SMALL_CNN, 16, 4, "bf16", 2, 2, "per_sample"),
    ("vit_fp32_K2_aug", VIT_TINY, 6, 4, "fp32", 2, 1, "per_sample"),
])
def test_processes_compose_to_the_single_process_step(name, model, B, S, precision, K, G, aug):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2604_04736_b200 import native
    mu, rho, x, yc = _case(model, B, S, precision)
    single = native.Context(model, precision=precision, max_B_loc=B, max_S_loc=S, dataset_size=500.0, aug=aug)
    mu_d, rho_d = torch.from_numpy(mu).cuda(), torch.from_numpy(rho).cuda()
    l1, g1, r1 = single.elbo_step(mu_d, rho_d, torch.from_numpy(x).cuda(), torch.from_numpy(yc).cuda(), B, S, 77, 9)
    g1, r1, l1 = g1.cpu().numpy(), r1.cpu().numpy(), float(l1)
    single.close()
    world = K * G
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "rank0.npz")
        mp.start_processes(_worker, args=(world, K, G, _free_port(), model, B, S, precision, aug, out), nprocs=world,
                           join=True, start_method="spawn")
        r = np.load(out)
        tol = 1e-5  # north_star: sharded vs single within 1e-5 relative
        assert _rel(r["gm"], g1) < tol, name
        assert _rel(r["gr"], r1) < tol, name
        assert abs(float(r["loss"]) - l1) <= tol * abs(l1), name
