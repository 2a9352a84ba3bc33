"""The N>1 host path on CPU: world-size-2 (and 4) process groups over gloo.

Each rank computes the oracle's partial ELBO sums for its K×G shard (paper_2604_04736_b200.plan),
the partials are SUM-allreduced over the process group (the one exchange of Alg. 2,
PAPER.md:263), and the finalized loss/gradients must equal the single-process oracle —
the same composition the CUDA path performs with NCCL.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_04736_b200 import plan, synth

MODEL = dict(kind="mlp", widths=[6, 9, 4], loss="ce")
CNN = dict(kind="resnet18", in_h=8, in_w=8, in_c=3, n_classes=10, base_width=2, loss="ce")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, K, G, model, S, B, aug, out):
    import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank 0 creates the "communicator id" and broadcasts it (bnn_get_unique_id analogue)
    obj = [os.urandom(128) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    uid = obj[0]
    K, G = plan.grid(mode, world, K, G)
    sh = plan.shard(rank, K, G, S, B)
    mu, rho = synth.init_params(model, seed=3, rho_mode="wide")
    x, yc, yr = synth.make_batch(model, B, seed=4)
    xs = x[sh["b0"]:sh["b1"]]
    ys = None if yc is None else yc[sh["b0"]:sh["b1"]]
    yrs = None if yr is None else yr[sh["b0"]:sh["b1"]]
    acc = O.elbo_partial(model, mu, rho, xs, ys, yrs, B, sh["b0"], S, sh["s0"], sh["s1"], 9, 2,
                         O.AUG_PER_SAMPLE if aug else O.AUG_NONE, nthreads=1)
    t = torch.from_numpy(acc)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    r = O.finalize(model, mu, rho, t.numpy(), 500.0)
    out[rank] = (r["loss"], r["grad_mu"], r["grad_rho"], uid)
    dist.destroy_process_group()


def _run(world, mode, K=None, G=None, model=MODEL, S=8, B=8, aug=False):
    import oracle as O
    O.lib()  # build before spawning
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), mode, K, G, model, S, B, aug, out), nprocs=world,
             join=True)
    mu, rho = synth.init_params(model, seed=3, rho_mode="wide")
    x, yc, yr = synth.make_batch(model, B, seed=4)
    ref = O.elbo_step(model, mu, rho, x, yc, yr, S, 9, 2, 500.0,
                      aug=O.AUG_PER_SAMPLE if aug else O.AUG_NONE, nthreads=1)
    uids = {out[r][3] for r in range(world)}
    assert len(uids) == 1  # every rank received rank 0's id
    for r in range(world):
        loss, gmu, grho, _ = out[r]
        assert loss == pytest.approx(ref["loss"], rel=1e-12)
        np.testing.assert_allclose(gmu, ref["grad_mu"], rtol=1e-10, atol=1e-14)
        np.testing.assert_allclose(grho, ref["grad_rho"], rtol=1e-10, atol=1e-14)


def test_plan_shards_partition_samples_and_examples():
    for K, G in [(1, 1), (4, 1), (1, 4), (4, 2), (2, 4)]:
        S, B = 32, 256
        seen = np.zeros((S, B), int)
        for r in range(K * G):
            sh = plan.shard(r, K, G, S, B)
            seen[sh["s0"]:sh["s1"], sh["b0"]:sh["b1"]] += 1
        assert np.all(seen == 1)
    with pytest.raises(ValueError):
        plan.shard(0, 3, 1, 8, 8)  # S mod K != 0
    with pytest.raises(ValueError):
        plan.grid("hybrid", 8, 3, 2)


def test_gloo_world2_sample_sharded():
    _run(2, "sample")


def test_gloo_world2_data_sharded():
    _run(2, "data")


def test_gloo_world4_hybrid_with_augmentation():
    _run(4, "hybrid", K=2, G=2, model=CNN, S=4, B=4, aug=True)


def test_gloo_world4_hybrid_mc_dropout():
    """MC dropout (f4): masks keyed by global sample and global example, so the 2×2 grid's
    allreduced partials equal the single process."""
    _run(4, "hybrid", K=2, G=2, model=dict(kind="mlp", widths=[6, 9, 4], loss="mse", method="mcd",
                                            dropout_p=0.25))


# ---------------------------------------------------------------- exact aggregation (f1), two collectives
def _worker_mean(rank, world, port, mode, K, G, model, S, B, aug, out):
    """the statistic of the mean prediction is exchanged between forward and
    backward (allgather + rank-ordered sum over the sample groups of this rank's data group,
    as bnn_elbo_step does over NCCL), then the gradient partials are SUM-allreduced."""
    import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    K, G = plan.grid(mode, world, K, G)
    sh = plan.shard(rank, K, G, S, B)
    k, g = rank // G, rank % G
    mu, rho = synth.init_params(model, seed=3, rho_mode="init")
    x, yc, yr = synth.make_batch(model, B, seed=4)
    sl = slice(sh["b0"], sh["b1"])
    a = O.AUG_PER_SAMPLE if aug else O.AUG_NONE
    st = torch.from_numpy(O.mean_stats(model, mu, rho, x[sl], None if yc is None else yc[sl], sh["b0"],
                                       sh["s0"], sh["s1"], 9, 2, a))
    allst = [torch.zeros_like(st) for _ in range(world)]
    dist.all_gather(allst, st)
    gst = None
    for r in range(g, world, G):
        gst = allst[r].clone() if gst is None else gst + allst[r]
    acc = O.elbo_partial_mean(model, mu, rho, x[sl], None if yc is None else yc[sl],
                              None if yr is None else yr[sl], B, sh["b0"], S, sh["s0"], sh["s1"], 9, 2,
                              gst.numpy(), add_loss=(k == 0), aug=a, nthreads=1)
    t = torch.from_numpy(acc)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    r_ = O.finalize(model, mu, rho, t.numpy(), 500.0)
    out[rank] = (r_["loss"], r_["grad_mu"], r_["grad_rho"])
    dist.destroy_process_group()


@pytest.mark.parametrize("model,world,mode,K,G,aug", [
    (MODEL, 2, "sample", None, None, False),
    (dict(kind="mlp", widths=[5, 7, 3], loss="mse"), 2, "sample", None, None, False),
    (MODEL, 4, "hybrid", 2, 2, False),
    (CNN, 2, "hybrid", 1, 2, True),
])
def test_gloo_mean_aggregation_equals_single_process(model, world, mode, K, G, aug):
    import oracle as O
    O.lib()
    S, B = 8, 8
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_mean, args=(world, _free_port(), mode, K, G, model, S, B, aug, out), nprocs=world,
             join=True)
    mu, rho = synth.init_params(model, seed=3, rho_mode="init")
    x, yc, yr = synth.make_batch(model, B, seed=4)
    ref = O.elbo_step(model, mu, rho, x, yc, yr, S, 9, 2, 500.0,
                      aug=O.AUG_PER_SAMPLE if aug else O.AUG_NONE, nthreads=1, agg="mean")
    for r in range(world):
        loss, gmu, grho = out[r]
        assert loss == pytest.approx(ref["loss"], rel=1e-12)
        np.testing.assert_allclose(gmu, ref["grad_mu"], rtol=1e-9, atol=1e-13)
        np.testing.assert_allclose(grho, ref["grad_rho"], rtol=1e-9, atol=1e-13)
