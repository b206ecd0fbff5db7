"""Multi-GPU kernels on one GPU: G 'virtual shards' driven in one process
(the exchanges done by hand in rank order), and a world_size-1 NCCL run of
ShardedOptimizer, against the single-GPU optimiser and the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import paper_1807_11824_b200 as T
    T.lib()
    return T


@pytest.fixture(scope="module")
def prob(orc):
    X = synth.make_x("C1", n=2000).numpy()
    idx, d2 = orc.knn(X, 90)
    rp, col, v64, v32, *_ = orc.compute_p(idx, d2, 30.0)
    return rp, col, v32


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


@pytest.mark.parametrize("G", [1, 3])
def test_virtual_shards_match_single_gpu(T, orc, prob, G):
    from paper_1807_11824_b200.sharded import GpuShardOps, local_csr, shard_range
    rp, col, v32 = prob
    dev = torch.device("cuda")
    N = len(rp) - 1
    Y0 = T.init_y(N, 42)
    rp_d, col_d, val_d = (torch.as_tensor(a, device=dev) for a in (rp, col, v32))
    ops = GpuShardOps(N, dev)
    cfg = T.default_config()
    shards = []
    for r in range(G):
        a, b, S = shard_range(N, G, r)
        shards.append((a, b, *local_csr(rp_d, col_d, val_d, a, b),
                       torch.zeros(b - a, 2, device=dev), torch.ones(b - a, 2, device=dev),
                       torch.zeros(b - a, 2, device=dev), torch.zeros(b - a, 2, device=dev),
                       GpuShardOps(N, dev)))       # one workspace (tree, shift) per rank
    Y = Y0.clone()
    zp = torch.zeros(G * 2, dtype=torch.float64, device=dev)
    n_iter = 3        # trajectories diverge chaotically; compare a few iterations
    Yo = Y0.cpu().numpy().astype(np.float64)
    vo, go = np.zeros_like(Yo), np.ones_like(Yo)
    for t in range(n_iter):
        for r, (a, b, rpl, cl, vl, v, g, rep, A, o) in enumerate(shards):
            o.attract(rpl, cl, vl, N, a, b, Y, A)
            o.forces(Y, N, a, b, 0.5, t > 0, rep, zp[2 * r:2 * r + 2])
        Ynew = torch.empty_like(Y)
        for r, (a, b, rpl, cl, vl, v, g, rep, A, o) in enumerate(shards):
            out = torch.empty(b - a, 2, device=dev)
            o.update(A, N, a, b, Y, rep, zp, G, t, 200.0, 12.0, cfg, v, g, out)
            Ynew[a:b] = out
        Y = Ynew
        # each sharded iteration vs one oracle iteration from the same state
        # (the GPU's Y of the previous iteration, recentred; its v and gains)
        Yo, vo, go = orc.optimize(rp, col, v32, Yo, vo, go, t0=t, n_iter=1, theta=0.5)
        Yc = Y.clone()
        ops.recentre(Yc, N)
        assert rel(Yc.cpu().numpy(), Yo) <= 1e-5, t
        Yo = Yc.cpu().numpy().astype(np.float64)
        vo = torch.cat([sh[5] for sh in shards]).cpu().numpy().astype(np.float64)
        go = torch.cat([sh[6] for sh in shards]).cpu().numpy().astype(np.float64)
    ops.recentre(Y, N)
    assert not ops.nonfinite()
    ref = T.Optimizer(rp_d, col_d, val_d, Y0, theta=0.5, relabel_every=0, use_graphs=False)
    Yref = ref.step(n_iter)
    assert rel(Y.cpu().numpy(), Yref.cpu().numpy().astype(np.float64)) < 1e-4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_world1_sharded_optimizer(T, prob):
    from paper_1807_11824_b200.sharded import ShardedOptimizer, local_csr
    rp, col, v32 = prob
    dev = torch.device("cuda")
    N = len(rp) - 1
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        rp_d, col_d, val_d = (torch.as_tensor(a, device=dev) for a in (rp, col, v32))
        Y0 = T.init_y(N, 7)
        opt = ShardedOptimizer(*local_csr(rp_d, col_d, val_d, 0, N), Y0, theta=0.5)
        opt.step(3)
        Y = opt.embedding()
        ref = T.Optimizer(rp_d, col_d, val_d, Y0, theta=0.5, relabel_every=0, use_graphs=False)
        Yref = ref.step(3)
        assert torch.isfinite(Y).all()
        assert rel(Y.cpu().numpy(), Yref.cpu().numpy().astype(np.float64)) < 1e-4
        # graph-replayed iterations (both schedule phases) == eager, bitwise
        cfg = T.default_config(exag_iters=4)
        a = ShardedOptimizer(*local_csr(rp_d, col_d, val_d, 0, N), Y0, theta=0.5, cfg=cfg)
        b = ShardedOptimizer(*local_csr(rp_d, col_d, val_d, 0, N), Y0, theta=0.5, cfg=cfg,
                             use_graphs=False)
        assert a.use_graphs and not b.use_graphs
        a.step(7)
        b.step(7)
        assert len(a._graphs) == 2
        assert torch.equal(a.embedding(), b.embedding())
    finally:
        dist.destroy_process_group()


def test_nccl_world1_sharded_run_end_to_end(T):
    """sharded.run (X shard H2D + all-gather, tsne_knn_rows, gathered lists, P,
    sharded iterations) against tsne_run_ex on the same pinned host X."""
    from paper_1807_11824_b200 import sharded
    X = synth.make_x("C2", n=3000)
    Xh = torch.empty(X.shape, dtype=torch.float32, pin_memory=True)
    Xh.copy_(X)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        Yh = torch.empty(3000, 2, dtype=torch.float32, pin_memory=True)
        Y, info = sharded.run(Xh, 3000, perplexity=30.0, theta=0.5, n_iter=5, Y_out=Yh,
                              device=torch.device("cuda"))
        torch.cuda.synchronize()
        assert info["K"] == 90 and info["knn_rows_uncertified"] == 0
        Yr, rinfo = T.run(Xh, perplexity=30.0, theta=0.5, n_iter=5, relabel_every=0,
                          use_graphs=False)
        assert rinfo["nnz"] == info["nnz"]
        assert torch.equal(Yh, Y.cpu())
        assert rel(Yh.numpy(), Yr.numpy().astype(np.float64)) < 1e-4
    finally:
        dist.destroy_process_group()


def test_virtual_shards_collapsed_cluster(T, orc):
    # The shard path's repulsive forces (the traversal over a rank's list of
    # owned points, with large deferred buckets walked by k_defer_large into the
    # rank's local numerators and Z partial) on a collapsed cluster: 3 virtual
    # shards assembled into the gradient 4 (alpha A - f / Z) vs the oracle's.
    from paper_1807_11824_b200.sharded import GpuShardOps, local_csr, shard_range
    N, G, exag = 40000, 3, 12.0          # ~120 points per finest cell: large buckets
    Y = synth.fixed_y("collapsed", N, seed=23)
    rp, col, v32, _ = synth.random_csr(N, 8, seed=13)
    dev = torch.device("cuda")
    rp_d, col_d, val_d = (torch.as_tensor(a, device=dev) for a in (rp, col, v32))
    Yd = torch.as_tensor(Y, device=dev)
    zp = torch.zeros(2 * G, dtype=torch.float64, device=dev)
    parts = []
    for r in range(G):
        a, b, _ = shard_range(N, G, r)
        o = GpuShardOps(N, dev)
        rpl, cl, vl = local_csr(rp_d, col_d, val_d, a, b)
        A = torch.zeros(b - a, 2, device=dev)
        rep = torch.zeros(b - a, 2, device=dev)
        o.attract(rpl, cl, vl, N, a, b, Yd, A)
        o.forces(Yd, N, a, b, 0.5, False, rep, zp[2 * r:2 * r + 2])
        parts.append((A, rep))
    torch.cuda.synchronize()
    Z = float(sum(zp[2 * r].item() for r in range(G)))
    g = torch.cat([4.0 * (exag * A.double() - rep.double() / Z) for A, rep in parts]).cpu().numpy()
    go, Zo = orc.gradient_bh(rp, col, v32, Y, 0.5, exag)
    assert abs(Z - Zo) <= 1e-6 * Zo
    assert rel(g, go) <= 1e-4
