"""Host logic of the multi-GPU path (paper_1807_11824_b200.sharded) on CPU:
world_size 2 over gloo, with the per-rank compute supplied by the fp64 oracle
(the GPU kernels need a GPU).  Checks the shard ranges, the exchange order
(partial Z summed in rank order, Y shards gathered into place) and the
recentring schedule against the unsharded iteration."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_1807_11824_b200.sharded import ShardedOptimizer, local_csr, shard_range


class Cfg:
    exag_iters, mom0, mom1, min_gain = 250, 0.5, 0.8, 0.01


class OracleShardOps:
    """Per-rank compute from the oracle (fp64 inside, fp32 state like the GPU),
    with the C ABI's contract: forces leaves Y untouched and records the
    recentring shift; update applies it to the owned rows."""

    def __init__(self, rp, col, val):
        self.rp, self.col, self.val = rp, col, val
        self.shift = np.zeros(2, np.float32)

    def forces(self, Y, N, row0, row1, theta, recentre, rep_local, zpart):
        import oracle
        self.shift = (Y.double().mean(0).float().numpy() if recentre
                      else np.zeros(2, np.float32))
        Ys = (Y - torch.as_tensor(self.shift)).numpy()
        f, z, _, _ = oracle.repulsive_bh(Ys, theta, pts=np.arange(row0, row1))
        rep_local[: row1 - row0] = torch.as_tensor(f, dtype=torch.float32)
        zpart[0] = float(z.sum())

    def attract(self, rp, col, val, N, row0, row1, Y, A_local):
        import oracle
        A = oracle.attractive(self.rp, self.col, self.val, Y.numpy())[row0:row1]
        A_local[: row1 - row0] = torch.as_tensor(A, dtype=torch.float32)

    def update(self, A_local, N, row0, row1, Y, rep, zparts, world, t, lr, exag, cfg, v, g, Yout):
        Z = 0.0
        for r in range(world):
            Z += float(zparts[2 * r])
        alpha = exag if t < cfg.exag_iters else 1.0
        mu = cfg.mom0 if t < cfg.exag_iters else cfg.mom1
        n = row1 - row0
        gr = 4.0 * (alpha * A_local[:n].double().numpy() - rep[:n].double().numpy() / Z)
        vv = v[:n].double().numpy()
        gg = g[:n].double().numpy()
        gg = np.where(np.sign(gr) != np.sign(vv), gg + 0.2, gg * 0.8)
        gg = np.maximum(gg, cfg.min_gain)
        vv = mu * vv - lr * gg * gr
        y = (Y[row0:row1] - torch.as_tensor(self.shift)).double().numpy() + vv
        v[:n] = torch.as_tensor(vv, dtype=torch.float32)
        g[:n] = torch.as_tensor(gg, dtype=torch.float32)
        Yout[:n] = torch.as_tensor(y, dtype=torch.float32)

    def recentre(self, Y, N):
        m = Y.double().mean(0).float()
        Y -= m


def problem(N=300):
    import oracle
    X = synth.make_x("C1", n=N).numpy()
    idx, d2 = oracle.knn(X, 45)
    rp, col, v64, v32, *_ = oracle.compute_p(idx, d2, 15.0)
    Y0 = oracle.init_y(N, 42).astype(np.float32) * 1e3
    return rp, col, v32, Y0


def _worker(rank, world, port, n_iter, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rp, col, val, Y0 = problem()
    N = Y0.shape[0]
    r0, r1, S = shard_range(N, world, rank)
    rpl, cl, vl = local_csr(torch.as_tensor(rp), torch.as_tensor(col), torch.as_tensor(val), r0, r1)
    opt = ShardedOptimizer(rpl, cl, vl, torch.as_tensor(Y0), theta=0.5,
                           ops=OracleShardOps(rp, col, val), cfg=Cfg())
    opt.step(n_iter)
    Y = opt.embedding().clone()
    if rank == 0:
        torch.save(Y, out)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_ranges_cover_points():
    for N in (2, 7, 1000, 1281167):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                a, b, S = shard_range(N, world, r)
                assert b - a <= S and S * world >= N
                seen.extend(range(a, b)) if N < 5000 else seen.append((a, b))
            if N < 5000:
                assert seen == list(range(N))


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_equals_unsharded(tmp_path, world):
    n_iter = 6
    out = str(tmp_path / "y.pt")
    mp.spawn(_worker, args=(world, _free_port(), n_iter, out), nprocs=world, join=True)
    Ys = torch.load(out).double().numpy()
    # the same iterations without sharding (one rank owning every row)
    rp, col, val, Y0 = problem()
    N = Y0.shape[0]
    ops = OracleShardOps(rp, col, val)
    Y = torch.as_tensor(Y0).clone()
    v = torch.zeros(N, 2)
    g = torch.ones(N, 2)
    rep = torch.zeros(N, 2)
    A = torch.zeros(N, 2)
    zp = torch.zeros(2, dtype=torch.float64)
    Yn = torch.zeros(N, 2)
    for t in range(n_iter):
        ops.attract(None, None, None, N, 0, N, Y, A)
        ops.forces(Y, N, 0, N, 0.5, t > 0, rep, zp)
        ops.update(A, N, 0, N, Y, rep, zp, 1, t, 200.0, 12.0, Cfg(), v, g, Yn)
        Y = Yn.clone()
    ops.recentre(Y, N)
    Y1 = Y.double().numpy()
    assert np.linalg.norm(Ys - Y1) / np.linalg.norm(Y1) < 1e-5
    # and against the oracle's own optimiser (fp64 state)
    import oracle
    Yo, _, _ = oracle.optimize(rp, col, val, Y0.astype(np.float64), n_iter=n_iter, theta=0.5)
    assert np.linalg.norm(Ys - Yo) / np.linalg.norm(Yo) < 1e-4


class FakeLib:
    """Records the arguments sharded.run passes to tsne_run_sharded (the GPU
    call itself needs a GPU) and writes a recognisable Y on rank 0."""

    def __init__(self):
        self.calls = []

    def tsne_run_sharded(self, X, n_local, N, D, perp, theta, lr, n_iter, exag, cfg, idbuf,
                         rank, world, Y, info):
        self.calls.append(dict(n_local=n_local, N=N, D=D, n_iter=n_iter, rank=rank, world=world,
                               uid=bytes(idbuf), K=cfg._obj.K, X=X.value, Y=Y.value))
        return 0


def _run_worker(rank, world, port, out):
    import ctypes

    from paper_1807_11824_b200 import sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fake = FakeLib()
    # rank 0's id: a stand-in for tsne_nccl_unique_id (which needs libnccl); the
    # broadcast over the process group is the logic under test
    import paper_1807_11824_b200 as T
    real = T.lib

    class WithFakeId:           # the real library (config defaults) with a stand-in id maker
        def __getattr__(self, name):
            return getattr(real(), name)

        @staticmethod
        def tsne_nccl_unique_id(buf):
            ctypes.memmove(buf, bytes(range(7, 135)), 128)
            return 0

    T.lib = WithFakeId
    try:
        X = synth.make_x("C1", n=301)
        N = X.shape[0]
        r0, r1, _ = shard_range(N, world, rank)
        Y, info = sharded.run(X[r0:r1].clone(), N, perplexity=15.0, n_iter=3, K=45,
                              device=torch.device("cpu"), _lib=fake)
    finally:
        T.lib = real
    torch.save((fake.calls, Y is not None, r0, r1), out + f".{rank}")
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_sharded_run_marshalling(tmp_path):
    """sharded.run on 3 ranks: every rank passes its own shard (N_local =
    its shard_range size), the same id (made on rank 0, broadcast), the same
    N, D, K and n_iter; only rank 0 gets an output buffer."""
    out = str(tmp_path / "run")
    mp.spawn(_run_worker, args=(3, _free_port(), out), nprocs=3, join=True)
    uids = set()
    for r in range(3):
        calls, has_y, r0, r1 = torch.load(out + f".{r}", weights_only=False)
        assert len(calls) == 1
        c = calls[0]
        assert c["rank"] == r and c["world"] == 3 and c["N"] == 301 and c["D"] == 50
        assert c["n_local"] == r1 - r0 and c["K"] == 45 and c["n_iter"] == 3
        assert (c["Y"] is not None) == (r == 0) and has_y == (r == 0)
        uids.add(c["uid"])
    assert uids == {bytes(range(7, 135))}
