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


class OracleRunOps(OracleShardOps):
    """OracleShardOps plus the supporting stages of sharded.run (kNN of a query
    range, P, Y0); the CSR of the iterations is the one compute_p returned."""

    def __init__(self):
        super().__init__(None, None, None)

    def knn_rows(self, X, K, q0, q1):
        import oracle
        idx, d2 = oracle.knn(X.numpy(), K, rows=np.arange(q0, q1))
        return torch.as_tensor(idx, dtype=torch.int32), torch.as_tensor(d2), 0

    def compute_p(self, idx, d2, perplexity):
        import oracle
        rp, col, v64, v32, *_ = oracle.compute_p(idx.numpy(), d2.numpy(), perplexity)
        self.rp, self.col, self.val = rp, col, v32
        return torch.as_tensor(rp), torch.as_tensor(col), torch.as_tensor(v32)

    def init_y(self, N, seed, device):
        import oracle
        return torch.as_tensor(oracle.init_y(N, seed).astype(np.float32) * 1e3)


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


def _run_worker(rank, world, port, n_iter, out):
    from paper_1807_11824_b200 import sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X = synth.make_x("C1", n=300)
    N = X.shape[0]
    r0, r1, _ = shard_range(N, world, rank)
    Y, info = sharded.run(X[r0:r1].clone(), N, perplexity=15.0, theta=0.5, n_iter=n_iter, K=45,
                          device=torch.device("cpu"), ops=OracleRunOps(), cfg=Cfg())
    if rank == 0:
        torch.save((Y.clone(), info), out)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_sharded_run_end_to_end(tmp_path):
    """sharded.run (X shards gathered, kNN by query range, kNN lists gathered,
    P, sharded iterations) equals the unsharded pipeline."""
    n_iter = 4
    out = str(tmp_path / "run.pt")
    mp.spawn(_run_worker, args=(3, _free_port(), n_iter, out), nprocs=3, join=True)
    Ys, info = torch.load(out)
    assert info["N"] == 300 and info["K"] == 45
    import oracle
    rp, col, val, Y0 = problem()
    assert info["nnz"] == len(col)
    Yo, _, _ = oracle.optimize(rp, col, val, Y0.astype(np.float64), n_iter=n_iter, theta=0.5)
    Ys = Ys.double().numpy()
    assert np.linalg.norm(Ys - Yo) / np.linalg.norm(Yo) < 1e-4
