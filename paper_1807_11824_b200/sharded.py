"""Multi-GPU Barnes-Hut t-SNE iterations: one process per GPU, points sharded
by index range, two NCCL exchanges per iteration (the paper
is single-GPU).

Per iteration, on every rank:
  1. forces   -- quadtree over the full replicated embedding (redundant, small),
                 theta traversal for the owned points, partial Z   [C ABI]
  2. exchange -- all-gather the partial Z of every rank (rank order)  [NCCL]
  3. update   -- attractive pass + Eq. 7 + D12 update of the owned rows [C ABI]
  4. exchange -- all-gather the updated Y shards                      [NCCL]
The host logic (ranges, exchange order, padding) lives here; all arithmetic
runs in the library's kernels (`GpuShardOps`).  The ops object is injectable
so the host logic can be tested on CPU with a gloo process group.
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist


def shard_range(N: int, world: int, rank: int):
    """Rows [row0, row1) owned by `rank`; S = ceil(N / world) is the padded
    shard size used by the all-gather of Y."""
    S = (N + world - 1) // world
    row0 = min(N, rank * S)
    row1 = min(N, row0 + S)
    return row0, row1, S


def local_csr(row_ptr: torch.Tensor, col: torch.Tensor, val: torch.Tensor, row0: int, row1: int):
    """The owned rows of a global CSR, as a self-contained local CSR (fresh,
    aligned allocations)."""
    rp = row_ptr[row0:row1 + 1]
    e0, e1 = int(rp[0]), int(rp[-1])
    return (rp - e0).contiguous().clone(), col[e0:e1].clone(), val[e0:e1].clone()


def _all_gather_flat(out: torch.Tensor, inp: torch.Tensor, group=None):
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp, group=group)
    else:
        world = dist.get_world_size(group)
        parts = list(out.chunk(world))
        dist.all_gather(parts, inp, group=group)


class GpuShardOps:
    """The C-ABI kernels of one rank (tsne_shard_forces / _update / tsne_recentre)."""

    def __init__(self, N: int, device):
        from . import _check, _ptr, _stream, _ws, lib
        self._check, self._ptr, self._stream, self.lib = _check, _ptr, _stream, lib()
        self.ws = _ws(self.lib.tsne_shard_workspace_size(N), device)
        self.flag = torch.zeros(1, dtype=torch.int32, device=device)

    def forces(self, Y, N, row0, row1, theta, recentre, rep_local, zpart):
        P = self._ptr
        self._check(self.lib.tsne_shard_forces(P(Y), N, row0, row1, float(theta), int(recentre),
                                               P(rep_local), P(zpart), P(self.ws), self.ws.numel(),
                                               self._stream()), "tsne_shard_forces")

    def update(self, rp, col, val, N, row0, row1, Y, rep_local, zparts, world, t, lr, exag, cfg,
               v_local, g_local, Y_out):
        P = self._ptr
        self._check(self.lib.tsne_shard_update(P(rp), P(col), P(val), N, row0, row1, P(Y),
                                               P(rep_local), P(zparts), world, int(t), float(lr),
                                               float(exag), C.byref(cfg), P(v_local), P(g_local),
                                               P(Y_out), P(self.flag), self._stream()),
                    "tsne_shard_update")

    def recentre(self, Y, N):
        P = self._ptr
        self._check(self.lib.tsne_recentre(P(Y), N, P(self.ws), self.ws.numel(), self._stream()),
                    "tsne_recentre")

    def nonfinite(self) -> bool:
        return bool(self.flag.item())


class ShardedOptimizer:
    """Owns this rank's rows of P and of the optimiser state; `step(n)` runs
    n iterations with the two exchanges; `embedding()` returns the full
    (recentred) Y on every rank."""

    def __init__(self, row_ptr_local, col_local, val_local, Y0: torch.Tensor, theta=0.5,
                 learning_rate=200.0, exaggeration=12.0, exag_iters=250, mom0=0.5, mom1=0.8,
                 min_gain=0.01, group=None, ops=None, cfg=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        N = Y0.shape[0]
        self.N = N
        self.row0, self.row1, self.S = shard_range(N, self.world, self.rank)
        n_local = self.row1 - self.row0
        dev = Y0.device
        self.rp, self.col, self.val = row_ptr_local, col_local, val_local
        if self.rp.numel() != n_local + 1:
            raise ValueError("row_ptr_local must have n_local + 1 entries")
        self.Yfull = torch.zeros(self.world * self.S, 2, dtype=torch.float32, device=dev)
        self.Yfull[:N] = Y0
        self.Y = self.Yfull[:N]                       # contiguous view
        self.Yloc = torch.zeros(self.S, 2, dtype=torch.float32, device=dev)
        self.v = torch.zeros(max(n_local, 1), 2, dtype=torch.float32, device=dev)
        self.g = torch.ones(max(n_local, 1), 2, dtype=torch.float32, device=dev)
        self.rep = torch.zeros(max(n_local, 1), 2, dtype=torch.float32, device=dev)
        self.zpart = torch.zeros(2, dtype=torch.float64, device=dev)
        self.zparts = torch.zeros(self.world * 2, dtype=torch.float64, device=dev)
        self.ops = ops if ops is not None else GpuShardOps(N, dev)
        if cfg is None:
            from . import default_config
            cfg = default_config(exag_iters=exag_iters, mom0=mom0, mom1=mom1, min_gain=min_gain)
        self.cfg = cfg
        self.theta, self.lr, self.exag = theta, learning_rate, exaggeration
        self.t = 0
        self.pending_recentre = False

    def step(self, n_iter: int = 1):
        for _ in range(n_iter):
            self.ops.forces(self.Y, self.N, self.row0, self.row1, self.theta,
                            self.pending_recentre, self.rep, self.zpart)
            _all_gather_flat(self.zparts, self.zpart, self.group)
            self.ops.update(self.rp, self.col, self.val, self.N, self.row0, self.row1, self.Y,
                            self.rep, self.zparts, self.world, self.t, self.lr, self.exag,
                            self.cfg, self.v, self.g, self.Yloc)
            _all_gather_flat(self.Yfull, self.Yloc, self.group)
            self.t += 1
            self.pending_recentre = True

    def embedding(self) -> torch.Tensor:
        if self.pending_recentre:
            self.ops.recentre(self.Y, self.N)
            self.pending_recentre = False
        return self.Y
