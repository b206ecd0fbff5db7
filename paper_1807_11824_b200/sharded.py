"""Multi-GPU Barnes-Hut t-SNE iterations: one process per GPU, points sharded
by index range, two NCCL exchanges per iteration (the paper
is single-GPU).

Per iteration, on every rank:
  1. forces   -- quadtree over the full replicated embedding (redundant, small),
                 theta traversal for the owned points, partial Z   [C ABI]
  1'. attract -- attractive sums of the owned rows, on a side stream
                 concurrently with 1 (it only reads Y)              [C ABI]
  2. exchange -- all-gather the partial Z of every rank (rank order)  [NCCL]
  3. update   -- Eq. 7 + D12 update of the owned rows (recentred)    [C ABI]
  4. exchange -- all-gather the updated Y shards                      [NCCL]
The host logic (ranges, exchange order, padding) lives here; all arithmetic
runs in the library's kernels (`GpuShardOps`).  The ops object is injectable
so the host logic can be tested on CPU with a gloo process group.

`run` is the multi-GPU end-to-end call (Algorithm 1): each rank
copies its own rows of X host->device, the rows are all-gathered over NCCL,
each rank finds the neighbours of its own query rows (tsne_knn_rows), the
kNN lists are all-gathered, P is built redundantly on every rank (it is
~50 ms at C5 and needs every row: symmetrisation), and the sharded
iterations run; rank 0 copies the final Y to the host.
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
    else:                       # gloo (CPU tests; CUDA tensors staged through the host)
        world = dist.get_world_size(group)
        if inp.is_cuda:
            host = torch.empty(out.shape, dtype=out.dtype)
            _all_gather_flat(host, inp.cpu(), group)
            out.copy_(host)
            return
        parts = list(out.chunk(world))
        dist.all_gather(parts, inp, group=group)


class GpuShardOps:
    """The C-ABI kernels of one rank (tsne_shard_forces / _update / tsne_recentre,
    and for `run`: tsne_knn_rows, tsne_compute_p, tsne_init_y)."""

    @staticmethod
    def knn_rows(X, K, q0, q1):
        from . import knn
        idx, d2, info = knn(X, K, rows=(q0, q1))
        return idx, d2, info["rows_uncertified"]

    @staticmethod
    def compute_p(idx, d2, perplexity):
        from . import compute_p
        return compute_p(idx, d2, perplexity)

    @staticmethod
    def init_y(N, seed, device):
        from . import init_y
        return init_y(N, seed, device=device)

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

    def attract(self, rp, col, val, N, row0, row1, Y, A_local):
        P = self._ptr
        self._check(self.lib.tsne_shard_attract(P(rp), P(col), P(val), N, row0, row1, P(Y),
                                                P(A_local), self._stream()), "tsne_shard_attract")

    def update(self, A_local, N, row0, row1, Y, rep_local, zparts, world, t, lr, exag, cfg,
               v_local, g_local, Y_out):
        P = self._ptr
        self._check(self.lib.tsne_shard_update(P(A_local), N, row0, row1, P(Y), P(rep_local),
                                               P(zparts), world, int(t), float(lr), float(exag),
                                               C.byref(cfg), P(v_local), P(g_local), P(Y_out),
                                               P(self.flag), P(self.ws), self.ws.numel(),
                                               self._stream()), "tsne_shard_update")

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
                 min_gain=0.01, group=None, ops=None, cfg=None, use_graphs=True):
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
        self.A = torch.zeros(max(n_local, 1), 2, dtype=torch.float32, device=dev)
        self.side = torch.cuda.Stream(device=dev) if dev.type == "cuda" else None
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
        self.exag_iters = int(cfg.exag_iters)
        # CUDA graphs of the steady-state iteration (kernels + both NCCL
        # exchanges), one per schedule phase: t < exag_iters and after (the
        # iteration number only selects alpha and the momentum, D13)
        self.use_graphs = (use_graphs and dev.type == "cuda" and ops is None
                           and dist.get_backend(group) == "nccl")
        self._graphs = {}

    def _iteration(self):
        if self.side is not None:          # attractive pass concurrently with the tree work
            main = torch.cuda.current_stream()
            self.side.wait_stream(main)
            with torch.cuda.stream(self.side):
                self.ops.attract(self.rp, self.col, self.val, self.N, self.row0, self.row1,
                                 self.Y, self.A)
        else:
            self.ops.attract(self.rp, self.col, self.val, self.N, self.row0, self.row1, self.Y,
                             self.A)
        self.ops.forces(self.Y, self.N, self.row0, self.row1, self.theta,
                        self.pending_recentre, self.rep, self.zpart)
        if self.side is not None:
            torch.cuda.current_stream().wait_stream(self.side)
        _all_gather_flat(self.zparts, self.zpart, self.group)
        self.ops.update(self.A, self.N, self.row0, self.row1, self.Y, self.rep, self.zparts,
                        self.world, self.t, self.lr, self.exag, self.cfg, self.v, self.g,
                        self.Yloc)
        _all_gather_flat(self.Yfull, self.Yloc, self.group)

    def step(self, n_iter: int = 1):
        for _ in range(n_iter):
            if self.use_graphs and self.pending_recentre:
                phase = int(self.t >= self.exag_iters)
                g = self._graphs.get(phase)
                if g is None:
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, capture_error_mode="thread_local"):
                        self._iteration()          # captured, not run
                    self._graphs[phase] = g
                g.replay()
            else:
                self._iteration()
            self.t += 1
            self.pending_recentre = True

    def embedding(self) -> torch.Tensor:
        if self.pending_recentre:
            self.ops.recentre(self.Y, self.N)
            self.pending_recentre = False
        return self.Y


def run(X_local: torch.Tensor, N: int, perplexity=30.0, theta=0.5, learning_rate=200.0,
        n_iter=1000, exaggeration=12.0, seed=42, K=0, exag_iters=250, Y_out=None,
        group=None, device=None, ops=None, cfg=None):
    """Multi-GPU end to end.  X_local: this rank's rows shard_range(N, world,
    rank) of X (float32, host -- pinned for speed -- or device).  Returns
    (Y, info) on every rank: Y the full embedding on the device; on rank 0
    it is also copied into Y_out (host or device) when given."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r0, r1, S = shard_range(N, world, rank)
    if X_local.dtype != torch.float32 or X_local.dim() != 2 or X_local.shape[0] != r1 - r0:
        raise ValueError("X_local must be float32 [row1-row0, D] for this rank's shard")
    D = X_local.shape[1]
    if device is None:
        device = X_local.device if X_local.is_cuda else torch.device("cuda", torch.cuda.current_device())
    if K <= 0:
        K = min(N - 1, int(3 * perplexity))                      # D4
    ops = ops if ops is not None else GpuShardOps(N, device)
    # 1. X: own rows host->device, then all-gather (padded to world * S rows)
    Xloc = torch.zeros(S, D, dtype=torch.float32, device=device)
    Xloc[: r1 - r0].copy_(X_local, non_blocking=True)
    Xfull = torch.empty(world * S, D, dtype=torch.float32, device=device)
    _all_gather_flat(Xfull, Xloc, group)
    del Xloc
    X = Xfull[:N]
    # 2. kNN of the own query rows against all N points
    idx_l, d2_l, uncert = ops.knn_rows(X, K, r0, r1)
    del X, Xfull
    idx_p = torch.zeros(S, K, dtype=torch.int32, device=device)
    d2_p = torch.zeros(S, K, dtype=torch.float64, device=device)
    idx_p[: r1 - r0] = idx_l
    d2_p[: r1 - r0] = d2_l
    del idx_l, d2_l
    idx = torch.empty(world * S, K, dtype=torch.int32, device=device)
    d2 = torch.empty(world * S, K, dtype=torch.float64, device=device)
    _all_gather_flat(idx, idx_p, group)
    _all_gather_flat(d2, d2_p, group)
    del idx_p, d2_p
    # 3. P on every rank (needs all rows), keep the own rows
    rp, col, val = ops.compute_p(idx[:N].contiguous(), d2[:N].contiguous(), perplexity)
    nnz = int(col.numel())
    del idx, d2
    rpl, cl, vl = local_csr(rp, col, val, r0, r1)
    del rp, col, val
    # 4. the sharded iterations
    opt = ShardedOptimizer(rpl, cl, vl, ops.init_y(N, seed, device), theta=theta,
                           learning_rate=learning_rate, exaggeration=exaggeration,
                           exag_iters=exag_iters, group=group, ops=ops, cfg=cfg)
    opt.step(n_iter)
    Y = opt.embedding()
    if rank == 0 and Y_out is not None:
        Y_out.copy_(Y)
    u = torch.tensor([float(uncert)], dtype=torch.float64, device=device)
    dist.all_reduce(u, group=group)
    return Y, {"N": N, "K": K, "nnz": nnz, "knn_rows_uncertified": int(u.item())}
