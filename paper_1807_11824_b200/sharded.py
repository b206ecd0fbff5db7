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

`run` is the multi-GPU end-to-end call (Algorithm 1): a thin
caller of the C ABI's tsne_run_sharded, which owns its NCCL communicator
(built from an id rank 0 makes and `run` broadcasts): each rank copies its
own rows of X host->device, the rows are all-gathered, each rank finds the
neighbours of its own query rows, the kNN lists are all-gathered, P is built
redundantly on every rank (it is ~40 ms at C5 and needs every row:
symmetrisation), and the sharded iterations run; rank 0 gets the final Y.
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
    """The C-ABI kernels of one rank (tsne_shard_forces / _attract / _update,
    tsne_recentre) for ShardedOptimizer."""

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


def nccl_unique_id(group=None, device=None) -> bytes:
    """An NCCL unique id (TSNE_NCCL_ID_BYTES bytes) made by rank 0 of `group`
    (tsne_nccl_unique_id) and broadcast to every rank over torch.distributed."""
    from . import _check, lib
    n = 128
    if dist.get_rank(group) == 0:
        buf = (C.c_uint8 * n)()
        _check(lib().tsne_nccl_unique_id(buf), "tsne_nccl_unique_id")
        t = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
    else:
        t = torch.zeros(n, dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        t = t.to(device if device is not None else torch.device("cuda", torch.cuda.current_device()))
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast(t, src=src, group=group)
    return bytes(t.cpu().tolist())


def run(X_local: torch.Tensor, N: int, perplexity=30.0, theta=0.5, learning_rate=200.0,
        n_iter=1000, exaggeration=12.0, seed=42, K=0, exag_iters=250, Y_out=None,
        group=None, device=None, use_graphs=True, _lib=None):
    """Multi-GPU end to end (tsne_run_sharded, Algorithm 1): one
    process per GPU; X_local = this rank's rows shard_range(N, world, rank) of
    X (float32, host -- pinned for speed -- or device).  The library builds its
    own NCCL communicator from an id that rank 0 makes and this function
    broadcasts over `group`; everything else (X all-gather, kNN of the own
    rows, list all-gather, P, the sharded iterations) runs inside the call.
    Returns (Y_out, info) on every rank; Y_out (host or device, N x 2) is
    written on rank 0 (allocated there on the host if not given)."""
    from . import RunInfo, _check, _ptr, default_config, lib
    L = _lib if _lib is not None else lib()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r0, r1, S = shard_range(N, world, rank)
    if X_local.dtype != torch.float32 or X_local.dim() != 2 or X_local.shape[0] != r1 - r0:
        raise ValueError("X_local must be float32 [row1-row0, D] for this rank's shard")
    X_local = X_local.contiguous()
    D = X_local.shape[1]
    if device is not None and device.type == "cuda" and device.index is not None:
        torch.cuda.set_device(device)
    if rank == 0 and Y_out is None:
        Y_out = torch.empty(N, 2, dtype=torch.float32)
    uid = nccl_unique_id(group, device)
    idbuf = (C.c_uint8 * len(uid)).from_buffer_copy(uid)
    cfg = default_config(K=int(K), exag_iters=exag_iters, seed=seed,
                         use_graphs=1 if use_graphs else 0)
    info = RunInfo()
    if X_local.is_cuda:
        torch.cuda.current_stream().synchronize()        # the call runs on its own stream
    _check(L.tsne_run_sharded(_ptr(X_local), r1 - r0, N, D, float(perplexity), float(theta),
                              float(learning_rate), int(n_iter), float(exaggeration),
                              C.byref(cfg), idbuf, rank, world,
                              _ptr(Y_out if rank == 0 else None), C.byref(info)),
           "tsne_run_sharded")
    out = {f: getattr(info, f) for f, _ in RunInfo._fields_}
    out["N"] = N
    return (Y_out if rank == 0 else None), out
