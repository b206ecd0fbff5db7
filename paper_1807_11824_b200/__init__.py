"""B200-native Barnes-Hut t-SNE (after t-SNE-CUDA, arXiv 1807.11824).

Thin Python binding over the C ABI of ``libtsne_b200.so`` (include/tsne.h):
argument marshalling only -- every step of the method runs in the library's
CUDA kernels.  PyTorch provides device memory (workspaces are torch tensors),
streams and process groups.  There is no CPU fallback: if the extension is
missing or no sm_100 device is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtsne_b200.so")

_lib = None


class TsneError(RuntimeError):
    pass


STATUS = {0: "TSNE_OK", 1: "TSNE_ERR_ARG", 2: "TSNE_ERR_CUDA", 3: "TSNE_ERR_WORKSPACE",
          4: "TSNE_ERR_NONFINITE", 5: "TSNE_ERR_NCCL", 6: "TSNE_ERR_DEGENERATE"}


class Config(C.Structure):
    _fields_ = [("K", C.c_int32), ("exag_iters", C.c_int32), ("mom0", C.c_float),
                ("mom1", C.c_float), ("min_gain", C.c_float), ("seed", C.c_uint64),
                ("Y_init", C.c_void_p), ("use_graphs", C.c_int32), ("relabel_every", C.c_int32),
                ("keep_state", C.c_int32), ("knn_tau", C.c_int32)]


class IvfParams(C.Structure):
    _fields_ = [("nlist", C.c_int32), ("m", C.c_int32), ("kmeans_iters", C.c_int32),
                ("train_per_list", C.c_int32), ("kprime", C.c_int32), ("seed", C.c_uint64)]


class KnnInfo(C.Structure):
    _fields_ = [("rows_uncertified", C.c_int64), ("candidates", C.c_int32),
                ("gemm_path", C.c_int32)]


class RunInfo(C.Structure):
    _fields_ = [("ms_knn", C.c_double), ("ms_p", C.c_double), ("ms_loop", C.c_double),
                ("ms_total", C.c_double), ("ms_h2d", C.c_double), ("ms_d2h", C.c_double),
                ("nnz", C.c_int64), ("knn_rows_uncertified", C.c_int64), ("K", C.c_int32),
                ("degenerate_rows", C.c_int32)]


EXPORTS = ["tsne_last_error", "tsne_abi_version", "tsne_config_default",
           "tsne_knn_workspace_size", "tsne_knn", "tsne_knn_rows", "tsne_compute_p_workspace_size",
           "tsne_compute_p", "tsne_gradient_workspace_size", "tsne_gradient",
           "tsne_optimize_workspace_size", "tsne_optimize", "tsne_optimize_release", "tsne_init_y", "tsne_run",
           "tsne_run_ex", "tsne_profile_iterations", "tsne_shard_workspace_size",
           "tsne_shard_forces", "tsne_shard_attract", "tsne_shard_update", "tsne_recentre",
           "tsne_kl_workspace_size", "tsne_kl", "tsne_nccl_unique_id", "tsne_run_workspace_size",
           "tsne_run_sharded", "tsne_ivfpq_params_default", "tsne_ivfpq_index_size",
           "tsne_ivfpq_layout", "tsne_ivfpq_workspace_size", "tsne_ivfpq_build",
           "tsne_ivfpq_search"]


def lib():
    """Load the in-tree extension (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise TsneError(f"{LIB_PATH} not built: run `python -m paper_1807_11824_b200.build` "
                        "(or __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    vp, i64, i32, f32, sz = C.c_void_p, C.c_int64, C.c_int32, C.c_float, C.c_size_t
    L.tsne_last_error.restype = C.c_char_p
    L.tsne_abi_version.restype = i32
    L.tsne_config_default.argtypes = [C.POINTER(Config)]
    L.tsne_knn_workspace_size.argtypes = [i64, i32, i32]
    L.tsne_knn_workspace_size.restype = sz
    L.tsne_knn.argtypes = [vp, i64, i32, i32, vp, vp, vp, sz, C.POINTER(KnnInfo), vp]
    L.tsne_knn_rows.argtypes = [vp, i64, i32, i32, i64, i64, vp, vp, vp, sz, C.POINTER(KnnInfo), vp]
    L.tsne_compute_p_workspace_size.argtypes = [i64, i32]
    L.tsne_compute_p_workspace_size.restype = sz
    L.tsne_compute_p.argtypes = [vp, vp, i64, i32, f32, vp, vp, vp, C.POINTER(i64), vp, vp, sz, vp]
    L.tsne_gradient_workspace_size.argtypes = [i64]
    L.tsne_gradient_workspace_size.restype = sz
    L.tsne_gradient.argtypes = [vp, vp, vp, i64, vp, f32, f32, vp, C.POINTER(C.c_double), vp, sz,
                                vp]
    L.tsne_optimize_workspace_size.argtypes = [i64, i64]
    L.tsne_optimize_workspace_size.restype = sz
    L.tsne_optimize.argtypes = [vp, vp, vp, i64, vp, vp, vp, i32, i32, f32, f32, f32,
                                C.POINTER(Config), vp, sz, vp]
    L.tsne_optimize_release.argtypes = [vp]
    L.tsne_optimize_release.restype = None
    L.tsne_init_y.argtypes = [i64, C.c_uint64, vp, vp]
    L.tsne_profile_iterations.argtypes = [vp, vp, vp, i64, vp, vp, vp, i32, i32, f32, f32, f32,
                                          C.POINTER(Config), C.POINTER(C.c_double),
                                          C.POINTER(i32), C.POINTER(C.c_double), vp, sz, vp]
    L.tsne_run.argtypes = [vp, i64, i32, f32, f32, f32, i32, f32, vp]
    L.tsne_run_ex.argtypes = [vp, i64, i32, f32, f32, f32, i32, f32, C.POINTER(Config), vp,
                              C.POINTER(RunInfo)]
    L.tsne_shard_workspace_size.argtypes = [i64]
    L.tsne_shard_workspace_size.restype = sz
    L.tsne_shard_forces.argtypes = [vp, i64, i64, i64, f32, i32, vp, vp, vp, sz, vp]
    L.tsne_shard_attract.argtypes = [vp, vp, vp, i64, i64, i64, vp, vp, vp]
    L.tsne_shard_update.argtypes = [vp, i64, i64, i64, vp, vp, vp, i32, i32, f32, f32,
                                    C.POINTER(Config), vp, vp, vp, vp, vp, sz, vp]
    L.tsne_recentre.argtypes = [vp, i64, vp, sz, vp]
    L.tsne_kl_workspace_size.argtypes = [i64]
    L.tsne_kl_workspace_size.restype = sz
    L.tsne_kl.argtypes = [vp, vp, vp, i64, vp, C.POINTER(C.c_double), C.POINTER(C.c_double), vp,
                          sz, vp]
    L.tsne_nccl_unique_id.argtypes = [vp]
    L.tsne_run_workspace_size.argtypes = [i64, i32, i32, i32]
    L.tsne_run_workspace_size.restype = sz
    L.tsne_run_sharded.argtypes = [vp, i64, i64, i32, f32, f32, f32, i32, f32, C.POINTER(Config),
                                   vp, i32, i32, vp, C.POINTER(RunInfo)]
    L.tsne_ivfpq_params_default.argtypes = [C.POINTER(IvfParams)]
    L.tsne_ivfpq_params_default.restype = None
    L.tsne_ivfpq_index_size.argtypes = [i64, i32, C.POINTER(IvfParams)]
    L.tsne_ivfpq_index_size.restype = sz
    L.tsne_ivfpq_layout.argtypes = [i64, i32, C.POINTER(IvfParams), C.POINTER(i64)]
    L.tsne_ivfpq_workspace_size.argtypes = [i64, i32, i32, C.POINTER(IvfParams)]
    L.tsne_ivfpq_workspace_size.restype = sz
    L.tsne_ivfpq_build.argtypes = [vp, i64, i32, C.POINTER(IvfParams), vp, sz, vp, sz, vp]
    L.tsne_ivfpq_search.argtypes = [vp, i64, i32, C.POINTER(IvfParams), vp, i32, i32, vp, vp, vp,
                                    sz, vp]
    for name in ["tsne_ivfpq_layout", "tsne_ivfpq_build", "tsne_ivfpq_search",
                 "tsne_nccl_unique_id", "tsne_run_sharded", "tsne_knn", "tsne_knn_rows", "tsne_compute_p", "tsne_gradient", "tsne_optimize", "tsne_init_y",
                 "tsne_run", "tsne_run_ex", "tsne_profile_iterations", "tsne_shard_forces",
                 "tsne_shard_attract", "tsne_shard_update", "tsne_recentre", "tsne_kl"]:
        getattr(L, name).restype = C.c_int
    _lib = L
    return L


def _check(rc: int, what: str, ok=(0,)):
    if rc not in ok:
        msg = lib().tsne_last_error().decode(errors="replace")
        raise TsneError(f"{what}: {STATUS.get(rc, rc)}: {msg}")
    return rc


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor | None):
    return C.c_void_p(0 if t is None else t.data_ptr())


def _dev(t: torch.Tensor, dtype, name):
    if not t.is_cuda:
        raise TsneError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TsneError(f"{name} must be {dtype} (got {t.dtype})")
    return t.contiguous()


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def default_config(**kw) -> Config:
    cfg = Config()
    lib().tsne_config_default(C.byref(cfg))
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


# ---------------------------------------------------------------- U1
def knn(X: torch.Tensor, K: int, rows=None):
    """Exact kNN: (idx int32 [n,K], d2 float64 [n,K], info dict).  `rows` =
    (q0, q1) restricts the queries to points q0..q1-1 (tsne_knn_rows, the
    multi-GPU shard); by default every point is a query (tsne_knn)."""
    X = _dev(X, torch.float32, "X")
    N, D = X.shape
    q0, q1 = (0, N) if rows is None else (int(rows[0]), int(rows[1]))
    idx = torch.empty(q1 - q0, K, dtype=torch.int32, device=X.device)
    d2 = torch.empty(q1 - q0, K, dtype=torch.float64, device=X.device)
    ws = _ws(lib().tsne_knn_workspace_size(N, D, K), X.device)
    info = KnnInfo()
    if rows is None:
        _check(lib().tsne_knn(_ptr(X), N, D, K, _ptr(idx), _ptr(d2), _ptr(ws), ws.numel(),
                              C.byref(info), _stream()), "tsne_knn")
    else:
        _check(lib().tsne_knn_rows(_ptr(X), N, D, K, q0, q1 - q0, _ptr(idx), _ptr(d2), _ptr(ws),
                                   ws.numel(), C.byref(info), _stream()), "tsne_knn_rows")
    return idx, d2, {"rows_uncertified": info.rows_uncertified, "candidates": info.candidates,
                     "gemm_path": {2: "tcgen05-sym", 1: "tcgen05", 0: "none"}[info.gemm_path]}


# ---------------------------------------------------------------- f2 IVF-PQ
def ivfpq_params(**kw) -> IvfParams:
    p = IvfParams()
    lib().tsne_ivfpq_params_default(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


class IvfPQ:
    """IVF-PQ index of the rows of X (tsne_ivfpq_build) and its kNN search
    (tsne_ivfpq_search): queries are the indexed points, self excluded."""

    def __init__(self, X: torch.Tensor, **params):
        X = _dev(X, torch.float32, "X")
        self.N, self.D = X.shape
        self.params = ivfpq_params(**params)
        nb = lib().tsne_ivfpq_index_size(self.N, self.D, C.byref(self.params))
        self.index = _ws(nb, X.device)
        ws = _ws(lib().tsne_ivfpq_workspace_size(self.N, self.D, 0, C.byref(self.params)),
                 X.device)
        _check(lib().tsne_ivfpq_build(_ptr(X), self.N, self.D, C.byref(self.params),
                                      _ptr(self.index), self.index.numel(), _ptr(ws), ws.numel(),
                                      _stream()), "tsne_ivfpq_build")
        lay = (C.c_int64 * 11)()
        _check(lib().tsne_ivfpq_layout(self.N, self.D, C.byref(self.params), lay),
               "tsne_ivfpq_layout")
        self.nlist, self.m, self.dsub, self.Dp = lay[0], lay[1], lay[2], lay[3]
        self._off = list(lay)

    def parts(self) -> dict:
        """Views of the index parts (tsne_ivfpq_layout): centroids, codebooks,
        codes (list order), list offsets, list entries, T tables."""
        b = self.index
        o = self._off

        def view(off, n, dt):
            itemsize = torch.empty(0, dtype=dt).element_size()
            return b[off: off + n * itemsize].view(dt)
        return {"centroids": view(o[4], self.nlist * self.Dp, torch.float32).view(self.nlist, self.Dp),
                "codebooks": view(o[5], self.m * 256 * self.dsub, torch.float32).view(self.m, 256, self.dsub),
                "codes": view(o[6], self.N * self.m, torch.uint8).view(self.N, self.m),
                "list_offsets": view(o[7], self.nlist + 1, torch.int32),
                "list_ids": view(o[8], self.N, torch.int32),
                "T": view(o[9], self.nlist * self.m * 256, torch.float32).view(self.nlist, self.m, 256),
                "ntrain": o[10]}

    def search(self, X: torch.Tensor, K: int, tau: int):
        X = _dev(X, torch.float32, "X")
        idx = torch.empty(self.N, K, dtype=torch.int32, device=X.device)
        d2 = torch.empty(self.N, K, dtype=torch.float64, device=X.device)
        ws = _ws(lib().tsne_ivfpq_workspace_size(self.N, self.D, K, C.byref(self.params)),
                 X.device)
        _check(lib().tsne_ivfpq_search(_ptr(X), self.N, self.D, C.byref(self.params),
                                       _ptr(self.index), int(K), int(tau), _ptr(idx), _ptr(d2),
                                       _ptr(ws), ws.numel(), _stream()), "tsne_ivfpq_search")
        return idx, d2


# ---------------------------------------------------------------- U2 + U3
def compute_p(idx: torch.Tensor, d2: torch.Tensor, perplexity: float, return_beta=False):
    """Sparse joint P in CSR: (row_ptr int64, col int32, val float32[, beta])."""
    idx = _dev(idx, torch.int32, "idx")
    d2 = _dev(d2, torch.float64, "d2")
    N, K = idx.shape
    dev = idx.device
    row_ptr = torch.empty(N + 1, dtype=torch.int64, device=dev)
    col = torch.empty(2 * N * K, dtype=torch.int32, device=dev)
    val = torch.empty(2 * N * K, dtype=torch.float32, device=dev)
    beta = torch.empty(N, dtype=torch.float64, device=dev)
    nnz = C.c_int64()
    ws = _ws(lib().tsne_compute_p_workspace_size(N, K), dev)
    rc = lib().tsne_compute_p(_ptr(idx), _ptr(d2), N, K, float(perplexity), _ptr(row_ptr),
                              _ptr(col), _ptr(val), C.byref(nnz), _ptr(beta), _ptr(ws),
                              ws.numel(), _stream())
    _check(rc, "tsne_compute_p", ok=(0, 6))
    n = nnz.value
    out = (row_ptr, col[:n].clone(), val[:n].clone())
    return out + (beta,) if return_beta else out


# ---------------------------------------------------------------- H1-H7
def gradient(row_ptr, col, val, Y: torch.Tensor, theta: float = 0.5, exaggeration: float = 1.0):
    """One BH gradient at fixed Y: (dY float32 [N,2], Z float)."""
    Y = _dev(Y, torch.float32, "Y")
    row_ptr = _dev(row_ptr, torch.int64, "row_ptr")
    col = _dev(col, torch.int32, "col")
    val = _dev(val, torch.float32, "val")
    N = Y.shape[0]
    dY = torch.empty_like(Y)
    Z = C.c_double()
    ws = _ws(lib().tsne_gradient_workspace_size(N), Y.device)
    _check(lib().tsne_gradient(_ptr(row_ptr), _ptr(col), _ptr(val), N, _ptr(Y), float(theta),
                               float(exaggeration), _ptr(dY), C.byref(Z), _ptr(ws), ws.numel(),
                               _stream()), "tsne_gradient")
    return dY, Z.value


# ---------------------------------------------------------------- f4
def kl(row_ptr, col, val, Y: torch.Tensor):
    """KL(P || Q) of the embedding Y with the exact normaliser Z (tsne_kl):
    returns (KL, Z)."""
    Y = _dev(Y, torch.float32, "Y")
    row_ptr = _dev(row_ptr, torch.int64, "row_ptr")
    col = _dev(col, torch.int32, "col")
    val = _dev(val, torch.float32, "val")
    N = Y.shape[0]
    out, Z = C.c_double(), C.c_double()
    ws = _ws(lib().tsne_kl_workspace_size(N), Y.device)
    _check(lib().tsne_kl(_ptr(row_ptr), _ptr(col), _ptr(val), N, _ptr(Y), C.byref(out),
                         C.byref(Z), _ptr(ws), ws.numel(), _stream()), "tsne_kl")
    return out.value, Z.value


# ---------------------------------------------------------------- H1-H8
@dataclass
class State:
    Y: torch.Tensor
    v: torch.Tensor
    gains: torch.Tensor
    t: int = 0


class Optimizer:
    """Holds the workspace of the iteration loop; step(n) runs n iterations.
    Consecutive step() calls continue the library's internal state (keep_state):
    the relabelled P and the CUDA graphs stay in the workspace, so step(a);
    step(b) equals step(a + b) bitwise.  Modifying `state` in between is
    detected (fingerprint) and restarts from the modified state."""

    def __init__(self, row_ptr, col, val, Y: torch.Tensor, theta=0.5, learning_rate=200.0,
                 exaggeration=12.0, exag_iters=250, mom0=0.5, mom1=0.8, min_gain=0.01,
                 use_graphs=True, relabel_every=64):
        self.row_ptr = _dev(row_ptr, torch.int64, "row_ptr")
        self.col = _dev(col, torch.int32, "col")
        self.val = _dev(val, torch.float32, "val")
        Y = _dev(Y, torch.float32, "Y").clone()
        self.N = Y.shape[0]
        self.state = State(Y, torch.zeros_like(Y), torch.ones_like(Y), 0)
        self.theta, self.lr, self.exag = float(theta), float(learning_rate), float(exaggeration)
        self.cfg = default_config(exag_iters=exag_iters, mom0=mom0, mom1=mom1, min_gain=min_gain,
                                  use_graphs=1 if use_graphs else 0,
                                  relabel_every=int(relabel_every), keep_state=1)
        self.nnz = int(self.col.numel())
        self.ws = _ws(lib().tsne_optimize_workspace_size(self.N, self.nnz), Y.device)

    def __del__(self):
        try:
            lib().tsne_optimize_release(_ptr(self.ws))
        except Exception:
            pass

    def step(self, n_iter: int = 1, stream=None):
        s = self.state
        st = C.c_void_p(stream) if stream is not None else _stream()
        _check(lib().tsne_optimize(_ptr(self.row_ptr), _ptr(self.col), _ptr(self.val), self.N,
                                   _ptr(s.Y), _ptr(s.v), _ptr(s.gains), s.t, int(n_iter),
                                   self.theta, self.lr, self.exag, C.byref(self.cfg),
                                   _ptr(self.ws), self.ws.numel(), st), "tsne_optimize")
        s.t += int(n_iter)
        return s.Y


def profile_iteration(opt: Optimizer, reps: int = 5, stream=None) -> dict:
    """Per-stage mean CUDA-event times (tsne_profile_iterations; advances the
    optimiser state by 2 * reps iterations like Optimizer.step)."""
    s = opt.state
    ms = (C.c_double * 5)()
    ts = (C.c_double * 5)()
    kern = C.c_int32()
    st = C.c_void_p(stream) if stream is not None else _stream()
    _check(lib().tsne_profile_iterations(_ptr(opt.row_ptr), _ptr(opt.col), _ptr(opt.val), opt.N,
                                         _ptr(s.Y), _ptr(s.v), _ptr(s.gains), s.t, int(reps),
                                         opt.theta, opt.lr, opt.exag, C.byref(opt.cfg), ms,
                                         C.byref(kern), ts, _ptr(opt.ws), opt.ws.numel(), st),
           "tsne_profile_iterations")
    s.t += 2 * int(reps)
    return {"tree_ms": ms[0], "traverse_ms": ms[1], "attract_ms": ms[2], "update_ms": ms[3],
            "iteration_overlapped_ms": ms[4], "kernels_per_iteration": kern.value,
            "traverse_per_point": {"visits": ts[0], "warp_max_visits": ts[1],
                                   "interactions": ts[2], "fp64_decisions": ts[3],
                                   "bucket_pairs": ts[4]}}


def init_y(N: int, seed: int = 42, device="cuda") -> torch.Tensor:
    Y = torch.empty(N, 2, dtype=torch.float32, device=device)
    _check(lib().tsne_init_y(N, seed, _ptr(Y), _stream()), "tsne_init_y")
    return Y


# ---------------------------------------------------------------- Algorithm 1
def run(X: torch.Tensor, perplexity=30.0, theta=0.5, learning_rate=200.0, n_iter=1000,
        exaggeration=12.0, Y_out: torch.Tensor | None = None, Y_init: torch.Tensor | None = None,
        seed: int = 42, K: int = 0, exag_iters: int = 250, use_graphs=True, relabel_every=64,
        knn_tau: int = 0):
    """End to end (tsne_run_ex).  X may live on the host (pinned for speed) or
    the device; Y_out (optional) likewise.  knn_tau > 0: the kNN by IVF-PQ with
    tau probes instead of the exact search.  Returns (Y_out, info dict)."""
    if X.dtype != torch.float32:
        raise TsneError("X must be float32")
    X = X.contiguous()
    N, D = X.shape
    if Y_out is None:
        Y_out = torch.empty(N, 2, dtype=torch.float32, device=X.device,
                            pin_memory=not X.is_cuda and X.is_pinned())
    yi = None
    if Y_init is not None:
        yi = _dev(Y_init, torch.float32, "Y_init")
    cfg = default_config(K=int(K), exag_iters=exag_iters, seed=seed,
                         Y_init=(yi.data_ptr() if yi is not None else None),
                         use_graphs=1 if use_graphs else 0, relabel_every=int(relabel_every),
                         knn_tau=int(knn_tau))
    info = RunInfo()
    if X.is_cuda or Y_out.is_cuda:
        torch.cuda.current_stream().synchronize()   # tsne_run_ex runs on its own stream
    _check(lib().tsne_run_ex(_ptr(X), N, D, float(perplexity), float(theta), float(learning_rate),
                             int(n_iter), float(exaggeration), C.byref(cfg), _ptr(Y_out),
                             C.byref(info)), "tsne_run_ex")
    return Y_out, {f: getattr(info, f) for f, _ in RunInfo._fields_}
