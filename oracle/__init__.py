"""fp64 CPU oracle for Barnes-Hut t-SNE (arXiv 1807.11824) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_1807_11824_b200``) never imports it, and the two share no
code: this module is a ctypes binding over ``oracle/tsne_oracle.c`` (plain C,
fp64), whose header lists which passage of PAPER.md each routine follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tsne_oracle.c")
_LIB = os.path.join(_HERE, "libtsne_oracle.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def _P(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        i64, i32, f64, f32, u32 = C.c_int64, C.c_int32, C.c_double, C.c_float, C.c_uint32
        P = C.POINTER
        L.oracle_knn.argtypes = [P(f32), i64, i32, i32, P(i32), P(f64)]
        L.oracle_knn_rows.argtypes = [P(f32), i64, i32, i32, P(i64), i64, P(i32), P(f64)]
        L.oracle_sqdist.argtypes = [P(f32), i32, i64, i64]
        L.oracle_sqdist.restype = f64
        L.oracle_calibrate_row.argtypes = [P(f64), i32, f64, P(f64), P(f64), P(i32)]
        L.oracle_calibrate.argtypes = [P(f64), i64, i32, f64, P(f64), P(f64), P(i32)]
        L.oracle_calibrate.restype = i64
        L.oracle_symmetrize.argtypes = [P(i32), P(f64), i64, i32, P(i64), P(i32), P(f64), P(f32)]
        L.oracle_symmetrize.restype = i64
        L.oracle_repulsive_bh.argtypes = [P(f32), i64, f64, P(i64), i64, P(f64), P(f64),
                                          P(f64), P(i64)]
        L.oracle_tree_dump.argtypes = [P(f32), i64, P(i32), P(i64), P(i32), P(f64), P(f64)]
        L.oracle_tree_dump.restype = i64
        L.oracle_attractive.argtypes = [P(i64), P(i32), P(f32), i64, P(f32), P(f64)]
        L.oracle_gradient_bh.argtypes = [P(i64), P(i32), P(f32), i64, P(f32), f64, f64,
                                         P(f64), P(f64)]
        L.oracle_gradient_exact_d.argtypes = [P(i64), P(i32), P(f64), i64, P(f64), f64,
                                              P(f64), P(f64)]
        L.oracle_kl_d.argtypes = [P(i64), P(i32), P(f64), i64, P(f64)]
        L.oracle_kl_d.restype = f64
        L.oracle_kl.argtypes = [P(i64), P(i32), P(f32), i64, P(f64)]
        L.oracle_kl.restype = f64
        L.oracle_philox4x32_10.argtypes = [P(u32), P(u32), P(u32)]
        L.oracle_init_y.argtypes = [i64, C.c_uint64, P(f64)]
        L.oracle_optimize.argtypes = [P(i64), P(i32), P(f32), i64, P(f64), P(f64), P(f64),
                                      i32, i32, f64, f64, f64, i32, f64, f64, f64]
        L.oracle_nn_preservation.argtypes = [P(i32), i32, i64, P(f64), i32]
        L.oracle_nn_preservation.restype = f64
        L.oracle_ivfpq_search.argtypes = [P(f32), i64, i32, i32, i32, i32, i32, P(f32), P(f32),
                                          P(i32), P(C.c_uint8), i32, i32, i32, i32, P(i32),
                                          P(f64)]
        L.oracle_nn_preservation_rows.argtypes = [P(i32), i32, i64, P(f64), i32, P(i64), i64]
        L.oracle_nn_preservation_rows.restype = f64
        L.oracle_run.argtypes = [P(f32), i64, i32, f64, f64, f64, i32, f64, i32, f64, f64, f64,
                                 C.c_uint64, P(f32), P(f64), P(f64), P(i32)]
        L.oracle_num_threads.restype = C.c_int
        L.oracle_set_num_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_num_threads(n: int) -> None:
    lib().oracle_set_num_threads(int(n))


# ---------------------------------------------------------------- O1 kNN
def knn(X: np.ndarray, K: int, rows: np.ndarray | None = None):
    """Exact kNN (O1).  Returns idx int32 (n,K), d2 float64 (n,K) ascending by (d2, idx)."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    N, D = X.shape
    if rows is None:
        idx = np.empty((N, K), np.int32)
        d2 = np.empty((N, K), np.float64)
        rc = lib().oracle_knn(_P(X, C.c_float), N, D, K, _P(idx, C.c_int32), _P(d2, C.c_double))
    else:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        idx = np.empty((len(rows), K), np.int32)
        d2 = np.empty((len(rows), K), np.float64)
        rc = lib().oracle_knn_rows(_P(X, C.c_float), N, D, K, _P(rows, C.c_int64), len(rows),
                                   _P(idx, C.c_int32), _P(d2, C.c_double))
    if rc != 0:
        raise ValueError("oracle_knn: bad arguments")
    return idx, d2


def sqdist(X: np.ndarray, i: int, j: int) -> float:
    X = np.ascontiguousarray(X, dtype=np.float32)
    return float(lib().oracle_sqdist(_P(X, C.c_float), X.shape[1], int(i), int(j)))


# ---------------------------------------------------------------- O2 calibration
def calibrate_row(d: np.ndarray, perplexity: float):
    d = np.ascontiguousarray(d, dtype=np.float64)
    K = d.shape[0]
    p = np.empty(K, np.float64)
    beta = C.c_double()
    it = C.c_int32()
    flag = lib().oracle_calibrate_row(_P(d, C.c_double), K, float(perplexity), _P(p, C.c_double),
                                      C.byref(beta), C.byref(it))
    return p, beta.value, int(flag), it.value


def calibrate(d2: np.ndarray, perplexity: float):
    d2 = np.ascontiguousarray(d2, dtype=np.float64)
    N, K = d2.shape
    P = np.empty((N, K), np.float64)
    beta = np.empty(N, np.float64)
    flags = np.empty(N, np.int32)
    lib().oracle_calibrate(_P(d2, C.c_double), N, K, float(perplexity), _P(P, C.c_double),
                           _P(beta, C.c_double), _P(flags, C.c_int32))
    return P, beta, flags


# ---------------------------------------------------------------- O3 symmetrise
def symmetrize(idx: np.ndarray, P_cond: np.ndarray):
    """Returns (row_ptr int64, col int32, val64 float64, val32 float32)."""
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    P_cond = np.ascontiguousarray(P_cond, dtype=np.float64)
    N, K = idx.shape
    rp = np.empty(N + 1, np.int64)
    col = np.empty(2 * N * K, np.int32)
    v64 = np.empty(2 * N * K, np.float64)
    v32 = np.empty(2 * N * K, np.float32)
    nnz = lib().oracle_symmetrize(_P(idx, C.c_int32), _P(P_cond, C.c_double), N, K,
                                  _P(rp, C.c_int64), _P(col, C.c_int32), _P(v64, C.c_double),
                                  _P(v32, C.c_float))
    if nnz < 0:
        raise MemoryError("oracle_symmetrize")
    return rp, col[:nnz].copy(), v64[:nnz].copy(), v32[:nnz].copy()


def compute_p(idx, d2, perplexity):
    P_cond, beta, flags = calibrate(d2, perplexity)
    rp, col, v64, v32 = symmetrize(idx, P_cond)
    return rp, col, v64, v32, P_cond, beta, flags


# ---------------------------------------------------------------- O4-O7 tree
def repulsive_bh(Y: np.ndarray, theta: float, pts: np.ndarray | None = None):
    """Returns (f (n,2), z (n,), Z or None, stats dict)."""
    Y = np.ascontiguousarray(Y, dtype=np.float32)
    N = Y.shape[0]
    n = N if pts is None else len(pts)
    f = np.empty((n, 2), np.float64)
    z = np.empty(n, np.float64)
    Z = C.c_double(0.0)
    st = np.zeros(3, np.int64)
    if pts is not None:
        pts = np.ascontiguousarray(pts, dtype=np.int64)
        pp = _P(pts, C.c_int64)
    else:
        pp = None
    rc = lib().oracle_repulsive_bh(_P(Y, C.c_float), N, float(theta), pp, n, _P(f, C.c_double),
                                   _P(z, C.c_double), C.byref(Z), _P(st, C.c_int64))
    if rc != 0:
        raise ValueError("oracle_repulsive_bh rc=%d" % rc)
    return f, z, (Z.value if pts is None else None), {
        "nodes": int(st[0]), "visits": int(st[1]), "interactions": int(st[2])}


def tree_dump(Y: np.ndarray):
    Y = np.ascontiguousarray(Y, dtype=np.float32)
    N = Y.shape[0]
    n = lib().oracle_tree_dump(_P(Y, C.c_float), N, None, None, None, None, None)
    level = np.empty(n, np.int32)
    count = np.empty(n, np.int64)
    leaf = np.empty(n, np.int32)
    com = np.empty((n, 2), np.float64)
    box = np.empty(3, np.float64)
    lib().oracle_tree_dump(_P(Y, C.c_float), N, _P(level, C.c_int32), _P(count, C.c_int64),
                           _P(leaf, C.c_int32), _P(com, C.c_double), _P(box, C.c_double))
    return {"level": level, "count": count, "leaf": leaf, "com": com,
            "r0": box[0], "cx": box[1], "cy": box[2]}


# ---------------------------------------------------------------- O8 / gradient
def attractive(row_ptr, col, val32, Y):
    Y = np.ascontiguousarray(Y, dtype=np.float32)
    N = Y.shape[0]
    A = np.empty((N, 2), np.float64)
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cl = np.ascontiguousarray(col, dtype=np.int32)
    vl = np.ascontiguousarray(val32, dtype=np.float32)
    lib().oracle_attractive(_P(rp, C.c_int64), _P(cl, C.c_int32), _P(vl, C.c_float), N,
                            _P(Y, C.c_float), _P(A, C.c_double))
    return A


def gradient_bh(row_ptr, col, val32, Y, theta, exaggeration=1.0):
    Y = np.ascontiguousarray(Y, dtype=np.float32)
    N = Y.shape[0]
    dY = np.empty((N, 2), np.float64)
    Z = C.c_double()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cl = np.ascontiguousarray(col, dtype=np.int32)
    vl = np.ascontiguousarray(val32, dtype=np.float32)
    rc = lib().oracle_gradient_bh(_P(rp, C.c_int64), _P(cl, C.c_int32), _P(vl, C.c_float), N,
                                  _P(Y, C.c_float), float(theta), float(exaggeration),
                                  _P(dY, C.c_double), C.byref(Z))
    if rc != 0:
        raise ValueError("oracle_gradient_bh rc=%d" % rc)
    return dY, Z.value


def gradient_exact(row_ptr, col, val64, Y64, exaggeration=1.0):
    Y64 = np.ascontiguousarray(Y64, dtype=np.float64)
    N = Y64.shape[0]
    dY = np.empty((N, 2), np.float64)
    Z = C.c_double()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cl = np.ascontiguousarray(col, dtype=np.int32)
    vl = np.ascontiguousarray(val64, dtype=np.float64)
    lib().oracle_gradient_exact_d(_P(rp, C.c_int64), _P(cl, C.c_int32), _P(vl, C.c_double), N,
                                  _P(Y64, C.c_double), float(exaggeration), _P(dY, C.c_double),
                                  C.byref(Z))
    return dY, Z.value


def kl(row_ptr, col, val, Y64):
    Y64 = np.ascontiguousarray(Y64, dtype=np.float64)
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cl = np.ascontiguousarray(col, dtype=np.int32)
    if np.asarray(val).dtype == np.float64:
        vl = np.ascontiguousarray(val, dtype=np.float64)
        return float(lib().oracle_kl_d(_P(rp, C.c_int64), _P(cl, C.c_int32), _P(vl, C.c_double),
                                       Y64.shape[0], _P(Y64, C.c_double)))
    vl = np.ascontiguousarray(val, dtype=np.float32)
    return float(lib().oracle_kl(_P(rp, C.c_int64), _P(cl, C.c_int32), _P(vl, C.c_float),
                                 Y64.shape[0], _P(Y64, C.c_double)))


# ---------------------------------------------------------------- D14 / O9-O10
def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    o = np.empty(4, np.uint32)
    lib().oracle_philox4x32_10(_P(c, C.c_uint32), _P(k, C.c_uint32), _P(o, C.c_uint32))
    return o


def init_y(N: int, seed: int = 42):
    Y = np.empty((N, 2), np.float64)
    lib().oracle_init_y(N, C.c_uint64(seed), _P(Y, C.c_double))
    return Y


DEFAULTS = dict(eta=200.0, exaggeration=12.0, exag_iters=250, mom0=0.5, mom1=0.8, min_gain=0.01)


def optimize(row_ptr, col, val32, Y, v=None, gains=None, t0=0, n_iter=1, theta=0.5,
             eta=200.0, exaggeration=12.0, exag_iters=250, mom0=0.5, mom1=0.8, min_gain=0.01):
    """Runs n_iter iterations from (Y, v, gains) in place (fp64); returns (Y, v, gains)."""
    Y = np.ascontiguousarray(Y, dtype=np.float64).copy()
    N = Y.shape[0]
    v = np.zeros((N, 2)) if v is None else np.ascontiguousarray(v, dtype=np.float64).copy()
    gains = np.ones((N, 2)) if gains is None else np.ascontiguousarray(gains, np.float64).copy()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cl = np.ascontiguousarray(col, dtype=np.int32)
    vl = np.ascontiguousarray(val32, dtype=np.float32)
    rc = lib().oracle_optimize(_P(rp, C.c_int64), _P(cl, C.c_int32), _P(vl, C.c_float), N,
                               _P(Y, C.c_double), _P(v, C.c_double), _P(gains, C.c_double),
                               int(t0), int(n_iter), float(theta), float(eta), float(exaggeration),
                               int(exag_iters), float(mom0), float(mom1), float(min_gain))
    if rc != 0:
        raise ValueError("oracle_optimize rc=%d" % rc)
    return Y, v, gains


def ivfpq_search(X, cent, cb, list_of, codes, K, tau, Kc, Pmax=64):
    """O13 IVF-PQ search given an index: cent [nlist, Dp], cb [m, 256, dsub],
    list_of [N] (coarse list of each point), codes [N, m] uint8 (by point).
    Returns idx int32 [N, K] (-1: not found), d2 float64 [N, K] (exact)."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    N, D = X.shape
    cent = np.ascontiguousarray(cent, dtype=np.float32)
    cb = np.ascontiguousarray(cb, dtype=np.float32)
    nlist, Dp = cent.shape
    m, _, dsub = cb.shape
    list_of = np.ascontiguousarray(list_of, dtype=np.int32)
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    idx = np.empty((N, K), np.int32)
    d2 = np.empty((N, K), np.float64)
    rc = lib().oracle_ivfpq_search(_P(X, C.c_float), N, D, Dp, nlist, m, dsub,
                                   _P(cent, C.c_float), _P(cb, C.c_float),
                                   _P(list_of, C.c_int32), _P(codes, C.c_uint8), int(K),
                                   int(tau), int(Kc), int(Pmax), _P(idx, C.c_int32),
                                   _P(d2, C.c_double))
    if rc != 0:
        raise ValueError("oracle_ivfpq_search rc=%d" % rc)
    return idx, d2


def nn_preservation(idx_x, Y64, k=10, rows=None):
    """O12 k-NN preservation; `rows` (optional) restricts the mean to those points
    (idx_x still holds every point's high-dimensional neighbours)."""
    idx_x = np.ascontiguousarray(idx_x, dtype=np.int32)
    Y64 = np.ascontiguousarray(Y64, dtype=np.float64)
    if rows is None:
        return float(lib().oracle_nn_preservation(_P(idx_x, C.c_int32), idx_x.shape[1],
                                                  Y64.shape[0], _P(Y64, C.c_double), int(k)))
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    return float(lib().oracle_nn_preservation_rows(_P(idx_x, C.c_int32), idx_x.shape[1],
                                                   Y64.shape[0], _P(Y64, C.c_double), int(k),
                                                   _P(rows, C.c_int64), len(rows)))


def run(X, perplexity=30.0, theta=0.5, eta=200.0, n_iter=1000, exaggeration=12.0,
        exag_iters=250, mom0=0.5, mom1=0.8, min_gain=0.01, seed=42, Y_init=None):
    """Full oracle pipeline.  Returns (Y fp64 (N,2), KL, knn idx)."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    N, D = X.shape
    K = min(N - 1, int(np.floor(3 * perplexity)))
    Y = np.empty((N, 2), np.float64)
    kl_out = C.c_double()
    idx = np.empty((N, K), np.int32)
    yi = None
    if Y_init is not None:
        Y_init = np.ascontiguousarray(Y_init, dtype=np.float32)
        yi = _P(Y_init, C.c_float)
    rc = lib().oracle_run(_P(X, C.c_float), N, D, float(perplexity), float(theta), float(eta),
                          int(n_iter), float(exaggeration), int(exag_iters), float(mom0),
                          float(mom1), float(min_gain), C.c_uint64(seed), yi, _P(Y, C.c_double),
                          C.byref(kl_out), _P(idx, C.c_int32))
    if rc != 0:
        raise ValueError("oracle_run rc=%d" % rc)
    return Y, kl_out.value, idx
