"""Host-side checks that need no GPU: the C-ABI library builds, loads, exports
every symbol include/tsne.h declares, validates arguments before touching the
device, and sizes workspaces."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tsne.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tsne_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_1807_11824_b200 import build
    build.build()
    import paper_1807_11824_b200 as T
    return T.lib()


def test_exports_every_header_symbol(L):
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(L, s), s


def test_binding_lists_all_exports():
    import paper_1807_11824_b200 as T
    assert set(T.EXPORTS) <= set(header_symbols())


def test_abi_version_and_defaults(L):
    import paper_1807_11824_b200 as T
    assert L.tsne_abi_version() >> 16 == 1
    cfg = T.default_config()
    assert (cfg.exag_iters, cfg.seed, cfg.use_graphs, cfg.relabel_every) == (250, 42, 1, 64)
    assert abs(cfg.mom0 - 0.5) < 1e-7 and abs(cfg.mom1 - 0.8) < 1e-7


def test_workspace_sizes_monotone(L):
    a = L.tsne_gradient_workspace_size(1000)
    b = L.tsne_gradient_workspace_size(100000)
    assert 0 < a < b and b % 256 == 0
    assert L.tsne_gradient_workspace_size(1) == 0
    assert L.tsne_knn_workspace_size(5000, 784, 90) > 5000 * 784 * 2
    assert L.tsne_compute_p_workspace_size(5000, 90) > 2 * 5000 * 90 * 16
    assert L.tsne_optimize_workspace_size(5000, 700000) > L.tsne_gradient_workspace_size(5000)
    assert 0 < L.tsne_kl_workspace_size(1000) < L.tsne_kl_workspace_size(1281167)


def test_argument_validation_without_device(L):
    import paper_1807_11824_b200 as T
    v = C.c_void_p(16)
    # theta < 0, N < 2, K >= N, perplexity >= K: TSNE_ERR_ARG before any CUDA call
    assert L.tsne_gradient(v, v, v, 100, v, -1.0, 1.0, v, None, v, 1 << 30, None) == 1
    assert b"theta" in L.tsne_last_error()
    assert L.tsne_gradient(v, v, v, 1, v, 0.5, 1.0, v, None, v, 1 << 30, None) == 1
    assert L.tsne_knn(v, 10, 5, 10, v, v, v, 1 << 30, None, None) == 1
    n = C.c_int64()
    assert L.tsne_compute_p(v, v, 100, 30, 40.0, v, v, v, C.byref(n), None, v, 1 << 30, None) == 1
    assert b"perplexity" in L.tsne_last_error()
    assert L.tsne_run(v, 100, 5, 30.0, -0.5, 200.0, 10, 12.0, v) == 1
    d = C.c_double()
    assert L.tsne_kl(v, v, v, 1, v, C.byref(d), None, v, 1 << 30, None) == 1
    assert L.tsne_kl(v, v, v, 100, v, None, None, v, 1 << 30, None) == 1


def test_workspace_too_small(L):
    v = C.c_void_p(256)
    rc = L.tsne_gradient(v, v, v, 1000, v, 0.5, 1.0, v, None, v, 16, None)
    assert rc == 3 and b"workspace" in L.tsne_last_error()


def test_no_cpu_fallback_without_gpu(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    v = C.c_void_p(256)
    need = L.tsne_gradient_workspace_size(1000)
    rc = L.tsne_gradient(v, v, v, 1000, v, 0.5, 1.0, v, None, v, need, None)
    assert rc == 2   # TSNE_ERR_CUDA: no device, and no host fallback exists


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1807_11824_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                for bad in ("import oracle", "from oracle", "tsne_oracle", "oracle_"):
                    assert bad not in txt, (f, bad)


def test_new_entry_points_validate_without_device(L):
    """tsne_run_sharded, tsne_ivfpq_* and tsne_optimize_release check their
    arguments before any CUDA call (S:L111 style errors)."""
    import paper_1807_11824_b200 as T
    v = C.c_void_p(256)
    uid = (C.c_uint8 * 128)()
    info = T.RunInfo()
    # N_local must be this rank's shard size: N = 100, world 3 -> S = 34, rank 2 owns 32 rows
    rc = L.tsne_run_sharded(v, 34, 100, 8, 10.0, 0.5, 200.0, 10, 12.0, None, uid, 2, 3, None,
                            C.byref(info))
    assert rc == 1 and b"N_local must be 32" in L.tsne_last_error()
    rc = L.tsne_run_sharded(v, 32, 100, 8, 10.0, 0.5, 200.0, 10, 12.0, None, uid, 3, 3, None,
                            C.byref(info))
    assert rc == 1 and b"rank" in L.tsne_last_error()
    # IVF-PQ: index layout defaults (|C| = sqrt(N), m = min(96, ceil(D / 8))) and bad tau
    p = T.ivfpq_params()
    lay = (C.c_int64 * 11)()
    assert L.tsne_ivfpq_layout(10000, 784, C.byref(p), lay) == 0
    assert (lay[0], lay[1], lay[2], lay[3]) == (100, 96, 9, 864)
    assert L.tsne_ivfpq_index_size(10000, 784, C.byref(p)) >= 10000 * 96 + 100 * 864 * 4
    rc = L.tsne_ivfpq_search(v, 10000, 784, C.byref(p), v, 32, 101, v, v, v, 1 << 40, None)
    assert rc == 1 and b"tau" in L.tsne_last_error()
    rc = L.tsne_ivfpq_build(v, 10000, 784, C.byref(T.ivfpq_params(m=4)), v, 1 << 40, v, 1 << 40,
                            None)
    assert rc == 1 and b"dsub" in L.tsne_last_error()
    L.tsne_optimize_release(v)          # unknown workspace: ignored
