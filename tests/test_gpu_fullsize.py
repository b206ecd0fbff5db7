"""Parity at BASELINE.json's full size (C5: N = 1,281,167, D = 2048, K = 90),
in the launch configuration bench.py times, on sampled outputs the oracle can
compute one by one (kNN rows, calibration of those rows, gradient rows) and
on invariants that hold at any size (P symmetric, sums to 1, nnz bounds)."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

N5 = synth.CONFIGS["C5"].N


@pytest.fixture(scope="module")
def T():
    import paper_1807_11824_b200 as T
    T.lib()
    return T


@pytest.fixture(scope="module")
def c5(T):
    X = synth.make_x("C5", device="cuda")
    idx, d2, info = T.knn(X, 90)
    rp, col, val, beta = T.compute_p(idx, d2, 30.0, return_beta=True)
    Xh = X.cpu().numpy()
    del X
    torch.cuda.empty_cache()
    return Xh, idx, d2, info, rp, col, val, beta


def test_c5_knn_sampled_rows(orc, c5):
    # 1024 rows of the full-size kNN (symmetric tcgen05 search, the bench's
    # launch configuration) against the oracle's brute-force fp64 rows
    Xh, idx, d2, info, *_ = c5
    assert info["gemm_path"].startswith("tcgen05") and info["rows_uncertified"] == 0
    rows = np.random.default_rng(5).choice(N5, 1022, replace=False)
    rows = np.append(rows, [0, N5 - 1])          # first and last (ragged tail)
    io, do = orc.knn(Xh, 90, rows=rows)
    ig = idx[torch.as_tensor(rows, device=idx.device)].cpu().numpy()
    dg = d2[torch.as_tensor(rows, device=d2.device)].cpu().numpy()
    np.testing.assert_allclose(dg, do, rtol=1e-10, atol=0)
    for a, b in np.argwhere(ig != io):
        dj = orc.sqdist(Xh, rows[a], ig[a, b])
        assert abs(dj - do[a, b]) <= 1e-6 * do[a, b]


def test_c5_calibration_sampled_rows(orc, c5):
    Xh, idx, d2, info, rp, col, val, beta = c5
    rows = np.random.default_rng(6).choice(N5, 64, replace=False)
    d2h = d2[torch.as_tensor(rows, device=d2.device)].cpu().numpy()
    bg = beta[torch.as_tensor(rows, device=beta.device)].cpu().numpy()
    for r, d in zip(range(len(rows)), d2h):
        p, b, flag, _ = orc.calibrate_row(d, 30.0)
        assert flag == 0 and abs(bg[r] / b - 1) < 1e-6


def test_c5_p_invariants(c5):
    Xh, idx, d2, info, rp, col, val, beta = c5
    nnz = col.numel()
    assert N5 * 90 <= nnz <= 2 * N5 * 90
    assert abs(float(val.double().sum()) - 1.0) < 1e-5
    # bitwise symmetry: the transposed pattern holds the same values
    rows = torch.repeat_interleave(torch.arange(N5, device=col.device),
                                   (rp[1:] - rp[:-1]).to(torch.int64))
    key = rows.to(torch.int64) * N5 + col.to(torch.int64)
    keyT = col.to(torch.int64) * N5 + rows.to(torch.int64)
    o = torch.argsort(key)
    oT = torch.argsort(keyT)
    assert torch.equal(key[o], keyT[oT])
    assert torch.equal(val[o], val[oT])


def test_c5_gradient_sampled_rows(T, orc):
    Y = synth.fixed_y("clustered", N5, seed=3,
                      labels=torch.randint(0, 1000, (N5,), generator=torch.Generator().manual_seed(3)))
    rp, col, val = synth.random_rows_csr(N5, 126)
    dev = torch.device("cuda")
    dY, Z = T.gradient(torch.as_tensor(rp, device=dev), torch.as_tensor(col, device=dev),
                       torch.as_tensor(val, device=dev), torch.as_tensor(Y, device=dev), 0.5, 12.0)
    f, z, Zo, _ = orc.repulsive_bh(Y, 0.5)
    A = orc.attractive(rp, col, val, Y)
    rows = np.random.default_rng(7).choice(N5, 4096, replace=False)
    go = 4.0 * (12.0 * A[rows] - f[rows] / Zo)
    gg = dY.cpu().numpy()[rows].astype(np.float64)
    assert abs(Z - Zo) <= 1e-6 * Zo
    assert np.linalg.norm(gg - go) / np.linalg.norm(go) <= 1e-4


def test_c5_optimizer_runs(T, c5):
    Xh, idx, d2, info, rp, col, val, beta = c5
    opt = T.Optimizer(rp, col, val, T.init_y(N5, 42), theta=0.5)
    Y = opt.step(50)
    assert torch.isfinite(Y).all()
    assert float(Y.double().mean(0).abs().max()) < 1e-4 * float(Y.abs().max())
