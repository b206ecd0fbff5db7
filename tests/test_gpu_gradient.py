"""GPU <-> oracle parity of the gradient step (H1-H7) through the C ABI.

Bar (north star): relative L2 of dY <= 1e-4 against the
oracle's BH gradient at theta = 0.5 (same tree definition D7-D11, decisions
as in fp64, D25), <= 1e-5 against the exact O(N^2) gradient at theta = 0.
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import paper_1807_11824_b200 as T
    assert torch.cuda.is_available()
    T.lib()
    return T


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def gpu_grad(T, rp, col, v32, Y, theta, exag=1.0):
    dev = torch.device("cuda")
    dY, Z = T.gradient(torch.as_tensor(rp, device=dev), torch.as_tensor(col, device=dev),
                       torch.as_tensor(v32, device=dev), torch.as_tensor(Y, device=dev), theta,
                       exag)
    return dY.cpu().numpy(), Z


@pytest.mark.parametrize("N", [2, 3, 37, 500])
def test_theta0_vs_exact(T, orc, N):
    rp, col, v32, v64 = synth.random_csr(N, min(8, N - 1), seed=N)
    Y = synth.fixed_y("gauss10", N, seed=1)
    for exag in (1.0, 12.0):
        g, Z = gpu_grad(T, rp, col, v32, Y, 0.0, exag)
        ge, Ze = orc.gradient_exact(rp, col, v32.astype(np.float64), Y.astype(np.float64), exag)
        assert abs(Z - Ze) <= 1e-6 * Ze
        # scale: the gradient, or its attractive term when they cancel (N = 2: p = q, g = 0)
        scale = max(np.linalg.norm(ge), np.linalg.norm(4 * exag * orc.attractive(rp, col, v32, Y)))
        assert np.linalg.norm(g - ge) <= 1e-5 * scale


@pytest.mark.parametrize("kind", ["gauss10", "clustered", "blobs"])
@pytest.mark.parametrize("N", [1000, 4099, 20000])
def test_theta05_vs_oracle_bh(T, orc, kind, N):
    rp, col, v32, _ = synth.random_csr(N, 10, seed=7)
    Y = synth.fixed_y(kind, N, seed=3)
    g, Z = gpu_grad(T, rp, col, v32, Y, 0.5, 12.0)
    go, Zo = orc.gradient_bh(rp, col, v32, Y, 0.5, 12.0)
    assert abs(Z - Zo) <= 1e-6 * Zo
    assert rel(g, go) <= 1e-4


@pytest.mark.parametrize("theta", [0.25, 0.8, 1.5])
def test_other_thetas(T, orc, theta):
    N = 6000
    rp, col, v32, _ = synth.random_csr(N, 10, seed=8)
    Y = synth.fixed_y("blobs", N, seed=4)
    g, Z = gpu_grad(T, rp, col, v32, Y, theta)
    go, Zo = orc.gradient_bh(rp, col, v32, Y, theta)
    assert abs(Z - Zo) <= 1e-6 * Zo
    assert rel(g, go) <= 1e-4


def test_duplicates_and_buckets(T, orc):
    # coincident points -> level-24 buckets (tested and exact), D9
    N = 3000
    Y = np.round(synth.fixed_y("gauss10", N, seed=5) / 2.0).astype(np.float32) * 2.0
    Y[:50] = Y[0]                       # one large bucket
    rp, col, v32, _ = synth.random_csr(N, 6, seed=9)
    for theta in (0.0, 0.5):
        g, Z = gpu_grad(T, rp, col, v32, Y, theta)
        go, Zo = orc.gradient_bh(rp, col, v32, Y, theta)
        assert abs(Z - Zo) <= 1e-6 * Zo
        assert rel(g, go) <= 1e-4


def test_all_points_identical(T, orc):
    N = 64
    Y = np.ones((N, 2), np.float32)
    rp, col, v32, _ = synth.random_csr(N, 4, seed=1)
    g, Z = gpu_grad(T, rp, col, v32, Y, 0.5)
    assert Z == N * (N - 1)            # every pair has w = 1
    assert np.abs(g).max() == 0.0


def test_five_point_example(T, orc):
    import json, os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                       "five_point_theta05.json")))
    Y = np.array(gold["points"], np.float32)
    rp = np.zeros(6, np.int64)             # P = 0: dY = -4 f / Z
    col = np.zeros(0, np.int32)
    val = np.zeros(0, np.float32)
    dev = torch.device("cuda")
    dY, Z = T.gradient(torch.as_tensor(rp, device=dev), torch.zeros(1, dtype=torch.int32, device=dev),
                       torch.zeros(1, dtype=torch.float32, device=dev), torch.as_tensor(Y, device=dev),
                       0.5, 1.0)
    _, zo, Zo, _ = orc.repulsive_bh(Y, 0.5)
    assert abs(Z - Zo) <= 1e-6 * Zo
    f0 = -dY[0].cpu().numpy() * Z / 4.0
    np.testing.assert_allclose(f0, gold["bh"]["f0"], rtol=1e-5)


def test_translation_and_determinism(T, orc):
    N = 5000
    rp, col, v32, _ = synth.random_csr(N, 10, seed=2)
    Y = synth.fixed_y("clustered", N, seed=6)
    g1, Z1 = gpu_grad(T, rp, col, v32, Y, 0.5)
    g2, Z2 = gpu_grad(T, rp, col, v32, Y, 0.5)
    assert np.array_equal(g1, g2) and Z1 == Z2          # bitwise deterministic
    g3, _ = gpu_grad(T, rp, col, v32, Y + np.float32(64.0), 0.5)
    assert rel(g3, g1.astype(np.float64)) < 1e-3


def test_real_p_from_oracle(T, orc):
    # P built by the oracle from C1 data (fp32-rounded), Y at a mid-run state
    X = synth.make_x("C1").numpy()
    idx, d2 = orc.knn(X, 90)
    rp, col, v64, v32, *_ = orc.compute_p(idx, d2, 30.0)
    Y = orc.init_y(1000, 42)
    Y, v, gn = orc.optimize(rp, col, v32, Y, n_iter=300, theta=0.5)
    Y = Y.astype(np.float32)
    for theta in (0.0, 0.5):
        g, Z = gpu_grad(T, rp, col, v32, Y, theta, 1.0)
        go, Zo = orc.gradient_bh(rp, col, v32, Y, theta, 1.0)
        assert rel(g, go) <= (1e-5 if theta == 0 else 1e-4)


@pytest.mark.parametrize("kind", ["gauss10", "blobs"])
def test_hub_rows(T, orc, kind):
    # rows of 2.5k-15k nonzeros (k_attract_long) among short ones (the TMA
    # pipeline), including rows between 256 and 2048 (8-deep gathers)
    N = 20000
    rp, col, v32, _ = synth.hub_csr(N, 8, (300, 700, 1500, 2100, 2500, 5000, 15000), seed=17)
    assert (np.diff(rp) > 2048).sum() >= 3
    Y = synth.fixed_y(kind, N, seed=9)
    g, Z = gpu_grad(T, rp, col, v32, Y, 0.5, 12.0)
    go, Zo = orc.gradient_bh(rp, col, v32, Y, 0.5, 12.0)
    assert rel(g, go) <= 1e-4
    # the attractive part alone, row by row, through a theta = 0.5 gradient at exaggeration
    # 1 and 2 (dY(2) - dY(1) = 4 A): checks the long rows' sums directly
    g1, _ = gpu_grad(T, rp, col, v32, Y, 0.5, 1.0)
    g2, _ = gpu_grad(T, rp, col, v32, Y, 0.5, 2.0)
    A = orc.attractive(rp, col, v32, Y)
    long_rows = np.nonzero(np.diff(rp) > 256)[0]
    np.testing.assert_allclose((g2 - g1)[long_rows] / 4.0, A[long_rows], rtol=2e-4,
                               atol=1e-6 * np.abs(A).max())


def test_long_uniform_rows(T, orc):
    # K = 150-like rows of 300 nonzeros everywhere (C4 shape)
    N = 8000
    rp, col, v32 = synth.random_rows_csr(N, 300, seed=5)
    Y = synth.fixed_y("clustered", N, seed=2)
    g1, _ = gpu_grad(T, rp, col, v32, Y, 0.5, 1.0)
    g2, _ = gpu_grad(T, rp, col, v32, Y, 0.5, 2.0)
    A = orc.attractive(rp, col, v32, Y)
    assert rel((g2 - g1) / 4.0, A) <= 1e-5


@pytest.mark.parametrize("name", ["five_point_theta05", "half_side_theta05"])
def test_hand_worked_goldens(T, name):
    """The GPU path on the hand-worked goldens (tests/golden): query point 0 has
    no attractive term (its CSR row is empty), so dY_0 = -4 f_0 / Z (Eq. 6-7);
    the half-side golden separates D7's half-side reading from the full-side
    and geometric-centre readings."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", name + ".json")))
    Y = np.array(g["points"], np.float32)
    rp = np.array([0, 0, 0, 0, 1, 2], np.int64)
    col = np.array([4, 3], np.int32)
    val = np.array([0.5, 0.5], np.float32)
    dY, Z = gpu_grad(T, rp, col, val, Y, g["theta"], 1.0)
    f0 = -dY[0].astype(np.float64) * Z / 4.0
    np.testing.assert_allclose(f0, g["bh"]["f0"], rtol=2e-6)


@pytest.mark.parametrize("case", ["identical_12000", "collapsed_clusters", "dense_cells"])
def test_dense_cells_and_coincident_points(T, orc, case):
    # Embeddings whose Morton keys pile up: thousands of coincident points (one
    # level-24 bucket, D9), clusters collapsed to 1e-5 (deep chains of one-child
    # cells), many dense cells of a few hundred points, plus a background.
    rng = np.random.default_rng(11)
    if case == "identical_12000":         # one bucket of 12000 coincident points + background
        Y = np.concatenate([np.full((12000, 2), 0.25), rng.normal(0, 10, (8000, 2))])
    elif case == "collapsed_clusters":    # buckets of ~9000 and ~3000 (merge / CTA paths)
        c = [rng.normal(m, 1e-5, (n, 2)) for m, n in (((5, 5), 9000), ((-7, 2), 3000),
                                                       ((1, -8), 600))]
        Y = np.concatenate(c + [rng.normal(0, 10, (7400, 2))])
    else:                                 # many buckets of a few hundred points
        Y = np.concatenate([rng.normal(rng.uniform(-20, 20, 2), 0.02, (300, 2))
                            for _ in range(60)] + [rng.normal(0, 10, (2000, 2))])
    Y = Y[rng.permutation(len(Y))].astype(np.float32)
    N = len(Y)
    rp, col, v32, _ = synth.random_csr(N, 10, seed=5)
    g, Z = gpu_grad(T, rp, col, v32, Y, 0.5, 12.0)
    go, Zo = orc.gradient_bh(rp, col, v32, Y, 0.5, 12.0)
    assert abs(Z - Zo) <= 1e-6 * Zo
    assert rel(g, go) <= 1e-4


def test_error_monotone_in_theta_gpu(T):
    # S:L271 (error monotone in theta) on the GPU path at N = 20000, against the
    # exact gradient (theta = 0 reaches every leaf)
    rp, col, v32, _ = synth.random_csr(20000, 10, seed=9)
    Y = synth.fixed_y("clustered", 20000, seed=4)
    g0, Z0 = gpu_grad(T, rp, col, v32, Y, 0.0, 1.0)
    errs = []
    for th in (0.1, 0.3, 0.5, 0.8, 1.2):
        g, Z = gpu_grad(T, rp, col, v32, Y, th, 1.0)
        errs.append(rel(g, g0))
    assert all(a < b for a, b in zip(errs, errs[1:])), errs
    assert errs[0] < 1e-3 and errs[-1] < 0.5


@pytest.mark.parametrize("N", [12000, 40000])
def test_sort_bucket_overflow(T, orc, N):
    # Two far clusters whose members interleave in index order at a regular
    # stride (every N/nsamp-th point in one, the rest in the other): a layout
    # adversarial to any sort that samples regular positions of its input
    # order (the exp/sample-sort-tree branch's tree build did; kept as a
    # parity case for extreme, index-interleaved clusters).
    nb = -(-N // 1843)
    nsamp = 8 * nb
    rng = np.random.default_rng(N)
    Y = (rng.standard_normal((N, 2)) * 0.5 + 20.0).astype(np.float32)
    samp = (np.arange(nsamp, dtype=np.int64) * N) // nsamp
    Y[samp] = (rng.standard_normal((nsamp, 2)) * 0.5 - 20.0).astype(np.float32)
    rp, col, v32, _ = synth.random_csr(N, 8, seed=11)
    g, Z = gpu_grad(T, rp, col, v32, Y, 0.5, 4.0)
    go, Zo = orc.gradient_bh(rp, col, v32, Y, 0.5, 4.0)
    assert abs(Z - Zo) <= 1e-6 * Zo
    assert rel(g, go) <= 1e-4


@pytest.mark.parametrize("N", [20000, 40000])
def test_collapsed_cluster_buckets(T, orc, N):
    # a collapsed cluster over 36 adjacent finest cells (synth 'collapsed'):
    # each point takes exact pairs with the neighbouring buckets it cannot
    # accept -- more than the traversal's per-lane deferral list holds; at
    # N = 40000 the buckets (~120 points) take the k_defer_large path
    Y = synth.fixed_y("collapsed", N, seed=21)
    rp, col, v32, _ = synth.random_csr(N, 8, seed=12)
    for theta in (0.5, 0.8):
        g, Z = gpu_grad(T, rp, col, v32, Y, theta, 12.0)
        go, Zo = orc.gradient_bh(rp, col, v32, Y, theta, 12.0)
        assert abs(Z - Zo) <= 1e-6 * Zo
        assert rel(g, go) <= 1e-4
