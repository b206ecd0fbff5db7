"""Pins for the oracle's O4-O8, O11, O12 (tree, traversal, forces, gradient, KL).

Pinned against: the theta = 0 special case ('theta = 0 giving the
O(N^2) algorithm') evaluated by a direct double loop written here; the
hand-worked five-point theta = 0.5 example (tests/golden); SPEC's hand
examples; central finite differences of KL (the gradient is its derivative);
scikit-learn's exact t-SNE gradient; invariants.
"""
import json
import os

import numpy as np
import pytest

import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def direct_sums(Y):
    """Plain O(N^2) sums of Eq. 4 / Eq. 6 numerators: z_i = sum_j w_ij,
    f_i = sum_j w_ij^2 (y_i - y_j), w = 1/(1 + |y_i - y_j|^2)."""
    Y = Y.astype(np.float64)
    d = Y[:, None, :] - Y[None, :, :]
    w = 1.0 / (1.0 + (d ** 2).sum(-1))
    np.fill_diagonal(w, 0.0)
    z = w.sum(1)
    f = ((w ** 2)[:, :, None] * d).sum(1)
    return f, z


@pytest.mark.parametrize("n", [10, 100, 512])
@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
def test_theta0_equals_direct_sums(orc, n, seed):
    # P:L130 + S:L265, acceptance criterion 1
    Y = synth.fixed_y("gauss10", n, seed=seed)
    f, z, Z, st = orc.repulsive_bh(Y, 0.0)
    fd, zd = direct_sums(Y)
    np.testing.assert_allclose(z, zd, rtol=1e-12)
    np.testing.assert_allclose(f, fd, rtol=1e-10, atol=1e-14 * np.abs(fd).max())
    assert abs(Z - zd.sum()) <= 1e-12 * zd.sum()
    assert st["interactions"] == n * (n - 1)


def test_five_point_hand_example(orc):
    g = json.load(open(os.path.join(GOLD, "five_point_theta05.json")))
    Y = np.array(g["points"], np.float32)
    f, z, Z, st = orc.repulsive_bh(Y, g["theta"])
    assert abs(z[0] - g["bh"]["z0"]) <= 1e-15
    np.testing.assert_allclose(f[0], g["bh"]["f0"], rtol=1e-14)
    f0, z0, _, _ = orc.repulsive_bh(Y, 0.0)
    assert abs(z0[0] - g["exact"]["z0"]) <= 1e-15
    np.testing.assert_allclose(f0[0], g["exact"]["f0"], rtol=1e-14)


def test_half_side_hand_example(orc):
    """D7 pinned: r_cell is HALF the side.  The decisive cell has r_half/D =
    0.257 in [0.25, 0.5), so the full-side reading (and the geometric-centre
    reading) give different z0, f0 -- hand-worked in tests/golden."""
    g = json.load(open(os.path.join(GOLD, "half_side_theta05.json")))
    Y = np.array(g["points"], np.float32)
    f, z, Z, st = orc.repulsive_bh(Y, g["theta"])
    assert abs(z[0] - g["bh"]["z0"]) <= 1e-15
    np.testing.assert_allclose(f[0], g["bh"]["f0"], rtol=1e-14)
    assert abs(z[0] - g["full_side_reading"]["z0"]) > 1e-3      # the readings are told apart
    f0, z0, _, _ = orc.repulsive_bh(Y, 0.0)
    assert abs(z0[0] - g["exact"]["z0"]) <= 1e-15
    np.testing.assert_allclose(f0[0], g["exact"]["f0"], rtol=1e-14)


def test_tree_invariants_unit_square(orc):
    # S:L256 unit-square corners: root count 4, COM (0.5, 0.5), four children of count 1
    Y = np.array([[0, 0], [0, 1], [1, 0], [1, 1]], np.float32)
    t = orc.tree_dump(Y)
    assert t["count"][0] == 4
    np.testing.assert_array_equal(t["com"][0], [0.5, 0.5])
    assert list(t["count"][1:]) == [1, 1, 1, 1] and all(t["leaf"][1:])
    assert t["r0"] == 0.5 * (1 + 2.0 ** -20) and t["cx"] == 0.5
    # centroid query: the 4-fold symmetry cancels the force
    Y5 = np.vstack([Y, [[0.5, 0.5]]]).astype(np.float32)
    for th in (0.0, 0.5, 1.0):
        f, z, _, _ = orc.repulsive_bh(Y5, th)
        assert np.abs(f[4]).max() < 1e-15 and z[4] > 0


def test_tree_counts_and_com(orc):
    Y = synth.fixed_y("blobs", 3000, seed=5)
    t = orc.tree_dump(Y)
    lvl, cnt, leaf, com = t["level"], t["count"], t["leaf"], t["com"]
    assert cnt[0] == 3000
    # pre-order: children of node k are the following nodes at level+1 until
    # the subtree ends; check sum of child counts == parent count
    n = len(lvl)
    for k in range(0, n, 7):
        if leaf[k]:
            assert cnt[k] == 1 or lvl[k] == 24
            continue
        s, m = 0, k + 1
        while m < n and lvl[m] > lvl[k]:
            if lvl[m] == lvl[k] + 1:
                s += cnt[m]
            m += 1
        assert s == cnt[k]
    assert abs(com[0] - Y.astype(np.float64).mean(0)).max() < 1e-12


def test_theta_error_monotone(orc):
    # S:L271 mean relative error non-increasing as theta decreases
    Y = synth.fixed_y("blobs", 2000, seed=11)
    fd, zd = direct_sums(Y)
    errs = []
    for th in (0.8, 0.5, 0.2, 0.0):
        f, z, Z, _ = orc.repulsive_bh(Y, th)
        errs.append(np.linalg.norm(f - fd) / np.linalg.norm(fd))
    assert all(a >= b for a, b in zip(errs, errs[1:]))
    assert errs[-1] < 1e-12 and errs[1] < 0.1


def test_attractive_two_point(orc):
    # S:L322 P12 = 0.5, y1 = (0,0), y2 = (2,0) -> pq = 0.1, F_attr[1] = (-0.2, 0)
    rp = np.array([0, 1, 2]); col = np.array([1, 0]); val = np.array([0.5, 0.5], np.float32)
    A = orc.attractive(rp, col, val, np.array([[0, 0], [2, 0]], np.float32))
    np.testing.assert_allclose(A, [[-0.2, 0.0], [0.2, 0.0]], rtol=1e-15)


def test_repulsive_two_point(orc):
    # S:L332 two points at distance 1: Z = 1, F_rep[1] = -f/Z = (0.25, 0)... pointing away
    Y = np.array([[0, 0], [1, 0]], np.float32)
    f, z, Z, _ = orc.repulsive_bh(Y, 0.5)
    assert Z == 1.0
    np.testing.assert_allclose(f[0], [-0.25, 0.0])          # (y_1 - y_2) / (1 + 1)^2
    np.testing.assert_allclose(-f[0] / Z, [0.25, 0.0])      # F_rep[1] = -f/Z


def _dense_P(N, seed=0):
    rng = np.random.default_rng(seed)
    M = rng.random((N, N))
    M = M + M.T
    np.fill_diagonal(M, 0)
    M /= M.sum()
    rp = np.arange(0, N * (N - 1) + 1, N - 1, dtype=np.int64)
    col = np.array([j for i in range(N) for j in range(N) if j != i], np.int32)
    val = np.array([M[i, j] for i in range(N) for j in range(N) if j != i])
    return M, rp, col, val


def test_exact_gradient_is_kl_derivative(orc):
    # acceptance criterion 2: Eq. 3 (Z restored, D1) vs central differences of KL
    N = 64
    for seed in range(5):
        M, rp, col, val = _dense_P(N, seed)
        Y = np.random.default_rng(100 + seed).normal(size=(N, 2)) * 2
        g, Z = orc.gradient_exact(rp, col, val, Y)
        h = 1e-5
        fd = np.empty_like(g)
        for i in range(N):
            for a in range(2):
                Yp = Y.copy(); Yp[i, a] += h
                Ym = Y.copy(); Ym[i, a] -= h
                fd[i, a] = (orc.kl(rp, col, val, Yp) - orc.kl(rp, col, val, Ym)) / (2 * h)
        assert np.linalg.norm(g - fd) / np.linalg.norm(g) < 1e-6


def test_exact_gradient_vs_sklearn(orc):
    from scipy.spatial.distance import squareform
    from sklearn.manifold._t_sne import _kl_divergence
    N = 50
    M, rp, col, val = _dense_P(N, 7)
    Y = np.random.default_rng(8).normal(size=(N, 2))
    g, Z = orc.gradient_exact(rp, col, val, Y)
    kl_s, g_s = _kl_divergence(Y.ravel().copy(), squareform(M, checks=False), 1, N, 2)
    np.testing.assert_allclose(g.ravel(), g_s, rtol=1e-9, atol=1e-12)
    assert abs(orc.kl(rp, col, val, Y) - kl_s) < 1e-9


def test_bh_theta0_equals_exact_gradient(orc):
    # survey 8(c): theta = 0 BH gradient == O11 exact gradient (N <= 500)
    N = 400
    rp, col, v32, v64 = synth.random_csr(N, 12, seed=1)
    Y = synth.fixed_y("gauss10", N, seed=2)
    for exag in (1.0, 12.0):
        g_bh, Z_bh = orc.gradient_bh(rp, col, v32, Y, 0.0, exag)
        g_ex, Z_ex = orc.gradient_exact(rp, col, v32.astype(np.float64), Y.astype(np.float64), exag)
        assert abs(Z_bh - Z_ex) <= 1e-12 * Z_ex
        assert np.linalg.norm(g_bh - g_ex) / np.linalg.norm(g_ex) < 1e-12


def test_gradient_invariants(orc):
    N = 300
    rp, col, v32, v64 = synth.random_csr(N, 10, seed=4)
    Y = synth.fixed_y("gauss10", N, seed=9)
    g, _ = orc.gradient_bh(rp, col, v32, Y, 0.0)
    assert np.abs(g.sum(0)).max() < 1e-12 * np.abs(g).sum()          # S:L358 action-reaction
    # translation invariance; use a dyadic shift so Y+c stays exact in fp32
    g2, _ = orc.gradient_bh(rp, col, v32, Y + np.float32(64.0), 0.5)
    g1, _ = orc.gradient_bh(rp, col, v32, Y, 0.5)
    assert np.linalg.norm(g2 - g1) / np.linalg.norm(g1) < 1e-4
    # n = 2, P12 = 1/2 -> p = q -> gradient exactly 0
    g0, _ = orc.gradient_bh(np.array([0, 1, 2]), np.array([1, 0]),
                            np.array([0.5, 0.5], np.float32),
                            np.array([[0, 0], [3, 1]], np.float32), 0.5)
    assert np.abs(g0).max() < 1e-17


def test_kl_nonneg_and_zero(orc):
    # S:L352 P = Q -> KL = 0 (n = 2); Gibbs: KL >= 0 for dense P
    rp, col = np.array([0, 1, 2]), np.array([1, 0])
    val = np.array([0.5, 0.5])
    assert abs(orc.kl(rp, col, val, np.array([[0.0, 0.0], [1.0, 2.0]]))) < 1e-15
    M, rp, col, val = _dense_P(40, 3)
    assert orc.kl(rp, col, val, np.random.default_rng(0).normal(size=(40, 2))) > 0
