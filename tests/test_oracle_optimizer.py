"""Pins for the oracle's optimiser (O9-O10) and full run.

The update rule and schedule are not in the paper (D12-D16); the long run is
chaotic, so it is pinned only by invariants (fixed point, recentring, KL
descent, cluster recovery) -- 'parity unpinned beyond invariants' in
DESIGN.md section 5.
"""
import numpy as np

import synth


def test_zero_gradient_fixed_point(orc):
    # S:L409 n = 2 with P12 = 1/2 -> gradient 0 -> coordinates unchanged (mean 0 already)
    rp, col, val = np.array([0, 1, 2]), np.array([1, 0]), np.array([0.5, 0.5], np.float32)
    Y0 = np.array([[-1.0, 0.5], [1.0, -0.5]])
    Y, v, g = orc.optimize(rp, col, val, Y0, n_iter=5, exaggeration=1.0)
    np.testing.assert_array_equal(Y, Y0)
    assert np.all(v == 0)


def test_first_step_closed_form_and_recentring(orc):
    # one step from v = 0, gains = 1: sign(v) = 0 != sign(g) -> gain 1.2 (D12),
    # v = -eta 1.2 g, y' = y + v, then minus the mean
    N = 200
    rp, col, v32, _ = synth.random_csr(N, 8, seed=2)
    Y0 = synth.fixed_y("gauss10", N, seed=3).astype(np.float64)
    g, _ = orc.gradient_bh(rp, col, v32, Y0.astype(np.float32), 0.5, 12.0)
    Y, v, gains = orc.optimize(rp, col, v32, Y0, n_iter=1, theta=0.5, eta=200.0, exaggeration=12.0)
    assert np.all(gains[g != 0] == 1.2)
    Yexp = Y0 - 200.0 * 1.2 * g
    Yexp -= Yexp.mean(0)
    np.testing.assert_allclose(Y, Yexp, rtol=1e-12, atol=1e-9)
    assert np.abs(Y.mean(0)).max() < 1e-12


def test_c1_run_descends_and_recovers_clusters(orc):
    # S:L424 KL(final) < KL(after exaggeration + 50); S:L419 cluster recovery
    from sklearn.cluster import KMeans
    from scipy.optimize import linear_sum_assignment
    X, lab = synth.make_x("C1", return_labels=True)
    X = X.numpy(); lab = lab.numpy()
    N = X.shape[0]
    idx, d2 = orc.knn(X, 90)
    rp, col, v64, v32, *_ = orc.compute_p(idx, d2, 30.0)
    Y = orc.init_y(N, 42)
    Y, v, g = orc.optimize(rp, col, v32, Y, n_iter=300, theta=0.5)
    kl300 = orc.kl(rp, col, v32, Y)
    Y, v, g = orc.optimize(rp, col, v32, Y, v, g, t0=300, n_iter=700, theta=0.5)
    kl1000 = orc.kl(rp, col, v32, Y)
    assert kl1000 < kl300
    assert np.isfinite(Y).all() and np.abs(Y).max() < 1e6
    km = KMeans(10, n_init=5, random_state=0).fit(Y)
    C = np.zeros((10, 10))
    for a, b in zip(lab, km.labels_):
        C[a, b] += 1
    r, c = linear_sum_assignment(-C)
    assert C[r, c].sum() / N >= 0.95
    nnp = orc.nn_preservation(idx, Y, 10)
    assert 0.2 < nnp <= 1.0


def test_init_y_distribution(orc):
    Y = orc.init_y(20000, 42)
    assert abs(Y.mean()) < 3 * 1e-4 / np.sqrt(40000) * 1.5
    assert abs(Y.std() / 1e-4 - 1) < 0.03
    np.testing.assert_array_equal(Y, orc.init_y(20000, 42))
    assert not np.array_equal(Y, orc.init_y(20000, 43))


def test_philox_known_answers(orc):
    # Random123 known-answer vectors for Philox4x32-10 (D14)
    kat = [([0, 0, 0, 0], [0, 0], [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]),
           ([0xffffffff] * 4, [0xffffffff] * 2, [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]),
           ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0],
            [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1])]
    for c, k, o in kat:
        assert orc.philox4x32_10(c, k).tolist() == o


def test_nn_preservation_identity(orc):
    # metrics example: embedding = the 2-D data itself -> preservation 1.0
    Y = synth.fixed_y("gauss10", 300, seed=1)
    idx, _ = orc.knn(Y, 10)
    assert orc.nn_preservation(idx, Y.astype(np.float64), 10) == 1.0


def _two_point_grad(Y, alpha, p):
    """Closed form of Eq. 7 for N = 2 with P_12 = P_21 = p (Eqs. 4-6 by hand):
    w = 1/(1 + |y1 - y2|^2), Z = 2w, A_1 = p w (y1 - y2), F_rep,1 = -w^2 (y1 - y2) / Z
    -> g_1 = 4 w (alpha p - 1/2) (y1 - y2), g_2 = -g_1."""
    d = Y[0] - Y[1]
    w = 1.0 / (1.0 + d @ d)
    g1 = 4.0 * w * (alpha * p - 0.5) * d
    return np.array([g1, -g1])


def test_two_steps_across_exaggeration_switch(orc):
    """O9-O10 pinned across t = 249 -> 250 (D12, D13): the step at t = 249
    uses alpha = exag and mu = mom0, the step at t = 250 alpha = 1 and mu = mom1;
    both gain branches (signs differ -> +0.2, same sign -> x0.8, sign(0) = 0), the
    min_gain floor, v != 0, and the recentring are exercised.  Fails under
    `t <= exag_iters`, swapped momenta, swapped gain branches or a missing floor
    (each checked by a temporary mutation of the oracle)."""
    p, eta, exag, mom0, mom1, floor_ = 0.25, 0.01, 12.0, 0.5, 0.8, 0.01
    rp, col, val = np.array([0, 1, 2]), np.array([1, 0]), np.array([p, p], np.float32)
    Y0 = np.array([[-0.75, 0.0], [0.5, 0.0]])
    v0 = np.array([[0.3, 0.0], [0.1, 0.0]])
    g0 = np.array([[1.0, 0.011], [0.5, 0.011]])
    # expected, by the rule written out
    Y, v, gains = Y0.copy(), v0.copy(), g0.copy()
    branches = set()
    for t in (249, 250):
        alpha, mu = (exag, mom0) if t < 250 else (1.0, mom1)
        g = _two_point_grad(Y, alpha, p)
        for a in range(2):
            for c in range(2):
                differ = np.sign(g[a, c]) != np.sign(v[a, c])
                branches.add((t, bool(differ)))
                gn = gains[a, c] + 0.2 if differ else gains[a, c] * 0.8
                gains[a, c] = max(gn, floor_)
                v[a, c] = mu * v[a, c] - eta * gains[a, c] * g[a, c]
                Y[a, c] = Y[a, c] + v[a, c]
        Y -= Y.mean(0)
    assert branches == {(249, True), (249, False), (250, True), (250, False)}
    assert gains[0, 1] == floor_ and gains[1, 1] == floor_
    Yo, vo, go = orc.optimize(rp, col, val, Y0, v0, g0, t0=249, n_iter=2, theta=0.5, eta=eta,
                              exaggeration=exag, exag_iters=250, mom0=mom0, mom1=mom1,
                              min_gain=floor_)
    np.testing.assert_allclose(go, gains, rtol=1e-14)
    np.testing.assert_allclose(vo, v, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(Yo, Y, rtol=1e-12, atol=1e-15)


def test_nn_preservation_hand_example(orc):
    """O12 10-NN preservation on a hand-worked case with value != 1:
    mean_i |NN_k^X(i) & NN_k^Y(i)| / k, NN^Y a brute-force 2-D kNN excluding i,
    ties by index, NN^X the first k entries of rows of stride Kx.
    Y on a line: 0, 1, 3, 3, 10 (points 2 and 3 coincide).  k = 2:
      NN^Y(0) = {1, 2}  (d 1; d 9 tie with 3 -> lower index 2)
      NN^Y(1) = {0, 2}  (d 1, 4; tie 2/3 -> 2)
      NN^Y(2) = {3, 1}  (d 0, 4)
      NN^Y(3) = {2, 1}  (d 0, 4)
      NN^Y(4) = {2, 3}  (d 49, 49)
    NN^X rows (first 2 of 3): {1,3}, {0,3}, {4,0}, {2,1}, {0,1}
    overlaps 1, 1, 0, 2, 0 -> (1+1+0+2+0) / (5*2) = 0.4 (ties taken by the higher
    index would give 2, 2, 0, 2, 0 -> 0.6; i counted as its own neighbour, less)."""
    Y = np.array([[0, 0], [1, 0], [3, 0], [3, 0], [10, 0]], np.float64)
    idx_x = np.array([[1, 3, 4], [0, 3, 4], [4, 0, 1], [2, 1, 0], [0, 1, 2]], np.int32)
    assert abs(orc.nn_preservation(idx_x, Y, 2) - 0.4) < 1e-15
    # k = 1: NN^Y = 1, 0, 3, 2, 2; NN^X = 1, 0, 4, 2, 0 -> 3/5
    assert abs(orc.nn_preservation(idx_x, Y, 1) - 0.6) < 1e-15


def test_nn_preservation_rows_hand_example(orc):
    """The sampled form of O12 on the hand-worked case above: per-point overlaps
    1, 1, 0, 2, 0 (k = 2), so rows {0, 3} give (1 + 2) / (2 * 2) = 0.75 and
    rows {2, 4} give 0; all rows reproduce the full mean."""
    Y = np.array([[0, 0], [1, 0], [3, 0], [3, 0], [10, 0]], np.float64)
    idx_x = np.array([[1, 3, 4], [0, 3, 4], [4, 0, 1], [2, 1, 0], [0, 1, 2]], np.int32)
    assert abs(orc.nn_preservation(idx_x, Y, 2, rows=[0, 3]) - 0.75) < 1e-15
    assert orc.nn_preservation(idx_x, Y, 2, rows=[2, 4]) == 0.0
    assert abs(orc.nn_preservation(idx_x, Y, 2, rows=np.arange(5)) - 0.4) < 1e-15
