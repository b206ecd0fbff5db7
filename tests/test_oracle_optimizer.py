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
