"""Pins for the oracle's O1 (kNN), O2 (calibration) and O3 (symmetrisation).

Each check is against something other than the oracle itself: SPEC's
hand examples, closed forms, invariants, and scikit-learn's independent
routines.
"""
import numpy as np
import pytest

import synth


# ------------------------------------------------------------------ O1 kNN
def test_knn_collinear_spec_example(orc):
    # S:L113 "3 collinear points at x=0,1,3 with k=1 -> 0->1, 1->0, 2->1"
    X = np.array([[0.0], [1.0], [3.0]], np.float32)
    idx, d2 = orc.knn(X, 1)
    assert idx[:, 0].tolist() == [1, 0, 1]
    assert d2[:, 0].tolist() == [1.0, 1.0, 4.0]


def test_knn_duplicate_tie_lower_index(orc):
    # S:L114 identical duplicates: distance 0, lower index wins the tie
    X = np.array([[5.0, 5.0], [1.0, 1.0], [5.0, 5.0], [5.0, 5.0]], np.float32)
    idx, d2 = orc.knn(X, 2)
    assert idx[0].tolist() == [2, 3] and d2[0].tolist() == [0.0, 0.0]
    assert idx[3].tolist() == [0, 2]
    # equal distances resolve by index: point 1 is equidistant from 0, 2, 3
    assert idx[1].tolist() == [0, 2]


def test_knn_separated_clusters(orc):
    # S:L115 well separated Gaussians: every neighbour shares the query's label
    X, lab = synth.make_x("C1", n=200, return_labels=True)
    idx, _ = orc.knn(X.numpy(), 5)
    lab = lab.numpy()
    assert (lab[idx] == lab[:, None]).all()


def test_knn_matches_sklearn_bruteforce(orc):
    from sklearn.neighbors import NearestNeighbors
    X = synth.make_x("C2", n=600).numpy()
    K = 20
    idx, d2 = orc.knn(X, K)
    nn = NearestNeighbors(n_neighbors=K + 1, algorithm="brute").fit(X.astype(np.float64))
    dist, ind = nn.kneighbors(X.astype(np.float64))
    # drop self (distance 0 in column 0 for distinct points)
    dist, ind = dist[:, 1:], ind[:, 1:]
    np.testing.assert_allclose(d2, dist ** 2, rtol=1e-9, atol=1e-9)
    same = ind == idx
    if not same.all():   # only near-ties may differ
        r, c = np.nonzero(~same)
        for a, b in zip(r, c):
            da, db = d2[a, c], dist[a, c] ** 2
            assert abs(da - db) <= 1e-6 * max(da, db)


def test_knn_permutation_equivariance(orc):
    # S:L138 permuting rows permutes the graph
    X = synth.make_x("C1", n=300).numpy()
    perm = np.random.default_rng(0).permutation(300)
    inv = np.argsort(perm)
    idx, d2 = orc.knn(X, 8)
    idx_p, d2_p = orc.knn(X[perm], 8)
    np.testing.assert_array_equal(d2_p, d2[perm])
    # neighbour sets agree after relabelling (order may only differ on exact ties)
    assert all(set(perm[idx_p[a]]) == set(idx[perm[a]]) for a in range(300))


def test_knn_rows_subset_equals_full(orc):
    X = synth.make_x("C3", n=300).numpy()
    idx, d2 = orc.knn(X, 10)
    rows = np.array([0, 17, 299])
    i2, e2 = orc.knn(X, 10, rows=rows)
    np.testing.assert_array_equal(i2, idx[rows])
    np.testing.assert_array_equal(e2, d2[rows])


# ------------------------------------------------------------------ O2 calibration
def _entropy_nats(p):
    q = p[p > 0]
    return float(-(q * np.log(q)).sum())


def test_calibrate_entropy_and_mass():
    import oracle as orc
    rng = np.random.default_rng(1)
    for _ in range(200):
        K = int(rng.integers(10, 151))
        perp = float(rng.uniform(2.0, K - 1.0))
        d = np.sort(rng.gamma(2.0, 3.0, K) + rng.uniform(0, 50))
        p, beta, flag, it = orc.calibrate_row(d, perp)
        assert flag == 0
        assert abs(p.sum() - 1.0) <= 1e-12
        # independent entropy formula -sum p ln p against the target ln(perp)
        assert abs(_entropy_nats(p) - np.log(perp)) <= 1e-9
        # the north-star bound
        assert abs(_entropy_nats(p) - np.log(perp)) <= 1e-5
        # Eq. 1 shape: p_j proportional to exp(-beta d_j), monotone in d
        assert np.all(np.diff(p) <= 1e-15)


def test_calibrate_spec_examples(orc):
    # S:L186 equidistant neighbours -> uniform (degenerate, any sigma admissible)
    p, beta, flag, _ = orc.calibrate_row(np.array([2.0, 2.0, 2.0]), 2.5)
    np.testing.assert_allclose(p, [1 / 3] * 3, rtol=0, atol=1e-15)
    assert flag == 1
    # S:L188 distances (1,4,9,16), perplexity 2: plug beta back into Eq. 1
    d = np.array([1.0, 4.0, 9.0, 16.0])
    p, beta, flag, _ = orc.calibrate_row(d, 2.0)
    q = np.exp(-beta * d)
    q /= q.sum()
    np.testing.assert_allclose(p, q, rtol=1e-12)
    assert abs(np.exp(_entropy_nats(q)) - 2.0) <= 1e-9
    # ties at the minimum beyond perplexity: uniform over the ties (D3)
    p, beta, flag, _ = orc.calibrate_row(np.array([1.0, 1.0, 1.0, 5.0, 9.0]), 2.0)
    assert flag == 1 and np.isinf(beta)
    np.testing.assert_allclose(p, [1 / 3, 1 / 3, 1 / 3, 0, 0])


def test_calibrate_scale_invariance(orc):
    # S:L213 d -> c d leaves p unchanged and maps beta -> beta / c
    rng = np.random.default_rng(2)
    for _ in range(50):
        d = np.sort(rng.uniform(1, 10, 90))
        c = float(rng.uniform(0.01, 100))
        p1, b1, _, _ = orc.calibrate_row(d, 30.0)
        p2, b2, _, _ = orc.calibrate_row(c * d, 30.0)
        np.testing.assert_allclose(p1, p2, rtol=1e-8, atol=1e-14)
        assert abs(b2 * c / b1 - 1) < 1e-8


def test_calibrate_vs_sklearn(orc):
    # sklearn's independent bisection (nats, stops at |dH| <= 1e-5): agree to its stop
    from sklearn.manifold._utils import _binary_search_perplexity
    X = synth.make_x("C2", n=400).numpy()
    idx, d2 = orc.knn(X, 90)
    P, beta, flags = orc.calibrate(d2, 30.0)
    Ps = _binary_search_perplexity(d2.astype(np.float32), 30.0, 0)
    rel = np.abs(P - Ps) / np.maximum(P, 1e-300)
    big = P > 1e-6
    assert rel[big].max() < 3e-3       # sklearn: fp32 distances + 1e-5 entropy stop
    assert np.abs(P - Ps).max() < 1e-5


# ------------------------------------------------------------------ O3 symmetrise
def test_symmetrize_two_points(orc):
    # S:L196 n=2 mutual, p=1 each way -> P12 = P21 = (1+1)/(2*2) = 0.5
    rp, col, v64, v32 = orc.symmetrize(np.array([[1], [0]]), np.array([[1.0], [1.0]]))
    assert rp.tolist() == [0, 1, 2] and col.tolist() == [1, 0]
    assert v64.tolist() == [0.5, 0.5]


def test_symmetrize_asymmetric_edge(orc):
    # S:L197 j in kNN(i) but not vice versa -> P_ij = p_{j|i}/2n on both rows
    idx = np.array([[1], [2], [1]])
    pc = np.array([[1.0], [1.0], [1.0]])
    rp, col, v64, _ = orc.symmetrize(idx, pc)
    n = 3
    P = np.zeros((n, n))
    for i in range(n):
        P[i, col[rp[i]:rp[i + 1]]] = v64[rp[i]:rp[i + 1]]
    assert P[0, 1] == P[1, 0] == 1.0 / 6
    assert P[1, 2] == P[2, 1] == 2.0 / 6


def test_symmetrize_invariants(orc):
    X = synth.make_x("C1", n=1000).numpy()
    K = 90
    idx, d2 = orc.knn(X, K)
    rp, col, v64, v32, P_cond, beta, flags = orc.compute_p(idx, d2, 30.0)
    N = 1000
    nnz = rp[-1]
    assert N * K <= nnz <= 2 * N * K
    assert abs(v64.sum() - 1.0) <= 1e-12
    # sorted, unique columns, no diagonal
    for i in range(0, N, 37):
        c = col[rp[i]:rp[i + 1]]
        assert np.all(np.diff(c) > 0) and i not in c
    # bitwise symmetry of the fp32 values
    import scipy.sparse as sp
    A = sp.csr_matrix((v32, col, rp), shape=(N, N))
    D = (A - A.T)
    assert D.nnz == 0 or np.abs(D.data).max() == 0.0
    # dense cross-check of the definition p_ij = (p_{j|i} + p_{i|j}) / 2N
    Pc = np.zeros((N, N))
    for i in range(N):
        Pc[i, idx[i]] = P_cond[i]
    Pd = (Pc + Pc.T) / (2 * N)
    np.testing.assert_allclose(A.toarray(), Pd.astype(np.float32), rtol=0, atol=0)
