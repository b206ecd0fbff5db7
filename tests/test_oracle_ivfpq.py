"""Pins of the oracle's IVF-PQ search (O13; Alg. 1 line 1) on
hand-built indexes, against what the definition fixes:
an exhaustive probe with a memorising codebook is exact kNN; one probe on
well-separated clusters stays in the query's cell; recall grows with tau."""
import numpy as np

import synth


def nearest(points, cents):
    d = ((points[:, None, :].astype(np.float64) - cents[None, :, :].astype(np.float64)) ** 2).sum(-1)
    return np.argmin(d, axis=1).astype(np.int32)        # ties: lowest index (argmin)


def memorising_index(X, cents):
    """m = 1 sub-quantiser over all D dims whose 256 codewords are the residuals
    themselves (N <= 256): q(y) = y exactly."""
    N, D = X.shape
    list_of = nearest(X, cents)
    cb = np.full((1, 256, D), 1e6, np.float32)
    cb[0, :N] = X - cents[list_of]
    codes = np.arange(N, dtype=np.uint8)[:, None]
    return cents.astype(np.float32), cb, list_of, codes


def test_exhaustive_probe_with_exact_codes_is_exact_knn(orc):
    rng = np.random.default_rng(1)
    X = rng.normal(0, 1, (200, 8)).astype(np.float32)
    cents = X[[0, 50, 100, 150]].copy()
    cent, cb, list_of, codes = memorising_index(X, cents)
    for K in (1, 5, 20):
        i1, d1 = orc.ivfpq_search(X, cent, cb, list_of, codes, K, tau=4, Kc=K + 10)
        i0, d0 = orc.knn(X, K)
        assert np.array_equal(i1, i0)
        np.testing.assert_allclose(d1, d0, rtol=1e-12, atol=0)


def test_one_probe_stays_in_the_query_cell(orc):
    rng = np.random.default_rng(2)
    means = np.array([[0, 0, 0, 0], [100, 0, 0, 0], [0, 100, 0, 0], [0, 0, 100, 0]], np.float32)
    X = np.concatenate([m + rng.normal(0, 1, (60, 4)) for m in means]).astype(np.float32)
    cent, cb, list_of, codes = memorising_index(X, means)
    idx, d2 = orc.ivfpq_search(X, cent, cb, list_of, codes, 10, tau=1, Kc=20)
    assert (idx >= 0).all()
    assert (list_of[idx] == list_of[:, None]).all()


def test_recall_monotone_in_tau(orc):
    # a coarse (16 cells) and lossy (32 codewords per sub-vector, 4 sub-vectors)
    # index of a Gaussian mixture; recall@10 vs exact kNN, means over 3 seeds
    recalls = {1: [], 4: [], 16: []}
    for seed in range(3):
        X = synth.make_x("C1", n=600, seed=10 + seed).numpy()[:, :16].copy()
        rng = np.random.default_rng(seed)
        cents = X[rng.choice(600, 16, replace=False)]
        list_of = nearest(X, cents)
        R = (X - cents[list_of]).astype(np.float32)
        cb = np.full((4, 256, 4), 1e6, np.float32)
        codes = np.empty((600, 4), np.uint8)
        for j in range(4):
            sub = R[:, 4 * j:4 * j + 4]
            cb[j, :32] = sub[rng.choice(600, 32, replace=False)]
            codes[:, j] = nearest(sub, cb[j, :32])
        ex, _ = orc.knn(X, 10)
        for tau in recalls:
            idx, _ = orc.ivfpq_search(X, cents, cb, list_of, codes, 10, tau=tau, Kc=40)
            rec = np.mean([len(set(a) & set(b)) / 10 for a, b in zip(idx, ex)])
            recalls[tau].append(rec)
    r = [np.mean(recalls[t]) for t in (1, 4, 16)]
    assert r[0] <= r[1] <= r[2] and r[2] > 0.9, r
