"""f2: IVF-PQ kNN on the GPU (tsne_ivfpq_build / _search)
against the oracle's search on the same index (O13), the index against the
definitions of its quantisers, and recall@K against the exact kNN (U1)."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import paper_1807_11824_b200 as T
    T.lib()
    return T


@pytest.fixture(scope="module")
def built(T):
    X = synth.make_x("C2", n=6000)
    Xd = X.to("cuda")
    ix = T.IvfPQ(Xd)
    P = {k: (v.cpu().numpy() if torch.is_tensor(v) else v) for k, v in ix.parts().items()}
    return X.numpy(), Xd, ix, P


def test_index_structure(built):
    X, Xd, ix, P = built
    N = X.shape[0]
    assert ix.nlist == round(N ** 0.5) and ix.m * ix.dsub == ix.Dp >= X.shape[1]
    off, ids = P["list_offsets"], P["list_ids"]
    assert off[0] == 0 and off[-1] == N and (np.diff(off) >= 0).all()
    assert np.array_equal(np.sort(ids), np.arange(N))
    for L in range(ix.nlist):                    # list entries in point order
        assert (np.diff(ids[off[L]:off[L + 1]]) > 0).all()


def test_lists_and_codes_follow_their_definitions(built):
    # q1: each point is in the list of its nearest centroid; q2: each code is the
    # nearest codeword of its residual sub-vector (fp64 here; fp32 GEMM distances
    # on the GPU, so near-ties may differ: at most 0.2% of the decisions)
    X, Xd, ix, P = built
    N, D = X.shape
    Xp = np.zeros((N, ix.Dp)); Xp[:, :D] = X
    C = P["centroids"].astype(np.float64)
    list_of = np.empty(N, np.int64)
    for L in range(ix.nlist):
        list_of[P["list_ids"][P["list_offsets"][L]:P["list_offsets"][L + 1]]] = L
    d = (Xp ** 2).sum(1)[:, None] + (C ** 2).sum(1)[None] - 2 * Xp @ C.T
    assert np.mean(np.argmin(d, 1) == list_of) > 0.998
    codes = np.empty((N, ix.m), np.int64)
    codes[P["list_ids"]] = P["codes"]
    R = Xp - C[list_of]
    cb = P["codebooks"].astype(np.float64)
    agree = 0
    for j in range(ix.m):
        sub = R[:, j * ix.dsub:(j + 1) * ix.dsub]
        dj = (sub ** 2).sum(1)[:, None] + (cb[j] ** 2).sum(1)[None] - 2 * sub @ cb[j].T
        agree += np.sum(np.argmin(dj, 1) == codes[:, j])
    assert agree / (N * ix.m) > 0.998


def test_search_matches_oracle_on_the_same_index(T, orc, built):
    X, Xd, ix, P = built
    N = X.shape[0]
    K, tau = 30, 6
    Kc = min(480, ((K + max(64, 5 * K) + 31) // 32) * 32)
    idx, d2 = ix.search(Xd, K, tau)
    idx, d2 = idx.cpu().numpy(), d2.cpu().numpy()
    list_of = np.empty(N, np.int32)
    for L in range(ix.nlist):
        list_of[P["list_ids"][P["list_offsets"][L]:P["list_offsets"][L + 1]]] = L
    codes = np.empty((N, ix.m), np.uint8)
    codes[P["list_ids"]] = P["codes"]
    io, do = orc.ivfpq_search(X, P["centroids"], P["codebooks"], list_of, codes, K, tau, Kc)
    same = np.all(idx == io, axis=1)
    # rows may differ only through near-ties of the fp32 look-up-table distances
    # at the probe or candidate boundary
    assert same.mean() > 0.99, same.mean()
    np.testing.assert_allclose(d2[same], do[same], rtol=1e-10, atol=0)
    assert (idx >= 0).all()


def test_recall_against_exact_knn(T):
    # SPEC S:L135's example shape (10k points, k = 32, tau = 10 -> recall >= 0.8),
    # on MNIST-shaped data; recall non-decreasing in tau
    X = synth.make_x("C2", n=10000, device="cuda")
    ex, _, _ = T.knn(X, 32)
    ex = ex.cpu().numpy()
    for kw in ({}, {"kprime": 96}):
        ix = T.IvfPQ(X, **kw)
        r = []
        for tau in (1, 4, 10, 32):
            idx, d2 = ix.search(X, 32, tau)
            idx = idx.cpu().numpy()
            r.append(np.mean([len(set(a) & set(b)) / 32 for a, b in zip(idx, ex)]))
        print("recall@32 at tau 1/4/10/32:", kw, r)
        if not kw:
            rec = r
    assert all(a <= b + 1e-9 for a, b in zip(rec, rec[1:])), rec
    assert rec[2] >= 0.8, rec          # defaults: m = min(96, D/8), K' = K + 5K


def test_run_with_ivfpq_knn(T, orc):
    # tsne_run_ex with the approximate kNN (knn_tau): the embedding's quality
    # against the exact-kNN pipeline on the same data (exact-Z KL of P_exact)
    X = synth.make_x("C2", n=8000)
    Xh = X.pin_memory()
    Ya, ia = T.run(Xh, perplexity=30.0, n_iter=500, knn_tau=16)
    Ye, ie = T.run(Xh, perplexity=30.0, n_iter=500)
    assert torch.isfinite(Ya).all() and ia["nnz"] > 0
    idx, d2 = orc.knn(X.numpy(), 90)
    rp, col, v64, v32, *_ = orc.compute_p(idx, d2, 30.0)
    kla = orc.kl(rp, col, v32, Ya.numpy().astype(np.float64))
    kle = orc.kl(rp, col, v32, Ye.numpy().astype(np.float64))
    print("KL (exact P) of the IVF-PQ run %.4f vs exact-kNN run %.4f" % (kla, kle))
    assert kla < 1.15 * kle
