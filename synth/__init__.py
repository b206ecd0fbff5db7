"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only draws inputs (the
high-dimensional data X, fixed embeddings Y for gradient parity) with the
shapes and value distributions of the paper's workloads.  The recipe is the
one in DESIGN.md section 4:

  x = post(mu_label + s * eps),  eps ~ N(0, I), rows shuffled by a seeded
  permutation so that clusters are not contiguous in memory.

Generation uses ``torch`` generators; the same (config, n, seed, device)
always gives the same bytes.  Tests generate on the CPU and copy to the GPU;
bench.py generates the 10.5 GB C5 matrix on the GPU and copies sampled rows
to the host for the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass(frozen=True)
class Config:
    name: str
    N: int
    D: int
    clusters: int
    sizes: str          # "equal" | "zipf"
    mu: str             # "uniform(a,b)" | "ink" | "normal(sd)"
    s: float
    post: str           # "identity" | "clip01" | "relu"
    perplexity: float
    seed: int
    paper: str          # PAPER.md passage the shape follows


CONFIGS = {
    "C1": Config("C1-synth", 1000, 50, 10, "equal", "uniform(0,10)", 1.0, "identity", 30.0, 1,
                 "P:L177 synthetic Gaussian clusters, 50-D"),
    "C2": Config("C2-mnist-shaped", 70000, 784, 10, "equal", "ink", 0.2, "clip01", 30.0, 2,
                 "P:L179 MNIST 60k+10k x 784"),
    "C3": Config("C3-cifar-shaped", 50000, 3072, 10, "equal", "uniform(0.3,0.6)", 0.25, "clip01",
                 30.0, 3, "P:L181 CIFAR-10 50k x 3072"),
    "C4": Config("C4-glove-shaped", 400000, 300, 2000, "zipf", "normal(0.3)", 0.35, "identity",
                 50.0, 4, "P:L626 GloVe x 300 (400k vocabulary)"),
    "C5": Config("C5-imagenet-resnet-shaped", 1281167, 2048, 1000, "equal", "normal(0.5)", 0.5,
                 "relu", 30.0, 5, "P:L35 ImageNet ResNet-200 codes 1.2M x 2048"),
}


def cluster_sizes(N: int, C: int, kind: str) -> np.ndarray:
    C = max(1, min(C, N))
    if kind == "equal":
        sizes = np.full(C, N // C, np.int64)
        sizes[: N % C] += 1
        return sizes
    w = 1.0 / np.arange(1, C + 1, dtype=np.float64)          # Zipf(1.0)
    sizes = np.maximum(1, np.floor(N * w / w.sum())).astype(np.int64)
    rem = N - int(sizes.sum())
    k = 0
    while rem != 0:                                            # hand out / take back the remainder
        step = 1 if rem > 0 else -1
        if step > 0 or sizes[k % C] > 1:
            sizes[k % C] += step
            rem -= step
        k += 1
    return sizes


def _mu(cfg: Config, C: int, D: int, g: torch.Generator, device) -> torch.Tensor:
    kind = cfg.mu
    if kind.startswith("uniform"):
        a, b = (float(t) for t in kind[8:-1].split(","))
        return a + (b - a) * torch.rand(C, D, generator=g, device=device)
    if kind == "ink":                                          # U[0,1] masked by Bernoulli(0.2)
        u = torch.rand(C, D, generator=g, device=device)
        m = (torch.rand(C, D, generator=g, device=device) < 0.2).float()
        return u * m
    if kind.startswith("normal"):
        sd = float(kind[7:-1])
        return sd * torch.randn(C, D, generator=g, device=device)
    raise ValueError(kind)


def make_x(cfg: Config | str, n: int | None = None, seed: int | None = None, device="cpu",
           chunk: int = 32768, return_labels: bool = False):
    """Generate X (n x D float32, row-major) for a config shape."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    N = cfg.N if n is None else int(n)
    D = cfg.D
    seed = cfg.seed if seed is None else int(seed)
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    sizes = cluster_sizes(N, cfg.clusters, cfg.sizes)
    C = len(sizes)
    mu = _mu(cfg, C, D, g, device)
    labels = torch.repeat_interleave(torch.arange(C, device=device),
                                     torch.as_tensor(sizes, device=device))
    perm = torch.randperm(N, generator=g, device=device)
    labels = labels[perm]
    X = torch.empty(N, D, dtype=torch.float32, device=device)
    for a in range(0, N, chunk):
        b = min(N, a + chunk)
        x = mu[labels[a:b]] + cfg.s * torch.randn(b - a, D, generator=g, device=device)
        if cfg.post == "clip01":
            x.clamp_(0.0, 1.0)
        elif cfg.post == "relu":
            x.clamp_(min=0.0)
        X[a:b] = x
    if return_labels:
        return X, labels
    return X


def fixed_y(kind: str, N: int, seed: int = 7, labels=None) -> np.ndarray:
    """Fixed embeddings for single-step gradient parity:
    'gauss10' = 10 N(0, I); 'clustered' = 30 mu_label + N(0, I);
    'tiny' = 1e-4 N(0, I) (the optimiser's start)."""
    g = torch.Generator().manual_seed(seed)
    if kind == "gauss10":
        Y = 10.0 * torch.randn(N, 2, generator=g)
    elif kind == "tiny":
        Y = 1e-4 * torch.randn(N, 2, generator=g)
    elif kind == "clustered":
        if labels is None:
            labels = torch.randint(0, 10, (N,), generator=g)
        labels = torch.as_tensor(labels)
        C = int(labels.max()) + 1
        mu = torch.randn(C, 2, generator=g)
        Y = 30.0 * mu[labels] + torch.randn(N, 2, generator=g)
    elif kind == "blobs":                                     # many small blobs (deep trees)
        C = max(1, N // 100)
        lab = torch.randint(0, C, (N,), generator=g)
        mu = 50.0 * torch.randn(C, 2, generator=g)
        Y = mu[lab] + 0.5 * torch.randn(N, 2, generator=g)
    elif kind.startswith("collapsed"):
        # a transient collapse of the exaggeration phase: the blobs of 'blobs'
        # plus N // 9 points packed into a 6 x 6 patch of adjacent finest
        # (level-24) cells near the origin, so the tree holds 36 neighbouring
        # buckets of ~N/324 points each (exact pairs with every bucket a point
        # cannot accept)
        C = max(1, N // 100)
        lab = torch.randint(0, C, (N,), generator=g)
        mu = 50.0 * torch.randn(C, 2, generator=g)
        Y = (mu[lab] + 0.5 * torch.randn(N, 2, generator=g)).to(torch.float64)
        M = N // 9
        span = float((Y.max(0).values - Y.min(0).values).max())
        h = span * (1 + 2.0 ** -20) / 2.0 ** 24          # finest cell side (D9)
        cell = torch.randint(0, 6, (M, 2), generator=g).to(torch.float64)
        off = 0.25 + 0.5 * torch.rand(M, 2, generator=g, dtype=torch.float64)
        Y[:M] = 0.5 + (cell + off) * h
    else:
        raise ValueError(kind)
    return Y.to(torch.float32).numpy()


def random_csr(N: int, k: int = 10, seed: int = 3):
    """A random symmetric sparse P (CSR, both triangles, rows sorted, sum 1)
    for attractive/gradient tests that do not need a kNN graph.  Values are
    drawn, not computed by the method."""
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(N), k)
    cols = rng.integers(0, N, size=N * k)
    keep = rows != cols
    r = np.concatenate([rows[keep], cols[keep]])
    c = np.concatenate([cols[keep], rows[keep]])
    key = np.unique(r.astype(np.int64) * N + c)
    r = (key // N).astype(np.int64)
    c = (key % N).astype(np.int32)
    vals = rng.random(len(key))
    # symmetric values: v(i,j) = v(j,i)
    lo = np.minimum(r, c).astype(np.int64) * N + np.maximum(r, c)
    uniq, inv = np.unique(lo, return_inverse=True)
    sym = rng.random(len(uniq))[inv]
    sym = sym / sym.sum()
    row_ptr = np.zeros(N + 1, np.int64)
    np.add.at(row_ptr, r + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    del vals
    return row_ptr, c, sym.astype(np.float32), sym


def random_rows_csr(N: int, k: int = 126, seed: int = 11):
    """A large random CSR (k sorted distinct-ish columns per row, positive
    values summing to 1) for full-size gradient checks; drawn, not computed
    by the method."""
    rng = np.random.default_rng(seed)
    cols = rng.integers(0, N, size=(N, k), dtype=np.int64).astype(np.int32)
    cols.sort(1)
    rp = np.arange(0, N * k + 1, k, dtype=np.int64)
    val = rng.random(N * k).astype(np.float32)
    val /= np.float32(val.sum(dtype=np.float64))
    return rp, cols.ravel(), val


def hub_csr(N: int, k: int = 8, hub_degrees=(2500, 5000, 9000, 15000), seed: int = 13):
    """random_csr plus a few hub points joined to many others (rows far longer
    than a kNN row: the attractive pass's long-row path), symmetric, sum 1;
    drawn, not computed by the method."""
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(N), k)
    cols = rng.integers(0, N, size=N * k)
    hubs = rng.choice(N, size=len(hub_degrees), replace=False)
    hr = [np.full(d, h) for h, d in zip(hubs, hub_degrees)]
    hc = [rng.choice(N, size=d, replace=False) for d in hub_degrees]
    rows = np.concatenate([rows] + hr)
    cols = np.concatenate([cols] + hc)
    keep = rows != cols
    r = np.concatenate([rows[keep], cols[keep]])
    c = np.concatenate([cols[keep], rows[keep]])
    key = np.unique(r.astype(np.int64) * N + c)
    r = (key // N).astype(np.int64)
    c = (key % N).astype(np.int32)
    lo = np.minimum(r, c).astype(np.int64) * N + np.maximum(r, c)
    uniq, inv = np.unique(lo, return_inverse=True)
    sym = rng.random(len(uniq))[inv]
    sym = sym / sym.sum()
    row_ptr = np.zeros(N + 1, np.int64)
    np.add.at(row_ptr, r + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    return row_ptr, c, sym.astype(np.float32), sym
