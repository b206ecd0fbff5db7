"""GPU <-> oracle parity of the exact-Z cost through the C ABI.

tsne_kl computes Z = sum_{k != l} (1 + d_kl^2)^-1 exactly (fp32 pairs, fp64
accumulation) and KL(P || Q) = sum_{P_ij > 0} P_ij ln(P_ij Z / w_ij) (Eq. 2,
P:L68-73).  The oracle's O12 (oracle_kl_d, fp64) and O11's Z are the
references.  Bars: Z within 1e-6 relative (fp32 pair terms carry ~1e-7 each,
the sums are fp64); KL within 1e-6 * max(1, |KL|) -- ln Z enters KL with weight
sum P = 1, so Z's relative error appears in KL as an absolute error (and KL
itself is 0 for N = 2).
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


def gpu_kl(T, rp, col, v32, Y):
    dev = torch.device("cuda")
    return T.kl(torch.as_tensor(rp, device=dev), torch.as_tensor(col, device=dev),
                torch.as_tensor(v32, device=dev), torch.as_tensor(Y, device=dev))


@pytest.mark.parametrize("N,kind", [(2, "gauss10"), (3, "gauss10"), (257, "gauss10"),
                                    (1000, "clustered"), (4099, "gauss10"), (9000, "blobs")])
def test_kl_and_z_vs_oracle(T, orc, N, kind):
    rp, col, v32, v64 = synth.random_csr(N, min(10, N - 1), seed=N + 5)
    Y = synth.fixed_y(kind, N, seed=3).astype(np.float32)
    kl, Z = gpu_kl(T, rp, col, v32, Y)
    Y64 = Y.astype(np.float64)
    kl_ref = orc.kl(rp, col, v32, Y64)            # O12 on the fp32 P the GPU sees
    assert abs(kl - kl_ref) <= 1e-6 * max(1.0, abs(kl_ref)), (kl, kl_ref)
    if N <= 4099:
        _, Z_ref = orc.gradient_exact(rp, col, v64, Y64)   # O11's exact Z
        assert abs(Z - Z_ref) <= 1e-6 * Z_ref, (Z, Z_ref)


def test_kl_zero_entries_and_identical_points(T, orc):
    # all points coincide: w = 1 for every pair, Z = N (N - 1); zero P entries are skipped
    N = 300
    rp, col, v32, _ = synth.random_csr(N, 6, seed=2)
    v32 = v32.copy()
    v32[::7] = 0.0
    Y = np.full((N, 2), 1.5, np.float32)
    kl, Z = gpu_kl(T, rp, col, v32, Y)
    assert Z == pytest.approx(N * (N - 1), rel=1e-12)
    assert kl == pytest.approx(orc.kl(rp, col, v32, Y.astype(np.float64)), rel=1e-6, abs=1e-6)


def test_kl_deterministic(T):
    N = 5000
    rp, col, v32, _ = synth.random_csr(N, 8, seed=9)
    Y = synth.fixed_y("gauss10", N, seed=4).astype(np.float32)
    a = gpu_kl(T, rp, col, v32, Y)
    b = gpu_kl(T, rp, col, v32, Y)
    assert a == b
