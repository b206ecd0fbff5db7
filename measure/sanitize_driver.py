"""Small invocations of every kernel of the library for compute-sanitizer
(measure/sanitize.sh): kNN (row sweep + fp64 re-rank + exact fallback), P,
gradient (tree build, bucket pairs, traversal, attractive pass), the optimiser
(graphs, diffusion order, Morton relabelling, keep_state resume), the exact-Z
cost, tsne_run_ex end to end, the multi-GPU shard kernels, and (--sym) the
symmetric tcgen05 kNN search at its smallest size (N = 2^18, D = 1024)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1807_11824_b200 as T  # noqa: E402
import synth  # noqa: E402


def main():
    dev = torch.device("cuda")
    N = 3000
    X = synth.make_x("C2", n=N).to(dev)
    idx, d2, info = T.knn(X, 90)
    rp, col, val = T.compute_p(idx, d2, 30.0)
    Y = torch.as_tensor(synth.fixed_y("clustered", N, seed=3), device=dev)
    T.gradient(rp, col, val, Y, 0.5, 12.0)
    T.gradient(rp, col, val, Y, 0.0, 1.0)
    opt = T.Optimizer(rp, col, val, T.init_y(N, 42), theta=0.5, relabel_every=16)
    opt.step(130)
    opt.step(6)                       # keep_state resume
    T.kl(rp, col, val, opt.state.Y)
    T.profile_iteration(opt, reps=1)
    T.run(X.cpu().pin_memory(), perplexity=30.0, n_iter=8)
    # shard kernels (one rank's share of a 2-way split, no exchange)
    from paper_1807_11824_b200.sharded import GpuShardOps, local_csr, shard_range
    ops = GpuShardOps(N, dev)
    a, b, _ = shard_range(N, 2, 1)
    rpl, cl, vl = local_csr(rp, col, val, a, b)
    A = torch.zeros(b - a, 2, device=dev)
    rep = torch.zeros(b - a, 2, device=dev)
    zp = torch.zeros(4, dtype=torch.float64, device=dev)
    Yf = T.init_y(N, 7)
    ops.attract(rpl, cl, vl, N, a, b, Yf, A)
    ops.forces(Yf, N, a, b, 0.5, True, rep, zp[2:])
    v, g, out = (torch.zeros(b - a, 2, device=dev), torch.ones(b - a, 2, device=dev),
                 torch.empty(b - a, 2, device=dev))
    ops.update(A, N, a, b, Yf, rep, zp, 2, 3, 200.0, 12.0, T.default_config(), v, g, out)
    ops.recentre(Yf, N)
    if "--sym" in sys.argv:
        Xs = synth.make_x("C5", n=1 << 18, device="cuda")[:, :1024].contiguous()
        i2, d22, inf2 = T.knn(Xs, 90)
        assert inf2["gemm_path"] == "tcgen05-sym", inf2
    torch.cuda.synchronize()
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
