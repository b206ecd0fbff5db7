"""theta-accuracy sweep at full size: the error of the
Barnes-Hut gradient against the exact one (theta = 0 reaches every leaf: the
exact sums) and the exact-Z cost of full runs, as functions of theta.

    python measure/theta_sweep.py [--config C5] [--out profiles/r2_theta_sweep.json]

1. P of the workload (tsne_knn + tsne_compute_p), Y0 = Philox seed 42.
2. The embedding after --iters iterations at theta = 0.5 (the bench's run).
3. At that fixed Y: dY(theta) for every theta (tsne_gradient), against theta = 0:
   relative L2 error of dY, relative error of Z, traversal time.
4. For every theta: --iters iterations from Y0 (tsne_optimize), then KL(P||Q)
   with the exact Z (tsne_kl) and the loop time.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1807_11824_b200 as T  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--thetas", default="0.1,0.2,0.3,0.5,0.8,1.0")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    N = a.n or cfg.N
    K = min(N - 1, int(3 * cfg.perplexity))
    X = synth.make_x(cfg, n=N, device="cuda")
    idx, d2, _ = T.knn(X, K)
    rp, col, val = T.compute_p(idx, d2, cfg.perplexity)
    del X, idx, d2
    torch.cuda.empty_cache()
    Y0 = T.init_y(N, 42)
    Yref = T.Optimizer(rp, col, val, Y0, theta=0.5).step(a.iters).clone()
    thetas = [float(t) for t in a.thetas.split(",")]
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def grad(theta):
        s, e = ev(), ev()
        s.record()
        g, Z = T.gradient(rp, col, val, Yref, theta, 1.0)
        e.record()
        torch.cuda.synchronize()
        return g.double(), Z, s.elapsed_time(e)

    g0, Z0, ms0 = grad(0.0)
    res = {"config": cfg.name, "N": N, "nnz": int(col.numel()), "iters": a.iters,
           "exact": {"theta": 0.0, "Z": Z0, "gradient_ms": ms0}, "gradient": [], "runs": []}
    for th in thetas:
        g, Z, ms = grad(th)
        res["gradient"].append({"theta": th, "rel_l2_err": float((g - g0).norm() / g0.norm()),
                                "Z_rel_err": abs(Z - Z0) / Z0, "gradient_ms": ms})
    for th in [0.0] + thetas if N <= 200000 else thetas:
        opt = T.Optimizer(rp, col, val, Y0, theta=th)
        t0 = time.perf_counter()
        Y = opt.step(a.iters)
        torch.cuda.synchronize()
        sec = time.perf_counter() - t0
        kl, Z = T.kl(rp, col, val, Y)
        res["runs"].append({"theta": th, "kl_exact_z": kl, "loop_s": sec})
    errs = [r["rel_l2_err"] for r in res["gradient"]]
    res["error_monotone_in_theta"] = all(x <= y for x, y in zip(errs, errs[1:]))
    line = json.dumps(res, indent=1)
    print(line)
    if a.out:
        open(a.out, "w").write(line + "\n")


if __name__ == "__main__":
    main()
