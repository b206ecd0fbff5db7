"""Oracle verification of the headline run (BASELINE.json north star: "oracle-
verified BH t-SNE embedding 1.28M x 2048 ... in 1000 iterations").

Not collected by pytest (it takes ~20 minutes of host time); run on the GPU box:

    python tests/run_c5_long_parity.py --out profiles/r2_c5_long_run.json

1. X: the C5 workload (synth, seed 5), generated on the GPU.
2. kNN + P on the GPU (tsne_knn, tsne_compute_p: their parity with the oracle
   is tested row by row in tests/test_gpu_fullsize.py).
3. From the same Y0 (Philox, seed 42) and the same P: 1000 GPU iterations
   (tsne_optimize, the bench's configuration) and 1000 oracle iterations
   (oracle_optimize, fp64, host cores).
4. Both embeddings scored by the oracle: KL(P||Q) with the exact O(N^2) Z
   (O12) and 10-NN preservation on 10000 sampled points (O12).
   The GPU's exact-Z cost (tsne_kl, f4) is reported beside it.
Bars (north star): |KL_gpu - KL_oracle| <= 1% of KL_oracle; 10-NN within 1 pp.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1807_11824_b200 as T  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--nn-rows", type=int, default=10000)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    oracle.build()
    cfg = synth.CONFIGS[a.config]
    N = a.n or cfg.N
    K = min(N - 1, int(3 * cfg.perplexity))
    res = {"config": cfg.name, "N": N, "D": cfg.D, "K": K, "iters": a.iters,
           "oracle_threads": oracle.num_threads()}
    t = time.time()
    X = synth.make_x(cfg, n=N, device="cuda")
    idx, d2, info = T.knn(X, K)
    rp, col, val = T.compute_p(idx, d2, cfg.perplexity)
    torch.cuda.synchronize()
    del X, d2
    torch.cuda.empty_cache()
    res["gpu_knn_p_s"] = time.time() - t
    res["knn_rows_uncertified"] = info["rows_uncertified"]
    res["nnz"] = int(col.numel())
    idx_h = idx.cpu().numpy()
    rph, colh, valh = rp.cpu().numpy(), col.cpu().numpy(), val.cpu().numpy()
    Y0 = T.init_y(N, 42)
    Y0h = Y0.cpu().numpy()
    # GPU: the bench's optimiser
    t = time.time()
    opt = T.Optimizer(rp, col, val, Y0, theta=0.5)
    Yg = opt.step(a.iters).cpu().numpy().astype(np.float64)
    res["gpu_loop_s"] = time.time() - t
    klg_gpu, _ = T.kl(rp, col, val, torch.as_tensor(Yg.astype(np.float32), device="cuda"))
    # oracle: the same schedule in fp64 on the host cores
    t = time.time()
    Yo, _, _ = oracle.optimize(rph, colh, valh, Y0h.astype(np.float64), n_iter=a.iters, theta=0.5)
    res["oracle_loop_s"] = time.time() - t
    klo_gpu, _ = T.kl(rp, col, val, torch.as_tensor(Yo.astype(np.float32), device="cuda"))
    # scores, both by the oracle
    t = time.time()
    kl_g = oracle.kl(rph, colh, valh, Yg)
    kl_o = oracle.kl(rph, colh, valh, Yo)
    res["oracle_kl_s"] = time.time() - t
    rows = np.random.default_rng(11).choice(N, min(N, a.nn_rows), replace=False)
    t = time.time()
    nn_g = oracle.nn_preservation(idx_h, Yg, 10, rows=rows)
    nn_o = oracle.nn_preservation(idx_h, Yo, 10, rows=rows)
    res["oracle_nn_s"] = time.time() - t
    res.update({
        "kl_gpu": kl_g, "kl_oracle": kl_o, "kl_rel_diff": abs(kl_g - kl_o) / kl_o,
        "kl_gpu_by_tsne_kl": klg_gpu, "kl_oracle_by_tsne_kl": klo_gpu,
        "nn10_gpu": nn_g, "nn10_oracle": nn_o, "nn10_diff_pp": 100 * abs(nn_g - nn_o),
        "nn10_rows": len(rows),
        "pass_kl_1pct": abs(kl_g - kl_o) <= 0.01 * kl_o, "pass_nn_1pp": abs(nn_g - nn_o) <= 0.01,
    })
    line = json.dumps(res, indent=1)
    print(line, flush=True)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")
    return 0 if (res["pass_kl_1pct"] and res["pass_nn_1pp"]) else 1


if __name__ == "__main__":
    sys.exit(main())
