"""f2 measurement: IVF-PQ kNN (tsne_ivfpq_build / _search) at a workload's
full size against the exact kNN (tsne_knn): recall@K and time per tau.

    python measure/ivfpq_recall.py [--config C5] [--out profiles/r2_ivfpq_C5.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1807_11824_b200 as T  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--taus", default="1,4,8,16,32")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    N = a.n or cfg.N
    K = min(N - 1, int(3 * cfg.perplexity))
    X = synth.make_x(cfg, n=N, device="cuda")
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    s, e = ev(), ev()
    s.record(); ex, _, info = T.knn(X, K); e.record(); torch.cuda.synchronize()
    res = {"config": cfg.name, "N": N, "D": cfg.D, "K": K,
           "exact_knn_ms": s.elapsed_time(e), "exact_path": info["gemm_path"], "runs": []}
    ex = ex.cpu().numpy()
    s.record(); ix = T.IvfPQ(X); e.record(); torch.cuda.synchronize()
    res.update({"build_ms": s.elapsed_time(e), "nlist": ix.nlist, "m": ix.m, "dsub": ix.dsub})
    sizes = torch.diff(ix.parts()["list_offsets"].long()).cpu().numpy()
    res["list_sizes"] = {"mean": float(sizes.mean()), "max": int(sizes.max()),
                         "p99": float(np.percentile(sizes, 99)), "empty": int((sizes == 0).sum()),
                         "mean_seen_by_a_point": float((sizes.astype(np.float64) ** 2).sum() / N)}
    print(res["list_sizes"], flush=True)
    rows = np.random.default_rng(0).choice(N, min(N, 200000), replace=False)
    for tau in [int(t) for t in a.taus.split(",") if int(t) <= ix.nlist]:
        s.record(); idx, d2 = ix.search(X, K, tau); e.record(); torch.cuda.synchronize()
        idx = idx.cpu().numpy()
        rec = float(np.mean([len(set(idx[r]) & set(ex[r])) / K for r in rows]))
        res["runs"].append({"tau": tau, "search_ms": s.elapsed_time(e), "recall_at_K": rec,
                            "recall_rows": len(rows)})
        print(res["runs"][-1], flush=True)
    line = json.dumps(res, indent=1)
    print(line)
    if a.out:
        open(a.out, "w").write(line + "\n")


if __name__ == "__main__":
    main()
