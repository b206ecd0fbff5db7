"""tsne_run_sharded on a world-size-1 NCCL group (one GPU) at a workload's full
size, against tsne_run_ex: the multi-GPU code path's per-stage times on one
GPU (its collectives are then local).

    python measure/sharded_world1.py [--config C5] [--iters 1000]
"""
import argparse
import json
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1807_11824_b200 as T  # noqa: E402
import synth  # noqa: E402
from paper_1807_11824_b200 import sharded  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    so = socket.socket(); so.bind(("127.0.0.1", 0)); port = so.getsockname()[1]; so.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    X = synth.make_x(cfg, device="cuda")
    Xh = torch.empty(X.shape, dtype=torch.float32, pin_memory=True)
    Xh.copy_(X)
    del X
    torch.cuda.empty_cache()
    N = Xh.shape[0]
    Ys, si = sharded.run(Xh, N, perplexity=cfg.perplexity, n_iter=a.iters,
                         device=torch.device("cuda", 0))
    Yr, ri = T.run(Xh, perplexity=cfg.perplexity, n_iter=a.iters)
    kl_s = T.kl(*T.compute_p(*T.knn(Xh.cuda(), min(N - 1, int(3 * cfg.perplexity)))[:2],
                             cfg.perplexity), Ys.cuda())[0] if N <= 200000 else None
    res = {"config": cfg.name, "N": N, "iters": a.iters,
           "tsne_run_sharded_world1": {k: si[k] for k in ("ms_h2d", "ms_knn", "ms_p", "ms_loop",
                                                            "ms_total", "nnz")},
           "tsne_run_ex": {k: ri[k] for k in ("ms_h2d", "ms_knn", "ms_p", "ms_loop", "ms_total",
                                              "nnz")},
           "kl_sharded": kl_s}
    print(json.dumps(res, indent=1))
    if a.out:
        open(a.out, "w").write(json.dumps(res, indent=1) + "\n")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
