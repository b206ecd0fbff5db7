"""Per-stage timing of the optimiser iteration at C5's N without the kNN stage
(measurement only): a random symmetric P (k nonzeros per row) and a clustered
late-phase embedding, tsne_optimize from t0 = 700 (steady-state tree builds:
the sort's previous order is the last iteration's).  Run plain for the
CUDA-event stage times, or under ncu with -k on the tree kernels for the
launch list (profiles/)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_11824_b200 as T  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1281167)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--kind", default="clustered")
    ap.add_argument("--warm", type=int, default=20)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    rp, col, v32, _ = synth.random_csr(a.n, a.k, seed=5)
    Y = synth.fixed_y(a.kind, a.n, seed=6)
    dev = torch.device("cuda")
    opt = T.Optimizer(torch.as_tensor(rp, device=dev), torch.as_tensor(col, device=dev),
                      torch.as_tensor(v32, device=dev), torch.as_tensor(Y, device=dev))
    opt.state.t = 700
    opt.step(a.warm)
    torch.cuda.synchronize()
    st = T.profile_iteration(opt, reps=a.reps)
    st.update({"N": a.n, "k": a.k, "kind": a.kind})
    print(json.dumps(st))


if __name__ == "__main__":
    main()
