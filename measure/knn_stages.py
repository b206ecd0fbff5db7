"""kNN stage times at C5 (TSNE_KNN_TIMING=1 prints the symmetric search's stages
to stderr); total time by CUDA events.  Measurement only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_11824_b200 as T  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS["C5"]
X = synth.make_x(cfg, device="cuda")
for r in range(2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    idx, d2, info = T.knn(X, 90)
    b.record()
    torch.cuda.synchronize()
    print("knn total ms", a.elapsed_time(b), info, flush=True)
