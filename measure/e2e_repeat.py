"""Wall clock vs device time of tsne_run_ex at C5, three calls in one process
(measurement only): separates host-side overhead variance from the device time."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_11824_b200 as T  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS["C5"]
X = synth.make_x(cfg, device="cuda")
Xh = torch.empty(X.shape, dtype=torch.float32, pin_memory=True)
Xh.copy_(X)
del X
torch.cuda.empty_cache()
Yh = torch.empty(cfg.N, 2, dtype=torch.float32, pin_memory=True)
out = []
for r in range(3):
    t0 = time.perf_counter()
    _, info = T.run(Xh, perplexity=cfg.perplexity, theta=0.5, n_iter=1000, Y_out=Yh)
    out.append({"wall_s": time.perf_counter() - t0, "device_s": info["ms_total"] / 1e3})
print(json.dumps(out))
