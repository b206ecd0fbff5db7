# Per-stage profile and traversal counters of C2 at t = 50 / 150 / 240 (bench.py times t = 50-250):
# shows how a transient collapse (exact bucket pairs) in one trajectory moves the timed value.
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_1807_11824_b200 as T
cfg = synth.CONFIGS["C2"]
X = synth.make_x(cfg, device="cuda")
K = int(3 * cfg.perplexity)
idx, d2, _ = T.knn(X, K)
rp, col, val = T.compute_p(idx, d2, cfg.perplexity)
opt = T.Optimizer(rp, col, val, T.init_y(cfg.N, 42, device="cuda"), theta=0.5)
out = {}
for t in (50, 150, 240):
    opt.step(t - opt.state.t)
    torch.cuda.synchronize()
    p = T.profile_iteration(opt, reps=3)
    out[t] = {"tree": p["tree_ms"], "trav": p["traverse_ms"], "it": p["iteration_overlapped_ms"], **p["traverse_per_point"]}
print(json.dumps(out))
