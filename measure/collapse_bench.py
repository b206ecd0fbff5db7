"""Time the BH gradient (tsne_gradient: tree, traversal, attractive pass) on a
fixed collapsed-cluster embedding (synth 'collapsed': N // 9 points over 36
adjacent finest cells) against the same N without the collapse ('blobs'), and
print the traversal counters of the collapsed case.  Measurement only."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_11824_b200 as T  # noqa: E402
import synth  # noqa: E402


def time_grad(rp, col, val, Y, reps=10):
    T.gradient(rp, col, val, Y, 0.5, 12.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        T.gradient(rp, col, val, Y, 0.5, 12.0)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 70000
    dev = torch.device("cuda")
    rp, col, v32, _ = synth.random_csr(N, 10, seed=5)
    rp, col, v32 = (torch.as_tensor(x, device=dev) for x in (rp, col, v32))
    out = {"N": N}
    for kind in ("blobs", "collapsed"):
        Y = torch.as_tensor(synth.fixed_y(kind, N, seed=21), device=dev)
        out[kind + "_ms"] = time_grad(rp, col, v32, Y)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
