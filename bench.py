"""bench.py -- throughput of the Barnes-Hut t-SNE iteration on B200.

Metric (BASELINE.json): BH t-SNE iterations/s (and end-to-end seconds) on the
ImageNet-ResNet-shaped workload C5: N = 1,281,167 points, D = 2048, perplexity
30 (K = 90), theta = 0.5.  A "step" is one t-SNE iteration: quadtree build ->
theta traversal (F_rep, Z) -> attractive pass fused with the update (DESIGN.md
section 7).  The supporting kNN and P stages run once before the timed loop
(timed and reported in `stages`), and again inside the end-to-end `e2e` leg
(tsne_run from pinned host X to host Y).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C5] [--npoints N_override] [--no-e2e] [--no-cpu]

`--impl reference` times the fp64 CPU oracle (oracle/) on the host cores, one
full-size oracle iteration per step.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "BH t-SNE iterations/s (N=1.28M, D=2048 ImageNet-ResNet-shaped)"

# nonzeros per row of the GPU's P on each workload (measured, profiles/r1_bench_C*_final.json):
# the reference arm times the oracle iteration on a CSR with this row length
NNZ_PER_ROW = {"C1": 96, "C2": 161, "C3": 149, "C4": 233, "C5": 146}


def measured_peaks():
    """L2 / L1 / FP64 peaks from measure/peaks.py (profiles/r2_peaks.json), if present."""
    p = os.path.join(ROOT, "profiles", "r2_peaks.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, dev=0):
        self.dev, self.rows, self.proc = dev, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[2 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def cpu_iteration_inputs(N, nnz_per_row=126, seed=0):
    """Iteration-shaped inputs for timing the oracle (synth only): a clustered
    2-D embedding and a CSR with the workload's mean row length."""
    Y = synth.fixed_y("clustered", N, seed=seed, labels=torch.randint(
        0, 1000, (N,), generator=torch.Generator().manual_seed(seed)))
    rng = np.random.default_rng(seed)
    cols = rng.integers(0, N, size=(N, nnz_per_row), dtype=np.int64).astype(np.int32)
    cols.sort(1)
    rp = np.arange(0, N * nnz_per_row + 1, nnz_per_row, dtype=np.int64)
    val = (rng.random(N * nnz_per_row) * (2.0 / (N * nnz_per_row))).astype(np.float32)
    return Y, rp, cols.ravel(), val


def time_oracle_iterations(N, n_iter, nnz_per_row, warmup=0):
    import oracle
    Y, rp, col, val = cpu_iteration_inputs(N, nnz_per_row)
    Yd = Y.astype(np.float64)
    v = np.zeros_like(Yd)
    g = np.ones_like(Yd)
    if warmup:
        Yd, v, g = oracle.optimize(rp, col, val, Yd, v, g, t0=0, n_iter=warmup, theta=0.5)
    times = []
    for k in range(n_iter):
        t = time.perf_counter()
        Yd, v, g = oracle.optimize(rp, col, val, Yd, v, g, t0=warmup + k, n_iter=1, theta=0.5)
        times.append(time.perf_counter() - t)
    return times, oracle.num_threads()


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = synth.CONFIGS[args.config]
    N = args.n or cfg.N
    nnz_row = args.nnz_per_row or NNZ_PER_ROW.get(args.config, 146)
    times, cores = time_oracle_iterations(N, args.steps, nnz_row, warmup=args.warmup)
    T = sum(times)
    v = args.steps / T
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "it/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": cfg.name, "N": N, "D": cfg.D,
                   "K": min(N - 1, int(3 * cfg.perplexity)), "perplexity": cfg.perplexity,
                   "theta": 0.5, "nnz_per_row": nnz_row,
                   "parallelism": "host cores (OpenMP over points)"},
        "cpu_baseline": {"value": v, "unit": "it/s", "cores": cores, "kind": "oracle",
                         "sample": f"{args.steps} full-size oracle iterations (fp64 tree + traversal "
                                   f"+ attractive + update) at N={N}, synthetic clustered Y and "
                                   f"{nnz_row} nnz/row CSR"},
        "e2e": {"value": v, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_e2e(T, Xh, cfg, N, args):
    """tsne_run_ex through the C ABI from pinned host X to pinned host Y."""
    Yh = torch.empty(N, 2, dtype=torch.float32, pin_memory=True)
    t0 = time.perf_counter()
    Yh, info = T.run(Xh, perplexity=cfg.perplexity, theta=0.5, n_iter=args.e2e_iters, Y_out=Yh)
    wall = time.perf_counter() - t0
    # value: the wall clock of the whole C-ABI call (allocation, H2D of X, kNN,
    # P, n_iter iterations, D2H of Y); CUDA events split the device part
    return {"value": args.e2e_iters / wall, "unit": "it/s", "seconds": wall,
            "device_event_seconds": info["ms_total"] / 1e3, "n_iter": args.e2e_iters,
            "h2d_bytes_per_step": 4 * N * cfg.D, "d2h_bytes_per_step": 8 * N,
            "split_ms": {k: info[k] for k in ("ms_h2d", "ms_knn", "ms_p", "ms_loop", "ms_d2h")},
            "knn_rows_uncertified": info["knn_rows_uncertified"], "nnz": info["nnz"], "_Y": Yh}


def run_e2e_sharded(Xh_local, cfg, N, args, rank, world, dev):
    """sharded.run on `world` GPUs from each rank's pinned host shard of X to
    pinned host Y on rank 0; CUDA events on every rank, max over ranks."""
    from paper_1807_11824_b200 import sharded
    Yh = torch.empty(N, 2, dtype=torch.float32, pin_memory=True) if rank == 0 else None
    torch.distributed.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    _, info = sharded.run(Xh_local, N, perplexity=cfg.perplexity, theta=0.5,
                          n_iter=args.e2e_iters, Y_out=Yh, device=dev)
    b.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    t = torch.tensor([a.elapsed_time(b) / 1e3, wall], dtype=torch.float64, device=dev)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    sec, wall = float(t[0]), float(t[1])
    return {"value": args.e2e_iters / sec, "unit": "it/s", "seconds": sec, "wall_seconds": wall,
            "n_iter": args.e2e_iters, "h2d_bytes_per_step": 4 * N * cfg.D,
            "d2h_bytes_per_step": 8 * N, "api": "paper_1807_11824_b200.sharded.run",
            "knn_rows_uncertified": info["knn_rows_uncertified"], "nnz": info["nnz"]}


def run_ours(args, rank, world):
    import paper_1807_11824_b200 as T
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    cfg = synth.CONFIGS[args.config]
    N = args.n or cfg.N
    K = min(N - 1, int(3 * cfg.perplexity))
    stages = {}
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    X = synth.make_x(cfg, n=N, device=dev)
    torch.cuda.synchronize()
    e2e = None
    if rank == 0 and world == 1 and not args.no_e2e:
        # end to end first, in a clean process state: pinned host X -> host Y
        Xh = torch.empty(X.shape, dtype=torch.float32, pin_memory=True)
        Xh.copy_(X)
        del X
        torch.cuda.empty_cache()
        e2e = run_e2e(T, Xh, cfg, N, args)
        X = Xh.to(dev)
        del Xh
    elif world > 1 and not args.no_e2e:
        from paper_1807_11824_b200.sharded import shard_range
        r0, r1, _ = shard_range(N, world, rank)
        Xh = torch.empty(r1 - r0, cfg.D, dtype=torch.float32, pin_memory=True)
        Xh.copy_(X[r0:r1])
        e2e = run_e2e_sharded(Xh, cfg, N, args, rank, world, dev)
        del Xh
        torch.cuda.empty_cache()
    a, b = ev(), ev()
    if world > 1:
        # the kNN sharded by query row (tsne_knn_rows), lists all-gathered
        from paper_1807_11824_b200.sharded import _all_gather_flat, shard_range
        r0, r1, S = shard_range(N, world, rank)
        torch.distributed.barrier()
        torch.cuda.synchronize()
        a.record()
        il, dl, kinfo = T.knn(X, K, rows=(r0, r1))
        ip = torch.zeros(S, K, dtype=torch.int32, device=dev)
        dp = torch.zeros(S, K, dtype=torch.float64, device=dev)
        ip[: r1 - r0], dp[: r1 - r0] = il, dl
        idx = torch.empty(world * S, K, dtype=torch.int32, device=dev)
        d2 = torch.empty(world * S, K, dtype=torch.float64, device=dev)
        _all_gather_flat(idx, ip)
        _all_gather_flat(d2, dp)
        idx, d2 = idx[:N].contiguous(), d2[:N].contiguous()
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b)], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        stages["knn_ms"] = float(t.item())
        del il, dl, ip, dp
    else:
        a.record()
        idx, d2, kinfo = T.knn(X, K)
        b.record()
        torch.cuda.synchronize()
        stages["knn_ms"] = a.elapsed_time(b)
    del X
    a.record()
    rp, col, val = T.compute_p(idx, d2, cfg.perplexity)
    b.record()
    torch.cuda.synchronize()
    stages["p_ms"] = a.elapsed_time(b)
    nnz = int(col.numel())
    # rows of d2 for the oracle's calibration timing (cpu_baseline.e2e_extrapolated)
    cal_rows = np.random.default_rng(3).choice(N, min(N, 20000), replace=False)
    d2_sample = d2[torch.as_tensor(cal_rows, device=d2.device)].cpu().numpy() \
        if (rank == 0 and world == 1 and not args.no_cpu) else None
    del idx, d2
    quality = None
    if e2e is not None and "_Y" in e2e:
        # cost of the end-to-end embedding with the exact Z (tsne_kl),
        # outside every timed region; P here is the e2e run's P (same X, deterministic)
        Ye = e2e.pop("_Y").to(dev)
        a.record()
        kl, Z = T.kl(rp, col, val, Ye)
        b.record()
        torch.cuda.synchronize()
        quality = {"kl_exact_z": kl, "Z": Z, "n_iter": args.e2e_iters, "kl_ms": a.elapsed_time(b),
                   "api": "tsne_kl"}
        del Ye

    opt = T.Optimizer(rp, col, val, T.init_y(N, 42, device=dev), theta=0.5,
                      relabel_every=args.relabel_every)
    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        opt.step(args.warmup)
        # per-stage profile of a few eager iterations (events on the library's stream)
        torch.cuda.nvtx.range_push("profile")          # ncu --nvtx-include "profile/"
        prof = T.profile_iteration(opt, reps=5, stream=s.cuda_stream)
        torch.cuda.nvtx.range_pop()
        # the profile overwrote the optimiser's kept state: warm up again, so the
        # timed call continues a live state (no re-entry, no graph capture)
        opt.step(args.warmup, stream=s.cuda_stream)
        s.synchronize()
    if world == 1:
        with torch.cuda.stream(s):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with Clocks(dev.index) as clk:
                a.record(s)
                opt.step(args.steps, stream=s.cuda_stream)
                b.record(s)
                s.synchronize()
            ms = a.elapsed_time(b)
        launches = int(args.steps * prof.get("kernels_per_iteration", 0))
        # the timed steps fall in the early-exaggeration phase (t < 250); the late phase
        # (clusters formed, deeper traversals) is timed the same way, outside `value`
        if args.late_t > opt.state.t:
            with torch.cuda.stream(s):
                opt.step(args.late_t - opt.state.t, stream=s.cuda_stream)
                a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a2.record(s)
                opt.step(args.steps, stream=s.cuda_stream)
                b2.record(s)
                s.synchronize()
            stages["late_phase"] = {"t0": args.late_t, "iterations": args.steps,
                                    "ms_per_iteration": a2.elapsed_time(b2) / args.steps}
    else:
        # points sharded over the ranks, two NCCL exchanges per iteration
        from paper_1807_11824_b200.sharded import ShardedOptimizer, local_csr, shard_range
        del opt
        r0, r1, _ = shard_range(N, world, rank)
        sopt = ShardedOptimizer(*local_csr(rp, col, val, r0, r1), T.init_y(N, 42, device=dev),
                                theta=0.5)
        sopt.step(args.warmup)
        torch.cuda.synchronize()
        torch.distributed.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with Clocks(dev.index) as clk:
            a.record()
            sopt.step(args.steps)
            b.record()
            torch.cuda.synchronize()
        torch.distributed.barrier()
        ms = a.elapsed_time(b)
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        # per sharded iteration: bbox, 14 tree, owned flags + scan (2) + list, bucket pairs, traverse, attract (2),
        # attract, update, 2 NCCL all-gathers
        launches = int(args.steps * 26)
    stages.update({k: v for k, v in prof.items()})
    value = args.steps / (ms / 1e3)      # iterations of the whole job per second

    # roofline of the dominant kernel
    hbm, which = peaks()
    # k_attract_tma, algorithmic bytes per launch: col + val (8 B/nnz), row_ptr
    # (8 B/row), y_i (8 B/row), A out (8 B/row); the y_j gathers hit L2 (Y = 10 MB)
    bytes_attr = 8 * nnz + 8 * (N + 1) + 16 * N
    bytes_upd = 64 * N             # k_update: A, f, y, v, gains in; y', v, gains out
    stage_kern = {"attract_ms": "k_attract_tma", "traverse_ms": "k_traverse",
                  "tree_ms": "tree build (10 kernels)", "update_ms": "k_update"}
    # the dominant single kernel: the tree build is a chain of 14 short dependent
    # launches (latency bound), so the choice is between the
    # attractive pass and the traversal; within 10% the HBM-bound attractive pass
    # (algorithmic bytes: a roofline that exposes waste) is the one reported and
    # the traversal is given in its own terms under "traversal"
    kern = "attract_ms" if prof["attract_ms"] >= 0.9 * prof["traverse_ms"] else "traverse_ms"
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")      # dram bytes per launch (ncu)
    if os.path.exists(tf):
        traffic = json.load(open(tf)).get(stage_kern[kern])
        if cfg.name != "C5-imagenet-resnet-shaped":
            traffic = None                        # the ncu captures are of C5
    roof = {"kernel": stage_kern[kern], "kernel_ms": prof[kern],
            "iteration_overlapped_ms": prof.get("iteration_overlapped_ms")}
    if kern == "attract_ms":
        ach = bytes_attr / (prof[kern] / 1e3) / 1e9
        roof.update({"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                     "frac": ach / hbm, "traffic": traffic, "peak_source": which,
                     "algorithmic_bytes": bytes_attr})
    else:
        # k_traverse is issue bound: its roofline is the SM issue rate,
        # 148 SMs x 4 schedulers x 1 warp-instruction per clock at the measured SM clock;
        # achieved = the kernel's warp instructions per launch (ncu, profiles/traffic.json)
        # / its CUDA-event time.  The HBM-bound attractive pass is reported beside it.
        tj = json.load(open(tf)) if os.path.exists(tf) else {}
        # measured per workload (the count depends on the tree, i.e. on the data)
        inst = (tj.get("k_traverse_warp_inst") or {}).get(cfg.name) if kern == "traverse_ms" else None
        clk_mhz = clk.summary().get("sm_mhz") or 1965.0
        peak_issue = 148 * 4 * clk_mhz * 1e6 / 1e9            # G warp-instructions / s
        ach = inst / (prof[kern] / 1e3) / 1e9 if inst else None
        if kern == "tree_ms":
            roof["note"] = "tree build: 14 short dependent launches, latency bound (DESIGN.md 6.2)"
        elif inst is None:
            roof["note"] = "issue-rate roofline needs the ncu instruction count, measured for C5"
        roof.update({"bound": "alu" if kern == "traverse_ms" else "latency", "achieved": ach,
                     "peak": peak_issue if ach else None,
                     "unit": "G warp-instructions/s" if ach else None,
                     "frac": ach / peak_issue if ach else None,
                     "traffic": traffic, "peak_source": "148 SMs x 4 issue/clk x measured SM clock",
                     "warp_instructions_per_launch": inst})
        ach_attr = bytes_attr / (prof["attract_ms"] / 1e3) / 1e9
        roof["hbm_kernel"] = {"kernel": "k_attract_tma", "kernel_ms": prof["attract_ms"],
                              "bound": "hbm", "achieved": ach_attr, "peak": hbm, "unit": "GB/s",
                              "frac": ach_attr / hbm,
                              "traffic": (tj.get("k_attract_tma")
                                          if cfg.name == "C5-imagenet-resnet-shaped" else None),
                              "algorithmic_bytes": bytes_attr}
    roof["update_hbm_gbs"] = bytes_upd / (prof["update_ms"] / 1e3) / 1e9
    # the traversal in its own terms: node visits and interactions per
    # second (counters of one traversal of the profiled embedding, tsne_profile_iterations),
    # the 16-byte node records the lanes load per second against the measured L1 and L2
    # read peaks (measure/peaks.py), and, from the ncu capture of this workload
    # (profiles/traffic.json), the L2 bytes actually moved and the warp instructions
    # per warp step (a warp step = one node visit of the warp's slowest lane)
    tp = prof.get("traverse_per_point") or {}
    pk = measured_peaks()
    trav = None
    if tp.get("visits"):
        t_s = prof["traverse_ms"] / 1e3
        visits = tp["visits"] * N
        warp_steps = tp["warp_max_visits"] * N / 32.0
        node_gbs = 16.0 * visits / t_s / 1e9
        trav = {"kernel": "k_traverse", "ms": prof["traverse_ms"],
                "per_point": tp,
                "node_visits_per_s": visits / t_s,
                "interactions_per_s": tp["interactions"] * N / t_s,
                "node_record_gbs": node_gbs,
                "l1_peak_gbs": pk.get("l1_read_gbs"), "l2_peak_gbs": pk.get("l2_read_gbs"),
                "node_record_frac_of_l1": node_gbs / pk["l1_read_gbs"] if pk.get("l1_read_gbs") else None}
        tj2 = json.load(open(tf)) if os.path.exists(tf) else {}
        nc = (tj2.get("k_traverse_ncu") or {}).get(cfg.name)
        if nc:
            trav["ncu"] = nc
            if nc.get("warp_inst"):
                trav["warp_instructions_per_warp_step"] = nc["warp_inst"] / warp_steps
            if nc.get("lts_bytes") and nc.get("duration_ns") and pk.get("l2_read_gbs"):
                l2 = nc["lts_bytes"] / nc["duration_ns"]
                trav["l2_gbs_ncu"] = l2
                trav["l2_frac_ncu"] = l2 / pk["l2_read_gbs"]
    # the kNN stage against the tensor roofline: algorithmic flops of the
    # candidate GEMM -- 2 D_p per (query, point) pair, each unordered pair once on the
    # symmetric path -- over the whole stage's time (locality order, pilot, sweep,
    # selection, fp64 re-rank included); peak = measured sustained bf16 (= fp16) rate
    knn_roof = None
    if stages.get("knn_ms"):
        Dp = (cfg.D + 63) // 64 * 64
        # per GPU: at N > 1 each rank sweeps its own N/world query rows against all N
        pairs = N * N / 2 if kinfo["gemm_path"] == "tcgen05-sym" else N * N / world
        flop = 2.0 * Dp * pairs
        pk = None
        pf = os.path.join(ROOT, "MEASURED_PEAKS.json")
        if os.path.exists(pf):
            pk = json.load(open(pf)).get("bf16_tflops_sustained")
        ach = flop / (stages["knn_ms"] / 1e3) / 1e12
        knn_roof = {"kernel": "kNN stage (%s)" % kinfo["gemm_path"], "bound": "tensor",
                    "achieved": ach, "peak": pk, "unit": "TFLOP/s",
                    "frac": ach / pk if pk else None, "flop": flop,
                    "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (fp16 runs at the bf16 rate)"}
    line = {
        "metric": METRIC, "value": value, "unit": "it/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "N": N, "D": cfg.D, "K": K, "perplexity": cfg.perplexity,
                   "parallelism": "points sharded x%d (NCCL all-gather of Y + Z partials)" % world
                   if world > 1 else "single GPU",
                   "theta": 0.5, "nnz": nnz, "l2": "inputs larger than L2 (CSR %.2f GB)" %
                   (8 * nnz / 1e9), "knn_path": kinfo["gemm_path"],
                   "knn_rows_uncertified": kinfo["rows_uncertified"]},
        "stages": stages,
        "roofline": roof,
        "traversal": trav,
        "knn_roofline": knn_roof,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        ns = args.cpu_iters
        times, cores = time_oracle_iterations(N, ns, max(1, round(nnz / N)))
        line["cpu_baseline"] = {"value": ns / sum(times), "unit": "it/s", "cores": cores,
                                "kind": "oracle",
                                "sample": f"{ns} full-size fp64 oracle iteration(s) at N={N} "
                                          f"(synthetic clustered Y, {round(nnz / N)} nnz/row)"}
        # the oracle end to end, extrapolated: brute-force kNN from
        # sampled query rows x N / rows, calibration from sampled rows of the GPU's
        # d2, 1000 iterations at the per-iteration time above; the symmetrisation
        # (one sort of 2NK edges) is not included, so this is a lower bound
        import oracle
        Xh = synth.make_x(cfg, n=N, device=dev).cpu().numpy()
        qrows = np.random.default_rng(4).choice(N, args.cpu_knn_rows, replace=False)
        t0 = time.perf_counter()
        oracle.knn(Xh, K, rows=qrows)
        knn_s = (time.perf_counter() - t0) * N / len(qrows)
        del Xh
        t0 = time.perf_counter()
        oracle.calibrate(d2_sample, cfg.perplexity)
        cal_s = (time.perf_counter() - t0) * N / len(d2_sample)
        it_s = 1000 * sum(times) / ns
        tot = knn_s + cal_s + it_s
        line["cpu_baseline"]["e2e_extrapolated"] = {
            "seconds": tot, "knn_s": knn_s, "calibration_s": cal_s, "iterations_1000_s": it_s,
            "sample": f"kNN: {len(qrows)} query rows x N/{len(qrows)}; calibration: "
                      f"{len(d2_sample)} rows x N/{len(d2_sample)}; symmetrisation excluded",
            "gpu_e2e_seconds": e2e["seconds"] if e2e else None,
            "ratio_cpu_over_gpu": tot / e2e["seconds"] if e2e else None}
    if e2e is not None:
        e2e.pop("_Y", None)
        line["e2e"] = e2e
    if quality is not None:
        line["quality"] = quality
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--npoints", "--n", dest="n", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=2)
    ap.add_argument("--cpu-knn-rows", type=int, default=64)
    ap.add_argument("--e2e-iters", type=int, default=1000)
    ap.add_argument("--late-t", type=int, default=700,
                    help="also time --steps iterations from this iteration (late phase); 0 = off")
    ap.add_argument("--nnz-per-row", type=int, default=0,
                    help="reference arm CSR row length (default: the workload's measured one)")
    ap.add_argument("--relabel-every", type=int, default=64)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        # TSNE_BENCH_BACKEND=gloo: exercise the N>1 code path with several
        # ranks on one GPU (functional check only; NCCL is the measured path)
        torch.distributed.init_process_group(os.environ.get("TSNE_BENCH_BACKEND", "nccl"))
    run_ours(args, rank, world)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
