#!/usr/bin/env python
"""Training-loop benchmark: train::train iterations per
second on one B200 at the reference's default TrainConfig (10000 primitives,
width 156, 90x360 grid), one JSON line in bench.py's shape.

    python tools/bench_train.py [--stage fine|coarse] [--iters K] [--warmup W]

One step = one training iteration of the stage (coarse: render -> hybrid loss ->
rasterize_backward -> Adam on the Gaussians; fine: deform-net forward with
activations -> render with residuals -> loss -> rasterize_backward ->
deform_backward -> Adam on net + Gaussians). The dataset is simulated by the
reference's own wavesim (oracle/_ref) once, before timing; it is resident in HBM.
value = device-timed iterations/s (CUDA events around the replayed iterations);
e2e = the same through the public API (Trainer.run: plan upload, graph replays,
log download) by wall clock. cpu_baseline = the reference's own train() (built
from its sources; its deform GEMMs are the Eigen-free restatement in
oracle/ref_shim) on the host cores for a bounded number of iterations.
"""
import argparse
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402

import bench  # noqa: E402  (ClockSampler)
import oracle as O  # noqa: E402
from paper_2506_12787_b200 import swr  # noqa: E402
from paper_2506_12787_b200.scene import make_scene  # noqa: E402


def gemm_flop_per_iter(n, width, D):
    """Algorithmic FP32 FLOPs of the network per fine iteration (forward +
    deform_backward, deform.cpp:140-326): forward rows x layer shapes, backward
    dW for every layer and dIN for layers 1..7 (hidden block only)."""
    cols = [D] + [width + D if i in (2, 4, 6) else width for i in range(1, 8)]
    fwd = sum(2 * width * c for c in cols) + 2 * 5 * width
    dw = sum(2 * width * c for c in cols) + 2 * 5 * width
    din = 7 * 2 * width * width + 2 * 5 * width
    return n * (fwd + dw + din)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stage", default="fine", choices=["fine", "coarse"])
    ap.add_argument("--iters", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--primitives", type=int, default=10000)
    ap.add_argument("--samples", type=int, default=64)
    ap.add_argument("--ref-iters", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    d = tempfile.mkdtemp(prefix="swr_train_ds_")
    O.make_dataset(d, 90, 360, args.samples, 3)
    ds = swr.Dataset(d)
    total = args.warmup + args.iters
    kw = dict(primitives=args.primitives, coarse_iters=total if args.stage == "coarse" else 0,
              fine_iters=total if args.stage == "fine" else 0, anneal_threshold=10000)
    cfg = swr.TrainConfig(**kw)
    tr = swr.Trainer(cfg, ds)
    tr.run(args.warmup)
    with bench.ClockSampler(0) as clk:
        t0 = time.perf_counter()
        log, dev_ms = tr.run(args.iters)
        wall = time.perf_counter() - t0
    value = args.iters / (dev_ms / 1e3)
    e2e = args.iters / wall
    D = 2 * (2 * cfg.bands_center + 1) + 3 * (2 * cfg.bands_position + 1)
    line = {
        "metric": f"train_{args.stage}_iterations_per_s", "value": round(value, 2), "unit": "it/s", "n_gpus": 1,
        "steps": args.iters, "warmup": args.warmup, "ms_per_step": round(dev_ms / args.iters, 4),
        "higher_is_better": True, "scaling": "replicas only", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: 90x360 dataset simulated by the reference's wavesim, resident in HBM",
        "config": {"workload": f"train::train {args.stage} stage, TrainConfig defaults", "primitives": args.primitives,
                   "width": cfg.width, "grid": [90, 360], "samples": args.samples,
                   "l2": "per-iteration working set (params, activations, spectra) < L2 except the dataset"},
        "e2e": {"value": round(e2e, 2), "unit": "it/s",
                "h2d_bytes_per_step": int(4 + 4 * (3 * (2 * cfg.bands_position + 1)) + 48),
                "d2h_bytes_per_step": 24},
        "loss_first_last": [float(log[0, 0]), float(log[-1, 0])],
        "clocks": clk.summary(),
    }
    if args.stage == "fine":
        f = gemm_flop_per_iter(args.primitives, cfg.width, D)
        line["network_gflop_per_step"] = round(f / 1e9, 3)
        line["network_tflops_if_all_time"] = round(f / (dev_ms / args.iters / 1e3) / 1e12, 2)
    if not args.no_cpu_baseline:
        ref_iters = args.ref_iters or (5 if args.stage == "fine" else 40)
        ref = O.Reference(scene=make_scene(4, seed=1, H=12, W=16, width=24))
        rc = swr.TrainConfig(**dict(kw, coarse_iters=ref_iters if args.stage == "coarse" else 0,
                                    fine_iters=ref_iters if args.stage == "fine" else 0))
        t0 = time.perf_counter()
        ref.train(d, rc)
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": round(ref_iters / dt, 3), "unit": "it/s", "cores": os.cpu_count(),
                                "kind": "reference",
                                "sample": f"{ref_iters} {args.stage} iterations of the reference train() "
                                          f"(incl. init), {dt:.1f} s"}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
