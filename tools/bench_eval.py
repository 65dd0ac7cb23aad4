#!/usr/bin/env python
"""Evaluation benchmark (SURVEY.md 8(f) ranks 1 + 3): train::evaluate over a
dataset split on one B200 — spectra.bin streamed by index (dataset.cpp reader),
rendered (MLP + raster) and scored (PSNR, SSIM, L1) on the device — vs the
reference's own train::evaluate on the host cores. One JSON line.

value = samples/s of swr_evaluate_dataset (wall clock around the C-ABI call:
it includes the file reads and H2D copies, i.e. it is also the e2e number);
also reported: swr_metrics alone on device-resident spectra (CUDA events)."""
import ctypes as C
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import oracle as O  # noqa: E402
from paper_2506_12787_b200 import swr  # noqa: E402
from paper_2506_12787_b200.scene import make_scene  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
d = tempfile.mkdtemp(prefix="swr_eval_ds_")
t0 = time.perf_counter()
h, bbox = O.make_dataset(d, 90, 360, count, 5)
gen_s = time.perf_counter() - t0
sc = make_scene(n, seed=1)
sc.bbox_min, sc.bbox_max = tuple(bbox[:3]), tuple(bbox[3:])
ck = swr.Checkpoint.from_scene(sc)
ck.set_manifest_hash(h)
ds = swr.Dataset(d)
swr.evaluate_dataset(ck, ds, swr.Dataset.ALL)  # warm (allocations, file cache)
with bench.ClockSampler(0) as clk:
    t0 = time.perf_counter()
    rows = swr.evaluate_dataset(ck, ds, swr.Dataset.ALL)
    wall = time.perf_counter() - t0
nrows = len(rows["psnr"])

# metrics alone, device-resident pairs
B = 1024
pred = torch.rand((B, 90, 360, 2), device="cuda")
tgt = torch.rand((B, 90, 360, 2), device="cuda")
outs = [torch.empty(B, dtype=torch.float64, device="cuda") for _ in range(3)]
stream = torch.cuda.Stream()
L = swr.lib()
call = lambda: swr._check(L.swr_metrics_device(ck.handle, pred.data_ptr(), tgt.data_ptr(), B, 1.0,
                                                 outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(),
                                                 C.c_void_p(stream.cuda_stream)))
for _ in range(3):
    call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(10):
    call()
e1.record(stream)
torch.cuda.synchronize()
met_ms = e0.elapsed_time(e1) / 10

line = {"metric": "evaluate_samples_per_s", "value": round(nrows / wall, 1), "unit": "samples/s", "n_gpus": 1,
        "steps": 1, "warmup": 1, "ms_per_step": round(wall * 1e3, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (render), f64 (metric statistics)",
        "data": f"{nrows}-sample 90x360 dataset simulated by the reference's wavesim ({gen_s:.1f} s), on disk",
        "config": {"workload": "train::evaluate(ck, ds, all): read + render + psnr/ssim/l1", "gaussians": n,
                   "samples": nrows},
        "e2e": {"value": round(nrows / wall, 1), "unit": "samples/s",
                "h2d_bytes_per_step": int(nrows * (12 + 259200)), "d2h_bytes_per_step": int(nrows * 24)},
        "metrics_only": {"value": round(B / (met_ms / 1e3), 1), "unit": "pairs/s", "ms_per_1024": round(met_ms, 3),
                         "note": "swr_metrics_device on device-resident pairs (psnr + ssim + l1)"},
        "clocks": clk.summary()}
ref = O.Reference(scene=sc)
ref.set_dataset(h, bbox)
ref.set_threads(os.cpu_count())
sub = min(nrows, 64)
# the reference evaluates the whole split; time it on a bounded subset dataset
d2 = tempfile.mkdtemp(prefix="swr_eval_small_")
h2, bbox2 = O.make_dataset(d2, 90, 360, sub, 5)
ref2 = O.Reference(scene=sc)
ref2.set_dataset(h2, bbox2)
ref2.set_threads(os.cpu_count())
t0 = time.perf_counter()
r = ref2.evaluate(d2, 2)
dt = time.perf_counter() - t0
line["cpu_baseline"] = {"value": round(len(r) / dt, 3), "unit": "samples/s", "cores": os.cpu_count(),
                        "kind": "reference", "sample": f"train::evaluate over a {len(r)}-sample dataset, {dt:.1f} s"}
print(json.dumps(line))
