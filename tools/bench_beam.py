#!/usr/bin/env python
"""Beam-scan benchmark: sim::beam_scan samples/s on one
B200 (90x360 grid, 16-element array) vs the reference's beam_scan on the host
cores. One JSON line. value = device-timed (CUDA events on the launch stream,
channels and spectra resident in HBM); e2e = swr_beam_scan with host buffers."""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import oracle as O  # noqa: E402
from paper_2506_12787_b200 import swr  # noqa: E402

H, W, K = 90, 360, 16
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
steps, warm = 50, 3
st = swr.Steering(H, W, k_elements=K)
rng = np.random.default_rng(0)
ch = rng.standard_normal((B, K)) + 1j * rng.standard_normal((B, K))
u = ch / np.abs(ch)
d_u = torch.from_numpy(np.ascontiguousarray(u).view(np.float64).copy()).cuda()
d_out = torch.empty((B, H, W, 2), dtype=torch.float64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.Stream()  # a real stream handle (0 would mean the steering handle's own stream)
torch.cuda.set_stream(stream)
L = swr.lib()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
for _ in range(warm):
    swr._check(L.swr_beam_scan_device(st._h, d_u.data_ptr(), B, d_out.data_ptr(), C.c_void_p(stream.cuda_stream)))
torch.cuda.synchronize()
with bench.ClockSampler(0) as clk:
    for i in range(steps):
        flush.zero_()
        ev[i][0].record(stream)
        swr._check(L.swr_beam_scan_device(st._h, d_u.data_ptr(), B, d_out.data_ptr(),
                                          C.c_void_p(stream.cuda_stream)))
        ev[i][1].record(stream)
    torch.cuda.synchronize()
ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
host_out = np.empty((B, H, W, 2))
t0 = time.perf_counter()
st.scan(ch)
e2e_s = time.perf_counter() - t0
ops = H * W * K * 8  # 4 mul + 4 add/sub per (cell, element), double
line = {"metric": "beam_scan_samples_per_s", "value": round(B / (ms / 1e3), 1), "unit": "samples/s", "n_gpus": 1,
        "steps": steps, "warmup": warm, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "replicas only", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic random channels", "config": {"workload": "sim::beam_scan batch", "grid": [H, W],
                                                          "k_elements": K, "batch": B, "l2": "flushed (256 MB write) between steps"},
        "roofline": {"bound": "fp64 (mul/add issue)", "achieved": round(B * ops / (ms / 1e3) / 1e12, 2),
                     "unit": "T double ops/s", "traffic_out_GB": round(B * H * W * 16 / 1e9, 3),
                     "achieved_write_GBs": round(B * H * W * 16 / (ms / 1e3) / 1e9, 1)},
        "e2e": {"value": round(B / e2e_s, 1), "unit": "samples/s", "h2d_bytes_per_step": B * K * 16,
                "d2h_bytes_per_step": B * H * W * 16},
        "clocks": clk.summary()}
# reference: beam_scan(channel, table) per sample (OpenMP over cells) on the host cores
n_ref = 64
t0 = time.perf_counter()
for b in range(n_ref):
    O.ref_beam_scan(ch[b], H, W)
dt = time.perf_counter() - t0
line["cpu_baseline"] = {"value": round(n_ref / dt, 2), "unit": "samples/s", "cores": os.cpu_count(), "kind": "reference",
                        "sample": f"{n_ref} beam_scan(channel, array, grid) calls (steering table rebuilt per call "
                                  f"as in that overload), {dt:.1f} s"}
print(json.dumps(line))
