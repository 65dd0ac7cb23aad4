"""Latency of small batches (the reference's call pattern: train::render_at in a
loop): wall time per swr_render call (host buffers), GPU time per
swr_render_device call (CUDA events, side stream), the per-stage split, the same
with the FP32 CUDA-core MLP, and a CUDA-graph replay of the device call."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
sc = make_scene(n, seed=0)
ck = swr.Checkpoint.from_scene(sc)
H, W = ck.H, ck.W
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
prec0 = ck.get_option("mlp_precision")


def dev_time(fn, n):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record(st)
    for _ in range(n):
        fn()
    e1.record(st)
    tw = (time.perf_counter() - t) / n
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3, tw * 1e6


for B in (1, 2, 4, 8, 16, 64):
    pos = random_positions(B, seed=1)
    n_it = 100 if B <= 16 else 30
    for _ in range(3):
        swr.render(ck, pos, aoa=False, pooled=False)
    t = time.perf_counter()
    for _ in range(n_it):
        swr.render(ck, pos, aoa=False, pooled=False)
    host = (time.perf_counter() - t) / n_it * 1e6
    dpos = torch.from_numpy(pos).cuda()
    dsp = torch.empty((B, H, W, 2), device="cuda")
    f = swr.OUT_SPECTRA
    call = lambda: swr.render_device(ck, dpos.data_ptr(), B, f, d_spec=dsp.data_ptr(), stream=st.cuda_stream)
    g_us, w_us = dev_time(call, n_it)
    ck.set_option("stage_timing", 1)
    ck.set_option("stage_reset", 1)
    for _ in range(n_it):
        call()
    torch.cuda.synchronize()
    ck.set_option("stage_timing", 0)
    stg = ck.stage_times() / n_it * 1e3
    ref = dsp.clone()
    ck.set_option("mlp_precision", 0)
    g32, _ = dev_time(call, n_it)
    ck.set_option("mlp_precision", prec0)
    gr = None
    try:
        call()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=st):
            call()
        gr, _ = dev_time(graph.replay, n_it)
        same = bool(torch.equal(dsp, ref))
    except Exception as ex:  # capture unsupported
        print("graph capture failed:", repr(ex)[:200], flush=True)
        same = None
    print(f"B={B:3d}: swr_render {host:7.1f} us; render_device GPU {g_us:6.1f} us (host {w_us:6.1f}); "
          f"fp32 MLP GPU {g32:6.1f} us; graph replay {gr if gr is None else round(gr, 1)} us (same={same}); "
          f"stages {np.round(stg, 1).tolist()}", flush=True)
