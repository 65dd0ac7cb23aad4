"""Where the end-to-end time goes at 10k Gaussians x 1,024 positions: device-only
render, a bare pinned D2H of the same spectra, and swr_render (pinned host buffers)
for several host-path chunk sizes (option copy_chunk)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
B = 1024
sc = make_scene(n, seed=0)
sc.rssi_cal = (1.0, 0.0)
ck = swr.Checkpoint.from_scene(sc)
ck.set_option("chunk", 1024 if n <= 20000 else 256)
H, W = ck.H, ck.W
pos = random_positions(B, seed=1)
flags = swr.OUT_SPECTRA | swr.OUT_POOLED | swr.OUT_RSSI | swr.OUT_AOA
st = torch.cuda.Stream()
dpos = torch.from_numpy(pos).cuda()
dsp = torch.empty((B, H, W, 2), device="cuda")
dp = torch.empty(B, dtype=torch.float64, device="cuda")
drc = torch.empty((B, 2), dtype=torch.int32, device="cuda")
dang = torch.empty((B, 2), dtype=torch.float64, device="cuda")
call = lambda: swr.render_device(ck, dpos.data_ptr(), B, flags, dsp.data_ptr(), dp.data_ptr(), dp.data_ptr(),
                                 drc.data_ptr(), dang.data_ptr(), stream=st.cuda_stream)
for _ in range(3):
    call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(st):
    e0.record(st)
    for _ in range(5):
        call()
    e1.record(st)
torch.cuda.synchronize()
print(f"device render (chunk {int(ck.get_option('chunk'))}): {e0.elapsed_time(e1) / 5:.3f} ms per 1024", flush=True)
keep = ck.get_option("chunk")
for chv in (256, 512):
    ck.set_option("chunk", chv)
    for _ in range(2):
        call()
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(5):
            call()
        e1.record(st)
    torch.cuda.synchronize()
    print(f"device render (chunk {chv}): {e0.elapsed_time(e1) / 5:.3f} ms per 1024", flush=True)
ck.set_option("chunk", keep)
h = torch.empty((B, H, W, 2)).pin_memory()
for _ in range(2):
    h.copy_(dsp, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    h.copy_(dsp, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print(f"bare D2H of {dsp.numel() * 4 / 1e6:.0f} MB: {dt * 1e3:.3f} ms ({dsp.numel() * 4 / dt / 1e9:.1f} GB/s)", flush=True)
hp = torch.from_numpy(pos).pin_memory()
hpl = torch.empty(B, dtype=torch.float64).pin_memory()
hrc = torch.empty((B, 2), dtype=torch.int32).pin_memory()
hang = torch.empty((B, 2), dtype=torch.float64).pin_memory()
L = swr.lib()
for cc in (128, 256, 512, 1024):
    ck.set_option("copy_chunk", cc)
    f = lambda: swr._check(L.swr_render(ck.handle, hp.data_ptr(), B, flags, h.data_ptr(), hpl.data_ptr(),
                                        hpl.data_ptr(), hrc.data_ptr(), hang.data_ptr()))
    for _ in range(2):
        f()
    t = time.perf_counter()
    for _ in range(5):
        f()
    dt = (time.perf_counter() - t) / 5
    print(f"swr_render copy_chunk {cc:4d}: {dt * 1e3:.3f} ms per 1024 ({B / dt:,.0f} spectra/s)", flush=True)
