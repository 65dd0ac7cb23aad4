"""D2H bandwidth into pinned host memory: one stream vs two concurrent streams (66 MB pieces)."""
import torch
n = 66 * 1024 * 1024 // 4
d = [torch.randn(n, device="cuda") for _ in range(4)]
h = [torch.empty(n, pin_memory=True) for _ in range(4)]
ss = [torch.cuda.Stream() for _ in range(4)]
for nst in (1, 2, 4):
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(8):
            st = ss[i % nst]
            st.wait_event(e0) if i < nst else None
            with torch.cuda.stream(st):
                h[i % 4].copy_(d[i % 4], non_blocking=True)
        for st in ss[:nst]:
            torch.cuda.current_stream().wait_stream(st)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if rep:
            print(f"{nst} stream(s): {8 * n * 4 / ms / 1e6:.1f} GB/s")
