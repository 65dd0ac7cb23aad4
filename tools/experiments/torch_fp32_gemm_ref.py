import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False
for (M, N, K) in [(10000, 156, 156), (10000, 156, 237), (10000, 156, 81), (156, 237, 10000)]:
    a = torch.randn(M, K, device="cuda"); b = torch.randn(K, N, device="cuda")
    for _ in range(5): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    print(f"M={M} N={N} K={K}: {ms*1e3:.1f} us, {2*M*N*K/ms/1e9:.1f} TF/s")
