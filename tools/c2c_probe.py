import torch, sys
for T, rows in ((10000, 12000), (65536, 2500), (16384, 8192), (5000, 24000)):
    x = torch.randn(rows, T, dtype=torch.complex64, device="cuda")
    for _ in range(3): y = torch.fft.fft(x, dim=1)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): y = torch.fft.fft(x, dim=1)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(T, rows, f"{ms:.3f} ms  {rows*T*16/ms/1e6:.0f} GB/s at 16 B/pt (one pass r+w)", flush=True)
