"""Measured FP64 tensor rate of this B200 via cuBLAS DGEMM (torch.matmul on
float64, 8192^3), the denominator for the FP64 accuracy mode's roofline.
GPU box only."""
import json
import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    a @ b
torch.cuda.synchronize()
best = 1e30
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    a @ b
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"dgemm_n": n, "ms": best, "fp64_tflops": 2 * n ** 3 / best / 1e9}))
