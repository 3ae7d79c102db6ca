"""Repro: pipelined host path (N >= 2048) with bands and trials vs the device path."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_1710_08037_b200 import connectivity as C

kind = sys.argv[1] if len(sys.argv) > 1 else "real"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 256
rng = np.random.default_rng(0)
B, R, N = 2, 3, 2304
if kind == "real":
    x = rng.standard_normal((B, R, N, T)).astype(np.float32)
else:
    x = (rng.standard_normal((B, R, N, T)) + 1j * rng.standard_normal((B, R, N, T))).astype(np.complex64)
xv = np.transpose(x, (0, 2, 3, 1))
h = C.plv_family(xv, input_kind=kind, bands=True)
d = C.plv_family(torch.from_numpy(x).cuda().permute(0, 2, 3, 1), input_kind=kind, bands=True)
print({m: bool(np.array_equal(h[m].values, d[m].values.cpu().numpy())) for m in ("plv", "iplv", "ciplv")})
