"""Normalise-stage timing (real fp32 input -> split planes) for several T, to
compare the fused Hilbert kernels with the cuFFT chain (run once plain and
once with PS_HILBERT=cufft).  GPU box only.
    python tools/hilbert_probe.py [T ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1710_08037_b200 import connectivity as C  # noqa: E402

Ts = [int(v) for v in sys.argv[1:]] or [1000, 2000, 2500, 4096, 5000, 8000, 10000, 12000]
for T in Ts:
    rows = max(2, (1 << 26) // T)  # ~67 M samples per call
    R = 4
    N = rows // R
    x = torch.randn((R, N, T), device="cuda").permute(1, 2, 0)
    outs = {"plv": torch.empty((1, N, N), device="cuda")}
    for _ in range(2):
        C.plv_family(x, input_kind="real", metrics=("plv",), out=outs, timing=True)
    ms = []
    for _ in range(3):
        r = C.plv_family(x, input_kind="real", metrics=("plv",), out=outs, timing=True)
        ms.append(r["plv"].meta["ms_normalize"])
    ms.sort()
    print(json.dumps({"T": T, "samples": N * R * T, "ms_normalize": ms[1],
                      "GB_per_s_at_12B": N * R * T * 12 / ms[1] / 1e6,
                      "hilbert": os.environ.get("PS_HILBERT", "fused")}), flush=True)
