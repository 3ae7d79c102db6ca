"""Times the host (e2e) entry point on C5 with pinned numpy buffers for the
current PS_* environment; one JSON line.  GPU box only."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1710_08037_b200 import connectivity as C  # noqa: E402
from paper_1710_08037_b200 import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
layout = sys.argv[2] if len(sys.argv) > 2 else ("upper" if cfg == "c5" else "full")
x = W.generate(cfg)
N, T, R, B, dt, kind = W.CONFIGS[cfg]
pin = torch.empty(x.shape[::-1][:0] + (R, N, T), dtype={"c64": torch.complex64, "f32": torch.float32,
                                                          "f64": torch.float64}[dt], pin_memory=True).numpy()
pin[...] = np.transpose(x, (2, 0, 1))
xv = np.transpose(pin, (1, 2, 0))
outs = {m: torch.zeros((1, N, N), dtype=torch.float32, pin_memory=True).numpy() for m in ("plv", "iplv", "ciplv")}
res = C.plv_family(xv, input_kind=kind, out=outs, layout=layout)
meta = {k: res["plv"].meta[k] for k in ("n_refined_pairs", "n_kernel_launches", "h2d_bytes", "d2h_bytes")}
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    C.plv_family(xv, input_kind=kind, out=outs, layout=layout)
    ts.append(time.perf_counter() - t0)
print(json.dumps({"cfg": cfg, "layout": layout, "env": {k: v for k, v in os.environ.items() if k.startswith("PS_")},
                  "ms": [round(t * 1e3, 2) for t in ts],
                  "pair_samples_per_s": W.pair_samples(N, T, R, B) / min(ts), "meta": meta}), flush=True)
