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
bands = x.ndim == 4
tdt = {"c64": torch.complex64, "f32": torch.float32, "f64": torch.float64}[dt]
if bands:  # [B, N, T, R] -> trials-outer storage [B, R, N, T]
    pin = torch.empty((B, R, N, T), dtype=tdt, pin_memory=True).numpy()
    pin[...] = np.transpose(x, (0, 3, 1, 2))
    xv = np.transpose(pin, (0, 2, 3, 1))
else:
    pin = torch.empty((R, N, T), dtype=tdt, pin_memory=True).numpy()
    pin[...] = np.transpose(x, (2, 0, 1))
    xv = np.transpose(pin, (1, 2, 0))
del x
outs = {m: torch.zeros((B, N, N), dtype=torch.float32, pin_memory=True).numpy() for m in ("plv", "iplv", "ciplv")}
res = C.plv_family(xv, input_kind=kind, out=outs, layout=layout, bands=bands)
meta = {k: res["plv"].meta[k] for k in ("n_refined_pairs", "n_kernel_launches", "h2d_bytes", "d2h_bytes")}
ts = []
for _ in range(int(os.environ.get("E2E_REPS", "3"))):
    t0 = time.perf_counter()
    C.plv_family(xv, input_kind=kind, out=outs, layout=layout, bands=bands)
    ts.append(time.perf_counter() - t0)
print(json.dumps({"cfg": cfg, "layout": layout, "env": {k: v for k, v in os.environ.items() if k.startswith("PS_")},
                  "ms": [round(t * 1e3, 2) for t in ts],
                  "pair_samples_per_s": W.pair_samples(N, T, R, B) / min(ts), "meta": meta}), flush=True)
