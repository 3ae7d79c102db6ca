"""Per-step stage times of the device path for one config (jitter check).
    python tools/step_jitter.py c2 [steps]   (GPU box only)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1710_08037_b200 import connectivity as C  # noqa: E402
from paper_1710_08037_b200 import workloads as W  # noqa: E402

cfg = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
N, T, R, B, dt, kind = W.CONFIGS[cfg]
x = W.generate(cfg)
bands = x.ndim == 4
store = np.ascontiguousarray(np.transpose(x, (2, 0, 1)) if not bands else np.transpose(x, (0, 3, 1, 2)))
xd = torch.from_numpy(store).cuda()
xv = xd.permute(1, 2, 0) if not bands else xd.permute(0, 2, 3, 1)
outs = {m: torch.empty((B, N, N), device="cuda") for m in ("plv", "iplv", "ciplv")}
for _ in range(3):
    C.plv_family(xv, input_kind=kind, bands=bands, out=outs)
import time  # noqa: E402

rows = []
for _ in range(steps):
    t0 = time.perf_counter()
    r = C.plv_family(xv, input_kind=kind, bands=bands, out=outs, timing=True)
    wall = (time.perf_counter() - t0) * 1e3
    m = r["plv"].meta
    rows.append((m["ms_normalize"], m["ms_gram"], m["ms_finish"], wall))
g = [r[1] for r in rows]
print(json.dumps({"cfg": cfg, "env": {k: v for k, v in os.environ.items() if k.startswith("PS_")},
                  "gram_ms": [round(v, 3) for v in g], "min": min(g), "median": float(np.median(g)), "max": max(g),
                  "wall_ms": [round(r[3], 2) for r in rows], "norm_ms": [round(r[0], 3) for r in rows],
                  "finish_ms": [round(r[2], 3) for r in rows]}))
