"""Time-resolved PLV (mode over_trials, Eq 8) throughput probe: device-resident
unit phasors [N, T, R] -> N x N x T outputs for PLV / iPLV / ciPLV.  Reports
the output bandwidth (the regime's bound: N^2 T outputs per metric) next to
the Gram work.  GPU box only.
    python tools/over_trials_probe.py N T R [full|upper]
(PS_DEBUG_EPI=4 / 8 / 12 skip the mirror / direct / both stores: experiments.)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1710_08037_b200 import connectivity as C  # noqa: E402

N, T, R = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (1024, 512, 64)
layout = sys.argv[4] if len(sys.argv) > 4 else "full"
g = torch.Generator(device="cuda").manual_seed(0)
ph = torch.rand((R, N, T), device="cuda", generator=g) * 6.283185307179586
z = torch.polar(torch.ones_like(ph), ph).to(torch.complex64).permute(1, 2, 0)  # [N, T, R] view
outs = {m: torch.empty((T, N, N), device="cuda") for m in ("plv", "iplv", "ciplv")}
for _ in range(2):
    C.plv_family(z, input_kind="phasor", mode="over_trials", out=outs, layout=layout)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 3
e0.record()
for _ in range(reps):
    r = C.plv_family(z, input_kind="phasor", mode="over_trials", out=outs, timing=True, layout=layout)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
out_bytes = 3 * (N * N if layout == "full" else N * (N + 1) // 2) * T * 4
print(json.dumps({"N": N, "T": T, "R": R, "layout": layout, "debug_epi": os.environ.get("PS_DEBUG_EPI", "0"), "ms": ms, "gram_ms": r["plv"].meta["ms_gram"],
                  "output_GBps": out_bytes / ms / 1e6,
                  "pair_samples_per_s": N * (N - 1) / 2 * T * R / ms * 1e3}))
