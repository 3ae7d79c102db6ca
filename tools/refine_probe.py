"""Cost of the ill-conditioned ciPLV refinement at scale: clusters of signals
sharing one zero-lag source (volume-conduction-like leakage), so every
within-cluster pair has |Re| close to 1.  Reports the stage times and the
number of refined pair-rounds.  GPU box only.
    python tools/refine_probe.py [N] [T] [cluster]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1710_08037_b200 import connectivity as C  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
T = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
K = int(sys.argv[3]) if len(sys.argv) > 3 else 64
g = torch.Generator(device="cuda").manual_seed(0)
src = torch.randn((N // K + 1, T), device="cuda", dtype=torch.complex64, generator=g)
lab = torch.arange(N, device="cuda") // K
a = src[lab] + 0.05 * torch.randn((N, T), device="cuda", dtype=torch.complex64, generator=g)
x = a.unsqueeze(-1)  # [N, T, 1]
for _ in range(2):
    r = C.plv_family(x, input_kind="analytic", timing=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
r = C.plv_family(x, input_kind="analytic", timing=True)
e1.record()
torch.cuda.synchronize()
m = r["plv"].meta
print(json.dumps({"N": N, "T": T, "cluster": K, "ms_call": e0.elapsed_time(e1), "ms_gram": m["ms_gram"],
                  "ms_finish": m["ms_finish"], "refined": m["n_refined_pairs"]}))
