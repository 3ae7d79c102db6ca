"""The split Gram's producer lockstep under a concurrently busy GPU: the same
call with and without a side stream of large matmuls; results must match
bit-for-bit and the time stay sane.  GPU box only."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1710_08037_b200 import connectivity as C  # noqa: E402

N, T = 8192, 4096
g = torch.Generator(device="cuda").manual_seed(0)
ph = torch.rand((1, N, T), device="cuda", generator=g) * 6.283185307179586
z = torch.polar(torch.ones_like(ph), ph).to(torch.complex64).permute(1, 2, 0)
ref = C.plv_family(z, input_kind="phasor")
torch.cuda.synchronize()
t0 = time.perf_counter()
ref = C.plv_family(z, input_kind="phasor")
torch.cuda.synchronize()
t_alone = time.perf_counter() - t0
side = torch.cuda.Stream()
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
with torch.cuda.stream(side):
    for _ in range(200):
        a = (a @ a) * 1e-3
t0 = time.perf_counter()
got = C.plv_family(z, input_kind="phasor")
torch.cuda.synchronize()
t_busy = time.perf_counter() - t0
same = all(torch.equal(got[m].values, ref[m].values) for m in ("plv", "iplv", "ciplv"))
print(json.dumps({"alone_ms": t_alone * 1e3, "with_side_matmuls_ms": t_busy * 1e3, "bit_identical": same}))
