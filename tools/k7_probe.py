"""K7 timing probe (GPU box): N x T phasors, unmasked vs every row masked,
device path, per-stage times.  python tools/k7_probe.py [N] [T] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1710_08037_b200 import connectivity as C  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
T = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
rng = np.random.default_rng(104)
ph = rng.uniform(0, 2 * np.pi, size=(N, T)).astype(np.float32)
z = np.exp(1j * ph).astype(np.complex64)
zm = z.copy()
zm[rng.uniform(size=(N, T)) < 0.01] = 0
xd = torch.from_numpy(z).cuda()[:, :, None]
xm = torch.from_numpy(zm).cuda()[:, :, None]
for label, x in (("plain", xd), ("masked", xm)):
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = C.plv_family(x, input_kind="phasor", precision="split", timing=True)
        e1.record()
        e1.synchronize()
        mt = r["plv"].meta
        print(f"{label:7s} total {e0.elapsed_time(e1):7.3f} ms  norm {mt['ms_normalize']:.3f}  gram {mt['ms_gram']:.3f}  "
              f"finish {mt['ms_finish']:.3f}  variant {mt['gram_variant']}  launches {mt['n_kernel_launches']}",
              flush=True)
