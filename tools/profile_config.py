"""Runs the hot path a few times on one (optionally reduced) config -- the
command the ncu captures in profiles/ wrap.  GPU box only.
    python tools/profile_config.py c4 --bands 1 --iters 3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1710_08037_b200 import connectivity as C  # noqa: E402
from paper_1710_08037_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--bands", type=int, default=0)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--precision", default="split")
args = ap.parse_args()
kw = {}
if args.config == "c4" and args.bands:
    kw["bands"] = W.C4_BANDS[: args.bands]
x = W.generate(args.config, **kw)
N, T, R, B, dt, kind = W.CONFIGS[args.config]
bands = x.ndim == 4
store = np.ascontiguousarray(np.transpose(x, (2, 0, 1)) if not bands else np.transpose(x, (0, 3, 1, 2)))
xd = torch.from_numpy(store).cuda()
xv = xd.permute(1, 2, 0) if not bands else xd.permute(0, 2, 3, 1)
for _ in range(args.iters):
    r = C.plv_family(xv, input_kind=kind, bands=bands, precision=args.precision, timing=True)
    print({k: r["plv"].meta[k] for k in ("ms_normalize", "ms_gram", "ms_finish", "n_refined_pairs")}, flush=True)
torch.cuda.synchronize()
