"""Small calls through every entry point, meant to run under
`compute-sanitizer --tool memcheck` (and racecheck / synccheck) on the GPU box:
device / host / pipelined (column and streamed row stages) / staged /
device-to-host paths, split and fp64, real (fused T=4096,
cuFFT odd T, band-pass), analytic, phasor, time-resolved, coherence."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1710_08037_b200 import connectivity as C  # noqa: E402
from paper_1710_08037_b200 import sharding, signalprep  # noqa: E402

rng = np.random.default_rng(0)
x = rng.standard_normal((40, 1001, 2)).astype(np.float32)
for prec in ("split", "fp64"):
    C.plv_family(x, input_kind="real", precision=prec)
x4 = rng.standard_normal((2, 33, 4096)).astype(np.float32).transpose(1, 2, 0)
C.plv_family(x4, input_kind="real")
z = np.exp(1j * rng.uniform(0, 6.3, (300, 64, 3))).astype(np.complex64)
for red in ("mean", "none", "pool"):
    C.plv_family(z, input_kind="phasor", trial_reduce=red, metrics=("plv", "iplv", "ciplv", "cre", "cim"))
C.plv_family(z, input_kind="phasor", mode="over_trials")
f = signalprep.design_bandpass_fir((0.2, 0.6), 60)
C.plv_family(x[:10], input_kind="real", fir=f, pad_samples=100)
signalprep.filter_two_pass(x[:5], f, 99)
C.coherence_matrix(x[:12], C.WelchConfig(128, 64), (0.2, 1.0), mode="max", metrics=("coh", "icoh"))
C.coherence_matrix(x[:12], C.WelchConfig(128, 64), (0.2, 1.0), mode="mean")
# pipelined host path (N >= 2048, >= 148 tiles) with bands and trials, small T
xb = rng.standard_normal((2, 2, 2304, 32)).astype(np.float32)
C.plv_family(np.transpose(xb, (0, 2, 3, 1)), input_kind="real", bands=True)
# staged device path
a = torch.from_numpy((rng.standard_normal((2600, 64)) + 1j * rng.standard_normal((2600, 64))).astype(np.complex64))
a = a.cuda()
cols = sharding.stage_cols(2600, n_stages=3, min_width=512)
C.plv_family(a, input_kind="analytic", stages=(cols, [None] * (len(cols) - 1)), shard=(1, 2))
# streamed host path (upper layout, row stages, device-published band flags),
# sharded, bands + trial mean, fp64 (event-released bands)
C.plv_family(np.transpose(xb, (0, 2, 3, 1)), input_kind="real", bands=True, layout="upper")
xs = rng.standard_normal((2304, 48)).astype(np.float32)
C.plv_family(xs, input_kind="real", layout="upper", shard=(1, 2))
C.plv_family(xs.astype(np.float64), input_kind="real", layout="upper", precision="fp64")
# device input -> host outputs (ps_plv_family_to_host), streamed and not
outs = {m: np.zeros((1, 2600, 2600), np.float32) for m in ("plv", "iplv", "ciplv")}
C.plv_family(a, input_kind="analytic", layout="upper", out=outs)
C.plv_family(a, input_kind="analytic", layout="full", out=outs)
torch.cuda.synchronize()
print("sanitize smoke done")
