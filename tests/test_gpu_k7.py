"""K7 mask-count Gram (SPEC.md:260 per-pair effective T).

When samples are masked, T_ij = sum_t u_i(t) u_j(t) comes from one tcgen05
product of the 0/1 indicator planes (exact) and the metric epilogue keeps its
interior fast path.  Checked against the oracle (device path, both
precisions, every trial-reduce mode, over_trials, ragged N), against the
plane-scan fallback (PS_NO_K7=1, subprocess) bit for bit, and timed at
N = 4096, T = 16384 with every row masked: within 1.2x of the unmasked call.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import plv_oracle as O
from paper_1710_08037_b200 import connectivity as C

pytestmark = pytest.mark.gpu
METRICS = ("plv", "iplv", "ciplv")
TOL = {"split": 1e-5, "fp64": 1e-12}
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def masked_phasors(N, T, R, frac, seed, B=None):
    rng = np.random.default_rng(seed)
    shape = (N, T, R) if B is None else (B, N, T, R)
    z = np.exp(1j * rng.uniform(0, 2 * np.pi, size=shape))
    # shared component so that pairs are not all near-zero PLV
    src = np.exp(1j * rng.uniform(0, 2 * np.pi, size=shape[-2:]))
    z = 0.6 * z + 0.8 * src
    z /= np.abs(z)
    m = rng.uniform(size=shape) < frac
    # bursts too: contiguous masked runs in a few rows
    z[m] = 0
    idx = (slice(None),) * (z.ndim - 3)
    z[idx + (slice(3, 9), slice(100, 400))] = 0
    return z


def maxerr(a, b):
    return float(np.max(np.abs(np.asarray(a, dtype=np.float64) - b)))


@pytest.mark.parametrize("prec", ["split", "fp64"])
@pytest.mark.parametrize("reduce_", ["mean", "none", "pool"])
def test_k7_matches_oracle(prec, reduce_):
    z = masked_phasors(301, 1500, 3, 0.02, seed=100)
    ref = O.plv_family(z, input_kind="phasor", trial_reduce=reduce_)
    res = C.plv_family(z, input_kind="phasor", precision=prec, trial_reduce=reduce_)
    for m in METRICS:
        e = maxerr(res[m].values, ref[m])
        assert e <= TOL[prec], (prec, reduce_, m, e)
    assert res["plv"].meta["n_masked_samples"] == int(np.sum(z == 0))


def test_k7_bands_device_upper_and_over_trials():
    import torch

    z = masked_phasors(260, 700, 4, 0.05, seed=101, B=2)
    x = torch.from_numpy(z).cuda()
    res = C.plv_family(x, input_kind="phasor", bands=True, layout="upper")
    for b in range(2):
        ref = O.plv_family(z[b], input_kind="phasor")
        iu = np.triu_indices(260)
        for m in METRICS:
            got = res[m].values[b].cpu().numpy()
            assert maxerr(got[iu], ref[m][iu]) <= 1e-5, (b, m)
    zt = masked_phasors(130, 40, 64, 0.1, seed=102)
    ref = O.plv_family_over_trials(zt, zt == 0)
    got = C.plv_family(zt, input_kind="phasor", mode="over_trials")
    for m in METRICS:
        assert maxerr(got[m].values, ref[m]) <= 1e-5, m


_SCAN = r'''
import json, sys, numpy as np
sys.path.insert(0, {root!r})
from tests.test_gpu_k7 import masked_phasors
from paper_1710_08037_b200 import connectivity as C
z = masked_phasors(300, 2000, 2, 0.03, seed=103)
out = {{}}
for prec in ("split", "fp64"):
    r = C.plv_family(z, input_kind="phasor", precision=prec)
    np.save({path!r} + "_" + prec + ".npy", np.stack([np.asarray(r[m].values) for m in ("plv", "iplv", "ciplv")]))
'''


def test_k7_equals_plane_scan_bit_for_bit(tmp_path):
    res = {}
    for label, env_extra in (("k7", {}), ("scan", {"PS_NO_K7": "1"})):
        path = str(tmp_path / label)
        env = dict(os.environ, **env_extra)
        code = _SCAN.format(root=ROOT, path=path)
        subprocess.run([sys.executable, "-c", code], check=True, env=env, cwd=ROOT)
        res[label] = {p: np.load(path + "_" + p + ".npy") for p in ("split", "fp64")}
    for p in ("split", "fp64"):
        assert np.array_equal(res["k7"][p], res["scan"][p]), p


def test_k7_every_row_masked_n4096_t16384():
    import torch

    N, T = 4096, 16384
    rng = np.random.default_rng(104)
    ph = rng.uniform(0, 2 * np.pi, size=(N, T)).astype(np.float32)
    lat = rng.uniform(0, 2 * np.pi, size=(16, T)).astype(np.float32)
    ph = ph * 0.3 + lat[np.arange(N) % 16]
    z = np.exp(1j * ph).astype(np.complex64)
    zm = z.copy()
    zm[rng.uniform(size=(N, T)) < 0.01] = 0     # every row masked (~1% of its samples)
    zm[np.arange(N), rng.integers(0, T, size=N)] = 0
    xd = torch.from_numpy(z).cuda()[:, :, None]
    xm = torch.from_numpy(zm).cuda()[:, :, None]

    def timed(x):
        best = None
        for _ in range(4):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = C.plv_family(x, input_kind="phasor", precision="split")
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        return r, best

    _, t_plain = timed(xd)
    res, t_mask = timed(xm)
    assert res["plv"].meta["n_masked_samples"] == int(np.sum(zm == 0))
    rows = np.unique(np.concatenate([np.arange(0, 256), np.arange(N - 256, N), np.arange(2048, 2304)]))
    ref = O.plv_family_rows(zm[:, :, None], rows, "phasor")
    r = torch.as_tensor(rows, device="cuda")
    errs = {m: maxerr(res[m].values[r].double().cpu().numpy(), ref[m]) for m in METRICS}
    print(f"[k7] N={N} T={T} every row masked: unmasked {t_plain:.3f} ms, masked {t_mask:.3f} ms "
          f"(x{t_mask / t_plain:.3f}); rows={len(rows)} x all columns " +
          " ".join(f"{m}={e:.3e}" for m, e in errs.items()), flush=True)
    for m, e in errs.items():
        assert e <= 1e-5, (m, e)
    assert t_mask <= 1.2 * t_plain, (t_mask, t_plain)
