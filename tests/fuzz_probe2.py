"""Randomised cases for the time-resolved mode (Eq 8) and the analytic-signal /
band-pass front end against the CPU oracle (the checker).  GPU box only.
    python tests/fuzz_probe2.py [n_cases] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import plv_oracle as O  # noqa: E402
from paper_1710_08037_b200 import connectivity as C  # noqa: E402
from paper_1710_08037_b200 import signalprep  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rng = np.random.default_rng(seed)
fails = 0
for case in range(n_cases):
    which = str(rng.choice(["over_trials", "analytic", "bandpass"]))
    dbl = bool(rng.integers(2))
    host = bool(rng.integers(2))
    desc = dict(case=case, which=which, dbl=dbl, host=host)
    try:
        if which == "over_trials":
            N = int(rng.choice([2, 5, 33, 129, 260]))
            T = int(rng.choice([2, 3, 16, 40, 65]))
            R = int(rng.choice([2, 5, 16, 37, 64, 130]))
            prec = str(rng.choice(["split", "fp64"]))
            layout = str(rng.choice(["full", "upper"]))
            desc.update(N=N, T=T, R=R, prec=prec, layout=layout)
            a = rng.standard_normal((N, T, R)) + 1j * rng.standard_normal((N, T, R))
            a[:: max(1, N // 4)] *= np.exp(1j * rng.uniform(0, np.pi, (1, T, 1)))
            if rng.integers(2) and R > 4:
                a[rng.integers(N), rng.integers(T), :3] = 0
            a = a.astype(np.complex128 if dbl else np.complex64)
            z, mask = O.normalize_phasors(a.astype(np.complex128))
            ref = O.plv_family_over_trials(z, mask)
            xin = a if host else torch.from_numpy(a).cuda()
            res = C.plv_family(xin, input_kind="analytic", precision=prec, mode="over_trials", layout=layout)
            tol = 1e-12 if (prec == "fp64" and dbl) else 1e-5
            for m in ("plv", "iplv", "ciplv"):
                if m == "ciplv" and R < 16:
                    continue
                v = res[m].values
                v = v.double().cpu().numpy() if isinstance(v, torch.Tensor) else np.asarray(v, dtype=np.float64)
                r = np.asarray(ref[m])
                assert v.shape == r.shape, (v.shape, r.shape)
                if layout == "upper":
                    iu = np.triu_indices(N)
                    v, r = v[iu[0], iu[1]], r[iu[0], iu[1]]
                err = float(np.max(np.abs(v - r)))
                if not err <= tol:
                    fails += 1
                    print("FAIL", m, f"{err:.3e}", desc, flush=True)
                    break
        else:
            N = int(rng.choice([1, 3, 17, 40]))
            T = int(rng.choice([64, 101, 256, 1000, 1024, 1201, 2048, 3000, 4096]))
            R = int(rng.choice([1, 2, 3]))
            desc.update(N=N, T=T, R=R)
            x = rng.standard_normal((N, T, R))
            if rng.integers(2) and N > 1:
                x[rng.integers(N)] *= 10.0 ** rng.integers(-5, 6)
            x = x.astype(np.float64 if dbl else np.float32)
            xin = x if host else torch.from_numpy(x).cuda()
            if which == "analytic":
                ar = O.analytic_signal(x.astype(np.float64), axis=1)
                a = signalprep.analytic_signal(xin).data
            else:
                order = int(rng.choice([o for o in (20, 50, 100) if o + 1 < T]))
                pad = int(rng.choice([0, 7, 30, min(T - 1, 200)]))
                lo, hi = sorted(rng.uniform(0.05, 0.9, 2))
                if hi - lo < 0.05:
                    hi = min(0.95, lo + 0.1)
                desc.update(order=order, pad=pad, band=(round(lo, 3), round(hi, 3)))
                f = signalprep.design_bandpass_fir((lo * np.pi, hi * np.pi), order)
                ar = O.bandpass_analytic(x.astype(np.float64), f.taps, pad)
                a = signalprep.analytic_signal(xin, fir=f, pad_samples=pad).data
            a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
            assert a.shape == ar.shape, (a.shape, ar.shape)
            if which == "analytic" and not np.array_equal(a.real, x):
                fails += 1
                print("FAIL Re(a) != x", desc, flush=True)
                continue
            scale = np.max(np.abs(ar), axis=(1, 2))
            scale[scale == 0] = 1.0
            rel = float(np.max(np.max(np.abs(a - ar), axis=(1, 2)) / scale))
            tol = 1e-12 if dbl else 3e-6
            if not rel <= tol:
                fails += 1
                print("FAIL", f"{rel:.3e}", desc, flush=True)
    except Exception as exc:  # noqa: BLE001
        fails += 1
        print("EXC ", type(exc).__name__, str(exc).splitlines()[0][:200] if str(exc) else "", desc, flush=True)
print(f"fuzz2: {n_cases} cases, {fails} failures (seed {seed})", flush=True)
sys.exit(1 if fails else 0)
