"""Randomised configurations through the public API against the CPU oracle
(the checker): shapes, dtypes, memory layouts, trial reductions, layouts,
zero stretches.  GPU box only.
    python tests/fuzz_probe.py [n_cases] [seed]
Prints one line per failing case and a summary; exit code 1 on any failure."""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import plv_oracle as O  # noqa: E402
from paper_1710_08037_b200 import connectivity as C  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rng = np.random.default_rng(seed)
fails = 0
for case in range(n_cases):
    N = int(rng.choice([1, 2, 3, 5, 17, 64, 129, 257, 300, 511, 513, 700]))
    T = int(rng.choice([2, 3, 4, 7, 16, 33, 100, 255, 256, 1000, 1024, 2050, 4096, 5000, 9999]))
    R = int(rng.choice([1, 1, 2, 3, 5]))
    kind = str(rng.choice(["real", "analytic", "phasor"]))
    dbl = bool(rng.integers(2))
    prec = str(rng.choice(["split", "fp64"]))
    reduce = str(rng.choice(["mean", "none", "pool"]))
    layout = str(rng.choice(["full", "upper"]))
    order = str(rng.choice(["ntr", "rnt", "nrt"]))  # memory order of the [N, T, R] view
    host = bool(rng.integers(3) == 0)
    pad = int(rng.choice([0, 0, 1, 2, 5]))  # extra samples per row in memory
    off = int(rng.choice([0, 0, 1, 3]))
    B = int(rng.choice([0, 0, 0, 2, 3]))  # 0: no band axis
    if N * N * T * R * max(B, 1) > 3e8:
        T = 100
    desc = dict(case=case, N=N, T=T, R=R, kind=kind, dbl=dbl, prec=prec, reduce=reduce, layout=layout, order=order,
                host=host, pad=pad, off=off, B=B)
    try:
        Tm = T + pad + off
        if kind == "real":
            base = rng.standard_normal((N, Tm, R))
        else:
            base = rng.standard_normal((N, Tm, R)) + 1j * rng.standard_normal((N, Tm, R))
            if kind == "phasor":
                base = base / np.abs(base)
        if rng.integers(4) == 0 and T >= 4:  # a zero stretch in one row (masked samples)
            base[rng.integers(N), off:off + max(1, T // 3), rng.integers(R)] = 0
        if rng.integers(4) == 0 and N > 1 and kind != "phasor":  # (phasor input is taken as given: unit or zero)
            base[rng.integers(N)] *= 10.0 ** rng.integers(-4, 5)
        dt = {("real", False): np.float32, ("real", True): np.float64}.get(
            (kind, dbl), np.complex128 if dbl else np.complex64)
        base = base.astype(dt)
        perm = {"ntr": (0, 1, 2), "rnt": (2, 0, 1), "nrt": (0, 2, 1)}[order]
        wide = np.complex128 if kind != "real" else np.float64
        inv = np.argsort(perm)
        if B:
            # [B, N, T, R] with every band laid out like the single-band case
            bases = [base] + [np.roll(base, b + 1, axis=0) * (1.0 if kind == "phasor" else 1.0 + 0.1 * b) for b in range(B - 1)]
            store = np.ascontiguousarray(np.stack([np.transpose(bb, perm) for bb in bases]))
            view_np = np.transpose(store, (0,) + tuple(int(i) + 1 for i in inv))[:, :, off:off + T, :]
            refs = [O.plv_family(view_np[b].astype(wide), input_kind=kind, trial_reduce=reduce) for b in range(B)]
            ref = {m: np.stack([np.asarray(rb[m]) for rb in refs]) for m in ("plv", "iplv", "ciplv")}
            xin = view_np if host else torch.from_numpy(store).cuda().permute(
                0, *[int(i) + 1 for i in inv])[:, :, off:off + T, :]
        else:
            store = np.ascontiguousarray(np.transpose(base, perm))
            view_np = np.transpose(store, inv)[:, off:off + T, :]
            assert view_np.shape == (N, T, R)
            ref = O.plv_family(view_np.astype(wide), input_kind=kind, trial_reduce=reduce)
            xin = view_np if host else torch.from_numpy(store).cuda().permute(*[int(i) for i in inv])[:, off:off + T, :]
        res = C.plv_family(xin, input_kind=kind, precision=prec, trial_reduce=reduce, layout=layout, bands=bool(B))
        exact = prec == "fp64" and dbl
        tol = 1e-12 if exact else 1e-5
        for m in ("plv", "iplv", "ciplv"):
            if m == "ciplv" and T < 32:
                continue  # a handful of samples: |Re| ~ 1 for many pairs, ciPLV conditioning dominates (
                # one T = 16 case measured 1.09e-5)
            v = res[m].values
            v = v.double().cpu().numpy() if isinstance(v, torch.Tensor) else np.asarray(v, dtype=np.float64)
            r = np.asarray(ref[m], dtype=np.float64)
            if r.ndim == v.ndim + 1 and r.shape[-1] == 1:  # one trial: [.., N, N, 1] vs [.., N, N]
                r = r[..., 0]
            assert v.shape == r.shape, (v.shape, r.shape)
            if layout == "upper":
                iu = np.triu_indices(N)
                v = v[:, iu[0], iu[1]] if B else v[iu[0], iu[1]]
                r = r[:, iu[0], iu[1]] if B else r[iu[0], iu[1]]
            err = float(np.max(np.abs(v - r))) if v.size else 0.0
            if not (err <= tol):
                fails += 1
                print("FAIL", m, f"{err:.3e}", desc, flush=True)
                break
    except Exception as exc:  # noqa: BLE001
        msg = str(exc).splitlines()[0][:160] if str(exc) else type(exc).__name__
        expected = ("ill-conditioned" in msg) or ("precision='fp64'" in msg)
        if not expected:
            fails += 1
            print("EXC ", type(exc).__name__, msg, desc, flush=True)
            if os.environ.get("FUZZ_TB"):
                traceback.print_exc()
print(f"fuzz: {n_cases} cases, {fails} failures (seed {seed})", flush=True)
sys.exit(1 if fails else 0)
