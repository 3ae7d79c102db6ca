"""Parity at BASELINE config scale (VERDICT r1 "next" #1).

The GPU runs every config at its FULL size; the CPU oracle (oracle/plv_oracle.py
plv_family_rows, FP64 / complex128) computes a structured row subset against
ALL columns:
  * rows 0-255 (the first 256-row panel),
  * the last, partial panel (C5: rows 19968-19999, since 20000 = 78 * 256 + 32),
  * one whole 256-row band in the middle,
so every column tile and the ragged edge are checked, not a random sample.
Both precisions: split (tcgen05 fp16 x 3) at 1e-5 and FP64 (DMMA) at 1e-12.
The C5 end-to-end host path (numpy pinned input -> ps_plv_family_host, upper
layout, streamed copy-out, refined entries patched on the host) must equal the
device path bit for bit, and the upper layout is the one checked for C5.
Errors are printed as "[scale-parity] ..." lines (kept in profiles/).
"""
import numpy as np
import pytest

from oracle import plv_oracle as O
from paper_1710_08037_b200 import connectivity as C
from paper_1710_08037_b200 import workloads as W

pytestmark = pytest.mark.gpu

METRICS = ("plv", "iplv", "ciplv")
TOL = {"split": 1e-5, "fp64": 1e-12}
PANEL = 256


def subset_rows(N):
    first = np.arange(0, min(PANEL, N))
    tail = N % PANEL or PANEL
    last = np.arange(N - tail, N)
    mid0 = (N // PANEL // 2) * PANEL
    mid = np.arange(mid0, min(N, mid0 + PANEL))
    return np.unique(np.concatenate([first, mid, last]))


def rows_of(mat, rows, upper):
    """Rows `rows` x all columns of a device matrix [N, N]; for the upper
    layout the entries j < i are read from (j, i)."""
    import torch

    r = torch.as_tensor(rows, device=mat.device)
    out = mat[r, :]
    if upper:
        N = mat.shape[0]
        lower = torch.arange(N, device=mat.device)[None, :] < r[:, None]
        out = torch.where(lower, mat[:, r].T, out)
    return out.double().cpu().numpy()


def report(label, prec, rows, errs):
    print(f"[scale-parity] {label} {prec} rows={len(rows)} x all columns " +
          " ".join(f"{m}={e:.3e}" for m, e in errs.items()), flush=True)


def check(label, prec, res, ref, rows, upper=False):
    errs = {}
    for m in METRICS:
        got = rows_of(res[m], rows, upper)
        errs[m] = float(np.max(np.abs(got - ref[m])))
    report(label, prec, rows, errs)
    for m, e in errs.items():
        assert e <= TOL[prec], (label, prec, m, e)


@pytest.fixture(scope="module")
def c5_case():
    x = W.c5()                                              # [20000, 16384, 1] complex64
    rows = subset_rows(x.shape[0])
    assert rows[-1] == 19999 and 19968 in rows and 0 in rows
    ref = O.plv_family_rows(x, rows, "analytic")
    return x, rows, ref


def test_c5_e2e_host_path_full_size(c5_case):
    """C5 at 20000 x 16384: device path (upper layout) vs the host e2e path the
    headline e2e number runs through -- bit-identical -- and vs the oracle."""
    import torch

    x, rows, ref = c5_case
    N = x.shape[0]
    xd = torch.from_numpy(np.ascontiguousarray(x[:, :, 0])).cuda()[:, :, None]
    dev = C.plv_family(xd, input_kind="analytic", precision="split", layout="upper")
    dres = {m: dev[m].values for m in METRICS}
    check("c5-device-upper", "split", dres, ref, rows, upper=True)
    del xd
    # e2e: numpy pinned input, host outputs, the streamed row-band copy-out
    xin = torch.empty((N, x.shape[1]), dtype=torch.complex64, pin_memory=True)
    xin.numpy()[...] = x[:, :, 0]
    hout = {m: torch.zeros((1, N, N), dtype=torch.float32, pin_memory=True).numpy() for m in METRICS}
    host = C.plv_family(xin.numpy()[:, :, None], input_kind="analytic", precision="split", layout="upper",
                        out=hout)
    meta = host["plv"].meta
    print(f"[scale-parity] c5-e2e h2d={meta['h2d_bytes']} d2h={meta['d2h_bytes']} "
          f"refined={meta['n_refined_pairs']}", flush=True)
    for m in METRICS:
        h = torch.from_numpy(hout[m][0]).cuda()
        same = torch.equal(h, dres[m])
        if not same:
            iu = torch.triu_indices(N, N, device=h.device)
            diff = (h[iu[0], iu[1]] - dres[m][iu[0], iu[1]]).abs().max().item()
            pytest.fail(f"c5 e2e {m}: host path differs from the device path (max |diff| {diff:.3e})")
        del h
    print("[scale-parity] c5-e2e host path == device path (bit-identical, all 3 metrics, 20000 x 20000 upper)",
          flush=True)


def test_c5_fp64_full_size(c5_case):
    import torch

    x, rows, ref = c5_case
    xd = torch.from_numpy(np.ascontiguousarray(x[:, :, 0])).cuda()[:, :, None]
    dev = C.plv_family(xd, input_kind="analytic", precision="fp64", layout="upper")
    check("c5-device-upper", "fp64", {m: dev[m].values for m in METRICS}, ref, rows, upper=True)


def _device_input(x):
    """[N, T, R] host (strided view of [R, N, T]) -> CUDA view with the same layout."""
    import torch

    store = np.ascontiguousarray(np.transpose(x, (2, 0, 1)))
    return torch.from_numpy(store).cuda().permute(1, 2, 0)


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_full_size_configs_both_precisions(cfg):
    N, T, R, B, dt, kind = W.CONFIGS[cfg]
    x = W.generate(cfg)
    rows = subset_rows(N)
    ref = O.plv_family_rows(x, rows, kind)
    xd = _device_input(x)
    for prec in ("split", "fp64"):
        res = C.plv_family(xd, input_kind=kind, precision=prec)
        check(f"{cfg}-device", prec, {m: res[m].values for m in METRICS}, ref, rows)
    if cfg == "c2":
        # the trial-group pipelined host path (numpy input) equals the device path
        import torch

        dres = C.plv_family(xd, input_kind=kind, precision="split")
        hres = C.plv_family(np.asarray(x), input_kind=kind, precision="split")
        for m in METRICS:
            assert torch.equal(torch.from_numpy(np.ascontiguousarray(hres[m].values)).cuda(), dres[m].values), m
        print("[scale-parity] c2 host path == device path (bit-identical)", flush=True)


def test_full_size_c4_band_both_precisions():
    # one C4 band at full size (2500 x 4096 x 60 trials, fp32 real, trial mean)
    N, T, R, B, dt, kind = W.CONFIGS["c4"]
    x = W.c4(bands=W.C4_BANDS[1:2])[0]                  # [N, T, R] view of [R, N, T]
    rows = subset_rows(N)
    ref = O.plv_family_rows(x, rows, "real")
    xd = _device_input(x)
    for prec in ("split", "fp64"):
        res = C.plv_family(xd, input_kind="real", precision=prec)
        check("c4-band1-device", prec, {m: res[m].values for m in METRICS}, ref, rows)
