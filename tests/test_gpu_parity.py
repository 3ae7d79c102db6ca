"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Tolerances (north star): max-abs <= 1e-5 for the split-precision path,
<= 1e-12 for the FP64 mode.  Full-size configs are checked through
size-independent properties plus exact oracle recomputation on random signal
subsets (a PLV-family entry depends only on its two rows).
"""
import os

import numpy as np
import pytest

from oracle import plv_oracle as O
from paper_1710_08037_b200 import connectivity as C
from paper_1710_08037_b200 import errors, signalprep
from paper_1710_08037_b200 import workloads as W

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(__file__), "golden")
TOL = {"split": 1e-5, "fp64": 1e-12}
METRICS = ("plv", "iplv", "ciplv")


def golden(name):
    return np.load(os.path.join(G, name + ".npz"), allow_pickle=False)


def maxerr(got, ref):
    return float(np.max(np.abs(np.asarray(got, dtype=np.float64) - ref)))


def check(res, ref, prec, label=""):
    errs = {m: maxerr(res[m].values, ref[m]) for m in METRICS}
    print(f"[parity] {label} {prec} " + " ".join(f"{m}={e:.3e}" for m, e in errs.items()))
    for m, e in errs.items():
        assert e <= TOL[prec], (label, prec, m, e)


# ------------------------------------------------------------ golden configs
@pytest.mark.parametrize("prec", ["split", "fp64"])
@pytest.mark.parametrize("name", ["c1_full", "c2_small", "c3_small", "c5_small"])
def test_golden_configs(name, prec):
    d = golden(name)
    res = C.plv_family(d["x"], input_kind=str(d["input_kind"]), precision=prec,
                       trial_reduce=str(d["trial_reduce"]))
    check(res, {m: d[m] for m in METRICS}, prec, name)


@pytest.mark.parametrize("prec", ["split", "fp64"])
def test_golden_c4_bands(prec):
    d = golden("c4_small")
    res = C.plv_family(d["x"], input_kind="real", precision=prec, bands=True)
    check(res, {m: d[m] for m in METRICS}, prec, "c4_small")


@pytest.mark.parametrize("prec", ["split", "fp64"])
def test_kat_offsets(prec):
    d = golden("kat_offsets")
    res = C.plv_family(d["z"], input_kind="phasor", precision=prec)
    check(res, {m: d[m] for m in METRICS}, prec, "kat_offsets")
    # zero-lag pairs hit the singularity rule exactly
    assert float(res["ciplv"].values[0, 0]) == 0.0


def test_kat_cancel():
    d = golden("kat_cancel")
    for prec in ("split", "fp64"):
        v = C.plv_matrix(d["z"], precision=prec).values
        assert abs(float(v[0, 1])) < TOL[prec]


# ------------------------------------------------------------ API surfaces
def test_host_and_device_paths_bit_identical():
    import torch

    x = W.c1()
    h = C.plv_family(x, precision="split")
    dv = C.plv_family(torch.from_numpy(x).cuda(), precision="split")
    for m in METRICS:
        assert np.array_equal(h[m].values, dv[m].values.cpu().numpy())


@pytest.mark.parametrize("kind", ["analytic", "real"])
def test_pipelined_host_path_matches_device_path(kind):
    # N >= 2048 with enough tiles takes the staged copy-in / Gram / copy-out
    # pipeline of ps_plv_family_host; it must equal the device path bit-exactly
    import torch

    rng = np.random.default_rng(11)
    N, T = 3000, 256
    if kind == "analytic":
        x = (rng.standard_normal((N, T)) + 1j * rng.standard_normal((N, T))).astype(np.complex64)
    else:
        x = rng.standard_normal((N, T)).astype(np.float32)
    x[5, :7] = 0  # masked samples on the pipelined path too
    h = C.plv_family(x, input_kind=kind, precision="split")
    d = C.plv_family(torch.from_numpy(x).cuda(), input_kind=kind, precision="split")
    for m in METRICS:
        assert np.array_equal(h[m].values, d[m].values.cpu().numpy()), m
    idx = np.sort(rng.choice(N, size=120, replace=False))
    idx[0] = 5
    ref = O.plv_family(x[idx][:, :, None], input_kind=kind)
    for m in METRICS:
        assert maxerr(h[m].values[np.ix_(idx, idx)], ref[m]) <= TOL["split"], m


@pytest.mark.parametrize("kind", ["analytic", "real"])
def test_pipelined_host_path_bands_and_trials(kind):
    # the pipelined host path with several (band, trial) units and trial means:
    # output slots per band (regression: they were sized for one slot)
    import torch

    rng = np.random.default_rng(13)
    B, R, N, T = 2, 3, 2304, 256
    if kind == "analytic":
        x = (rng.standard_normal((B, R, N, T)) + 1j * rng.standard_normal((B, R, N, T))).astype(np.complex64)
    else:
        x = rng.standard_normal((B, R, N, T)).astype(np.float32)
    xv = np.transpose(x, (0, 2, 3, 1))
    h = C.plv_family(xv, input_kind=kind, bands=True)
    assert h["plv"].values.shape == (B, N, N)
    if kind == "analytic":  # same planes on both paths: bit-identical
        d = C.plv_family(torch.from_numpy(x).cuda().permute(0, 2, 3, 1), input_kind=kind, bands=True)
        for m in METRICS:
            assert np.array_equal(h[m].values, d[m].values.cpu().numpy()), m
    idx = np.sort(rng.choice(N, size=64, replace=False))
    for b in range(B):
        ref = O.plv_family(xv[b][idx], input_kind=kind)
        for m in METRICS:
            assert maxerr(h[m].values[b][np.ix_(idx, idx)], ref[m]) <= TOL["split"], (b, m)


@pytest.mark.parametrize("prec,reduce_", [("fp64", "mean"), ("split", "none"), ("split", "pool"), ("fp64", "none")])
def test_pipelined_host_path_variants(prec, reduce_):
    # precision / trial-reduce combinations of the pipelined host path against
    # the device path (same planes, same kernels: bit-identical) and the oracle
    import torch

    rng = np.random.default_rng(14)
    R, N, T = 2, 3072, 96  # N >= 2048 and >= 148 output tiles: the pipelined path
    from paper_1710_08037_b200 import _native

    assert _native.tile_count(N, prec) >= 148
    z = np.exp(1j * rng.uniform(0, 2 * np.pi, (R, N, T))).astype(np.complex128)
    z[:, ::50] *= np.exp(1j * 0.3)
    zv = np.transpose(z, (1, 2, 0))
    metrics = ("plv", "iplv", "ciplv", "cre", "cim")
    h = C.plv_family(zv, input_kind="phasor", precision=prec, trial_reduce=reduce_, metrics=metrics)
    d = C.plv_family(torch.from_numpy(z).cuda().permute(1, 2, 0), input_kind="phasor", precision=prec,
                     trial_reduce=reduce_, metrics=metrics)
    for m in metrics:
        assert np.array_equal(h[m].values, d[m].values.cpu().numpy()), m
    idx = np.sort(rng.choice(N, size=48, replace=False))
    ref = O.plv_family(zv[idx], input_kind="phasor", trial_reduce=reduce_)
    for m in METRICS:
        got = h[m].values[np.ix_(idx, idx)] if reduce_ != "none" else h[m].values[np.ix_(idx, idx)]
        assert maxerr(got, ref[m]) <= TOL[prec], m


def test_staged_input_matches_device_path():
    # ps_plv_family_staged: rows arrive chunk by chunk (here: async copies on a
    # side stream standing in for the per-chunk NCCL broadcast of N>1 runs)
    import torch

    from paper_1710_08037_b200 import sharding

    rng = np.random.default_rng(12)
    N, T = 2600, 512
    x = (rng.standard_normal((N, T)) + 1j * rng.standard_normal((N, T))).astype(np.complex64)
    ref = C.plv_family(torch.from_numpy(x).cuda(), input_kind="analytic")
    src = torch.from_numpy(x).pin_memory()
    dst = torch.zeros((N, T), dtype=torch.complex64, device="cuda")
    cols = sharding.stage_cols(N, n_stages=4, min_width=512)
    side = torch.cuda.Stream()
    events = []
    with torch.cuda.stream(side):
        for c0, c1 in zip(cols[:-1], cols[1:]):
            dst[c0:c1].copy_(src[c0:c1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
            events.append(ev)
    got = C.plv_family(dst, input_kind="analytic", stages=(cols, events), timing=True)
    assert got["plv"].meta["ms_gram"] > 0.0  # bench.py's roofline reads it on the N > 1 path
    for m in METRICS:
        assert torch.equal(got[m].values, ref[m].values), m
    # sharded + staged: the union of two shards equals the full result
    parts = [C.plv_family(dst, input_kind="analytic", stages=(cols, [None] * (len(cols) - 1)), shard=(r, 2))
             for r in range(2)]
    for m in METRICS:
        assert torch.equal(parts[0][m].values + parts[1][m].values, ref[m].values), m


@pytest.mark.parametrize("prec", ["split", "fp64"])
def test_over_trials_time_resolved(prec):
    # Eq 8 / SPEC.md:153-157: one N x N matrix per sample, Gram over trials
    rng = np.random.default_rng(21)
    N, T, R = 150, 40, 37
    a = rng.standard_normal((N, T, R)) + 1j * rng.standard_normal((N, T, R))
    a[::9] *= np.exp(1j * rng.uniform(0, np.pi, (1, T, 1)))  # sample-dependent structure
    a[4, 3, :5] = 0            # masked trials at one sample
    z, mask = O.normalize_phasors(a)
    ref = O.plv_family_over_trials(z, mask)
    res = C.plv_family(a, input_kind="analytic", precision=prec, mode="over_trials")
    assert res["plv"].values.shape == (N, N, T) and res["plv"].n_observations == R
    check(res, ref, prec, "over_trials")
    v = C.plv_matrix(z, mode="over_trials", precision=prec).values
    assert maxerr(v, ref["plv"]) <= TOL[prec]


def test_deterministic_repeat():
    d = golden("c2_small")
    a = C.plv_family(d["x"], precision="split")
    b = C.plv_family(d["x"], precision="split")
    for m in METRICS:
        assert np.array_equal(a[m].values, b[m].values)


@pytest.mark.parametrize("reduce_", ["none", "pool", "mean"])
@pytest.mark.parametrize("prec", ["split", "fp64"])
def test_trial_reduce_modes(reduce_, prec):
    z = O.make_surrogate(70, 300, 5, seed=31)
    z[::7] *= np.exp(1j * 0.4)  # some structure
    ref = O.plv_family(z, input_kind="phasor", trial_reduce=reduce_)
    res = C.plv_family(z, input_kind="phasor", precision=prec, trial_reduce=reduce_)
    check(res, ref, prec, f"reduce={reduce_}")


@pytest.mark.parametrize("N,T,R", [(1, 16, 1), (2, 2, 1), (3, 7, 2), (129, 1001, 1), (257, 2001, 3),
                                   (300, 64, 1), (130, 8, 1)])
@pytest.mark.parametrize("prec", ["split", "fp64"])
def test_edge_shapes_real(N, T, R, prec):
    rng = np.random.default_rng(N * 1000 + T)
    x = rng.standard_normal((N, T, R))
    ref = O.plv_family(x, input_kind="real")
    res = C.plv_family(x, input_kind="real", precision=prec)
    check(res, ref, prec, f"real N={N} T={T} R={R}")


# ------------------------------------ band-pass front end
def _fir(order=300, lo=0.1, hi=0.2):
    return signalprep.design_bandpass_fir((lo * np.pi, hi * np.pi), order)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_filter_two_pass_matches_oracle(dt):
    rng = np.random.default_rng(31)
    x = rng.standard_normal((5, 1500, 2)).astype(dt)
    f = _fir()
    y = signalprep.filter_two_pass(x, f, 400)
    ref = O.filter_two_pass(x.astype(np.float64), f.taps, 400)
    assert y.dtype == dt and y.shape == x.shape
    e = maxerr(y, ref) / np.max(np.abs(ref))
    print(f"[parity] filter_two_pass {np.dtype(dt).name} rel={e:.3e}")
    assert e <= (1e-12 if dt is np.float64 else 2e-6)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_bandpass_analytic_matches_oracle(dt):
    rng = np.random.default_rng(32)
    x = rng.standard_normal((4, 2001, 3)).astype(dt)
    f = _fir(order=200)
    a = signalprep.analytic_signal(x, fir=f, pad_samples=333).data
    ref = O.bandpass_analytic(x.astype(np.float64), f.taps, 333)
    e = float(np.max(np.abs(a.astype(np.complex128) - ref)) / np.max(np.abs(ref)))
    print(f"[parity] bandpass analytic {np.dtype(dt).name} rel={e:.3e}")
    assert e <= (1e-12 if dt is np.float64 else 2e-6)
    # Re(a) is the filtered record
    assert maxerr(a.real, O.filter_two_pass(x.astype(np.float64), f.taps, 333)) <= (
        1e-12 if dt is np.float64 else 2e-6) * np.max(np.abs(ref))


@pytest.mark.parametrize("prec", ["split", "fp64"])
def test_plv_family_with_bandpass_front_end(prec):
    import torch

    x = W.c4(n_signals=24, n_samples=3000, n_trials=3, n_latent=3, bands=((8.0, 12.0),))[0]
    x = x.astype(np.float64) if prec == "fp64" else x
    f = _fir(order=400, lo=0.014, hi=0.026)  # ~7-13 Hz at 1 kHz
    ref = O.plv_family(x.astype(np.float64), input_kind="real", fir=(f.taps, 500))
    res = C.plv_family(x, input_kind="real", precision=prec, fir=f, pad_samples=500)
    check(res, ref, prec, "bandpass host")
    dev = C.plv_family(torch.from_numpy(np.ascontiguousarray(x)).cuda(), input_kind="real", precision=prec,
                       fir=f, pad_samples=500)
    for m in METRICS:
        assert maxerr(dev[m].values.cpu().numpy(), ref[m]) <= TOL[prec], m


def test_bandpass_pipelined_host_path_and_errors():
    import torch

    rng = np.random.default_rng(33)
    N, T = 2600, 600
    x = rng.standard_normal((N, T)).astype(np.float32)
    f = _fir(order=100, lo=0.2, hi=0.3)
    h = C.plv_family(x, input_kind="real", fir=f, pad_samples=150)
    d = C.plv_family(torch.from_numpy(x).cuda(), input_kind="real", fir=f, pad_samples=150)
    for m in METRICS:
        assert np.array_equal(h[m].values, d[m].values.cpu().numpy()), m
    idx = np.sort(rng.choice(N, size=64, replace=False))
    ref = O.plv_family(x[idx][:, :, None], input_kind="real", fir=(f.taps, 150))
    for m in METRICS:
        assert maxerr(h[m].values[np.ix_(idx, idx)], ref[m]) <= TOL["split"], m
    with pytest.raises(errors.SignalTooShortError):
        C.plv_family(x[:4, :101], input_kind="real", fir=f, pad_samples=10)
    with pytest.raises(errors.SignalTooShortError):
        signalprep.filter_two_pass(x[:4], f, 600)


# ---------------------------------- Welch coherence family
COH_METRICS = ("coh", "icoh", "cre", "cim")


@pytest.mark.parametrize("mode", ["max", "mean", "none"])
@pytest.mark.parametrize("prec", ["split", "fp64"])
def test_coherence_matrix_matches_oracle(mode, prec):
    rng = np.random.default_rng(51)
    x = rng.standard_normal((37, 3000, 2))
    x[5] = 0.7 * x[2] + 0.3 * np.roll(x[5], 3, axis=1)  # coupled pair
    x[9] = x[8]                                          # identical pair
    x = x.astype(np.float32) if prec == "split" else x
    cfg = C.WelchConfig(200, 100)
    ref = O.coherence_matrix(x.astype(np.float64), 200, 100, 0.2, 0.9, mode)
    res = C.coherence_matrix(x, cfg, (0.2, 0.9), mode=mode, metrics=COH_METRICS, precision=prec)
    errs = {m: maxerr(res[m].values, ref[m]) for m in COH_METRICS}
    print(f"[parity] coherence {mode} {prec} " + " ".join(f"{m}={e:.3e}" for m, e in errs.items()))
    for m, e in errs.items():
        assert e <= TOL[prec], (m, e)
    assert res["coh"].n_observations == 2 * 29


def test_coherence_matrix_bands_device_and_errors():
    import torch

    rng = np.random.default_rng(52)
    x = rng.standard_normal((2, 300, 1024, 3)).astype(np.float32)  # [B, N, T, R]
    cfg = C.WelchConfig(128, 64)
    res = C.coherence_matrix(torch.from_numpy(x).cuda(), cfg, (0.5, 1.5), mode="max", bands=True)
    got = res["coh"].values.cpu().numpy()
    for b in range(2):
        ref = O.coherence_matrix(x[b].astype(np.float64), 128, 64, 0.5, 1.5, "max")["coh"]
        assert maxerr(got[b], ref) <= TOL["split"]
    with pytest.raises(errors.WindowTooLongError):
        C.coherence_matrix(x[0], C.WelchConfig(2048, 0), (0.5, 1.5))
    with pytest.raises(errors.EmptyBandError):
        C.coherence_matrix(x[0], cfg, (0.001, 0.002))


def test_coherence_pair_spectra():
    rng = np.random.default_rng(53)
    x = rng.standard_normal((2, 5000, 2))
    x[1] += 0.5 * np.roll(x[0], 2, axis=1)
    cfg = C.WelchConfig(400, 200)
    c = C.coherence_welch(x, cfg)
    assert c.n_segments == 2 * 24 and c.values.shape == (201,)
    assert maxerr(c.values, O.coherence_welch(x, 400, 200)) <= 1e-12
    assert maxerr(C.coherence_weighted_phasor(x, cfg).values, O.coherence_weighted_phasor(x, 400, 200)) <= 1e-10
    assert maxerr(C.imaginary_coherency(x, cfg).values, O.imaginary_coherency(x, 400, 200)) <= 1e-12
    lo, hi = 0.570 * np.pi, 0.600 * np.pi
    assert abs(C.band_coherence(c, (lo, hi), "max") - O.band_coherence(c.values, 400, lo, hi, "max")) == 0.0


# ---------------------------------------- fused Hilbert kernel (fp32, T = 4096)
def test_fused_hilbert_t4096_bands():
    # odd N * R: the last row of the chunk has no partner in its FFT pair
    x = W.c4(n_signals=37, n_samples=4096, n_trials=3, n_latent=4)
    assert x.dtype == np.float32 and x.strides[2] == 4
    per = [O.plv_family(x[b].astype(np.float64), input_kind="real") for b in range(x.shape[0])]
    ref = {m: np.stack([p[m] for p in per]) for m in METRICS}
    res = C.plv_family(x, input_kind="real", precision="split", bands=True)
    check(res, ref, "split", "fused hilbert c4-like")
    assert not res["plv"].meta["input_copied"]


@pytest.mark.parametrize("T", [16, 30, 250, 1000, 1024, 2000, 2048, 2250, 4095, 4096, 10000, 12000])
def test_real_input_lengths_unequal_scales(T):
    # fp32 real rows, samples contiguous, odd and even T (4096: the fused
    # radix-16 kernel; others: the cuFFT chain, odd T with per-row scaling),
    # neighbouring rows 1e5 apart in scale and a zero stretch
    rng = np.random.default_rng(T)
    R = 2
    x = np.ascontiguousarray(rng.standard_normal((R, 7, T)).astype(np.float32)).transpose(1, 2, 0)
    x[3] *= 1e5          # rows sharing one packed FFT at very different scales
    x[4, :T // 5] = 0.0  # a zero stretch (amplitude-floor fixup path)
    ref = O.plv_family(x.astype(np.float64), input_kind="real")
    res = C.plv_family(x, input_kind="real", precision="split")
    check(res, ref, "split", f"real T={T}")
    m = O.normalize_phasors(O.analytic_signal(x.astype(np.float64), axis=1))[1]
    assert res["plv"].meta["n_masked_samples"] == int(m.sum())


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("T", [4, 6, 16, 250, 1000, 4098, 10000, 16384])
def test_even_T_half_length_chain_matches_r2c_chain(T, dt, monkeypatch):
    # even T: the row re-read as T / 2 complex samples, C2C -> collapsed
    # multiplier (hilbert_halfspec_kernel) -> C2C, against the oracle and
    # against cuFFT's R2C -> K2 -> C2R chain (PS_HILBERT_CHAIN forces one);
    # rows of very different scale (the half-length transform never mixes rows),
    # row distance > T (direct, unpacked input) and an odd row distance (packed)
    import torch

    rng = np.random.default_rng(T + 5)
    for ld, c0 in ((T, 0), (T + 2, 0), (T + 3, 0), (T + 2, 1)):
        # (T + 2, 1): even row distance but a base one element off the complex alignment (packed)
        buf = rng.standard_normal((6, ld)).astype(dt)
        buf[1] *= 1e5
        buf[4] *= 1e-5
        x = buf[:, c0:c0 + T]
        xd = torch.from_numpy(buf).cuda()[:, c0:c0 + T]  # device view, row distance ld
        ar = O.analytic_signal(x.astype(np.float64), axis=1)
        out = {}
        for chain in ("half", "r2c"):
            monkeypatch.setenv("PS_HILBERT_CHAIN", chain)
            a = signalprep.analytic_signal(xd).data.cpu().numpy()
            assert np.array_equal(a.real, x)  # Re(a) == x bit-exactly
            rel = np.max(np.abs(a - ar), axis=1) / np.max(np.abs(ar), axis=1)
            assert np.all(rel <= (1e-13 if dt is np.float64 else 2e-6)), (chain, ld, rel)
            out[chain] = a
        rel = np.max(np.abs(out["half"] - out["r2c"]), axis=1) / np.max(np.abs(ar), axis=1)
        assert np.all(rel <= (1e-13 if dt is np.float64 else 2e-6)), (ld, rel)
    monkeypatch.setenv("PS_HILBERT_CHAIN", "half")
    xs = np.ascontiguousarray(rng.standard_normal((2, 7, T)).astype(dt)).transpose(1, 2, 0)
    ref = O.plv_family(xs.astype(np.float64), input_kind="real")
    prec = "split" if dt is np.float32 else "fp64"
    check(C.plv_family(xs, input_kind="real", precision=prec), ref, prec, f"half chain T={T}")


@pytest.mark.parametrize("kind,dt", [("real", np.float32), ("real", np.float64), ("analytic", np.complex64)])
@pytest.mark.parametrize("T", [999, 1000, 2048, 4096])
def test_views_starting_off_the_vector_alignment(T, kind, dt):
    # device views that start 1 or 3 elements into their buffer: rows are not
    # aligned for 16-byte loads, for cuFFT's R2C (complex-type alignment) or for
    # re-reading a row as complex pairs -- every stage has to fall back to a
    # packed copy or scalar loads (a direct cuFFT call on such rows fails with
    # CUFFT_INVALID_VALUE)
    import torch

    rng = np.random.default_rng(T)
    N = 9
    for c0 in (1, 3):
        buf = rng.standard_normal((N, T + 8))
        if kind == "analytic":
            buf = buf + 1j * rng.standard_normal((N, T + 8))
        buf = buf.astype(dt)
        x = buf[:, c0:c0 + T]
        xd = torch.from_numpy(buf).cuda()[:, c0:c0 + T]
        ref = O.plv_family(x[:, :, None].astype(np.complex128 if kind == "analytic" else np.float64), input_kind=kind)
        for prec in ("split", "fp64"):
            res = C.plv_family(xd[:, :, None], input_kind=kind, precision=prec)
            tol = 1e-12 if (prec == "fp64" and dt is np.float64) else 1e-5
            for m in ("plv", "iplv", "ciplv"):
                err = float(np.max(np.abs(res[m].values.double().cpu().numpy() - ref[m])))
                assert err <= tol, (T, kind, c0, prec, m, err)


@pytest.mark.parametrize("prec,dt", [("split", np.float32), ("fp64", np.float64), ("fp64", np.float32)])
@pytest.mark.parametrize("T", [1001, 2047])
def test_odd_T_cufft_rows_of_unequal_scale(T, prec, dt):
    # odd T: cuFFT's batched R2C pairs rows into one complex transform; rows
    # are packed with per-row power-of-two scales so a 1e6-times larger
    # neighbour does not leak its rounding error into a row
    rng = np.random.default_rng(T + 1)
    x = np.ascontiguousarray(rng.standard_normal((2, 9, T)).astype(dt)).transpose(1, 2, 0)
    x[1] *= 1e6
    x[4] *= 1e-6
    ref = O.plv_family(x.astype(np.float64), input_kind="real")
    res = C.plv_family(x, input_kind="real", precision=prec)
    check(res, ref, prec, f"odd T={T} {np.dtype(dt).name}")
    a = signalprep.analytic_signal(x).data
    ar = O.analytic_signal(x.astype(np.float64), axis=1)
    rel = np.max(np.abs(a - ar), axis=(1, 2)) / np.max(np.abs(ar), axis=(1, 2))
    assert np.all(rel <= (1e-13 if dt is np.float64 else 2e-6)), rel
    assert np.array_equal(a.real, x)  # Re(a) == x bit-exactly


def test_bandpass_odd_padded_length_unequal_scales():
    # L = T + 2 pad odd: the length-L Hilbert FFT of the filtered record uses
    # the same per-row scaling
    rng = np.random.default_rng(77)
    x = np.ascontiguousarray(rng.standard_normal((1, 6, 1201))).transpose(1, 2, 0)
    x[2] *= 1e6
    f = _fir(order=100, lo=0.2, hi=0.4)
    a = signalprep.analytic_signal(x, fir=f, pad_samples=300).data
    ar = O.bandpass_analytic(x, f.taps, 300)
    rel = np.max(np.abs(a - ar), axis=(1, 2)) / np.max(np.abs(ar), axis=(1, 2))
    assert np.all(rel <= 1e-13), rel
    res = C.plv_family(x, input_kind="real", precision="fp64", fir=f, pad_samples=300)
    check(res, O.plv_family(x, input_kind="real", fir=(f.taps, 300)), "fp64", "bandpass odd L")


@pytest.mark.parametrize("T", [4096, 2048, 1024])
def test_fused_hilbert_mixed_row_scales(T):
    # rows sharing one packed FFT differ by 1e10 in amplitude (T = 2048 / 1024:
    # 2 / 4 row pairs per CTA iteration, 9 rows leave a partial last group)
    rng = np.random.default_rng(41)
    x = rng.standard_normal((9, T, 1)).astype(np.float32)
    x = np.ascontiguousarray(x[:, :, 0])[:, :, None]
    x[0] *= 1e6
    x[1] *= 1e-4
    x[4] *= 3e-30
    ref = O.plv_family(x.astype(np.float64), input_kind="real")
    res = C.plv_family(x, input_kind="real", precision="split")
    check(res, ref, "split", "fused hilbert mixed scales")


@pytest.mark.parametrize("T", [4096, 2048, 1024])
def test_fused_hilbert_amplitude_floor_fixup(T):
    rng = np.random.default_rng(42)
    x = rng.standard_normal((7, T)).astype(np.float32)
    x[1, T // 4:T // 4 + T // 10] = 0.0
    x[4, 100:130] = 0.0
    x[6, T - 40:] = 0.0
    x = x[:, :, None]
    ref = O.plv_family(x.astype(np.float64), input_kind="real", amp_floor=0.05)
    res = C.plv_family(x, input_kind="real", precision="split", amp_floor=0.05)
    check(res, ref, "split", "fused hilbert floor")
    m = O.normalize_phasors(O.analytic_signal(x.astype(np.float64), axis=1), amp_floor=0.05)[1]
    assert res["plv"].meta["n_masked_samples"] == int(m.sum())


def test_hilbert_t65536_rows():
    # fp32 real rows of T = 65536 (C3's length, cuFFT chain): odd row count,
    # rows 1e6 apart in scale, an amplitude-floor fixup row.  (A zero stretch
    # of T/5 at this length leaves H in the fp32 FFT noise floor inside it:
    # 1.4e-5 PLV error through cuFFT, so the stretch here is shorter.)
    rng = np.random.default_rng(65536)
    T = 65536
    x = rng.standard_normal((9, T)).astype(np.float32)
    x[2] *= 1e6
    x[3] *= 1e-6
    x[5, 5000:9000] = 0.0
    x = x[:, :, None]
    for floor in (1e-6, 0.05):
        ref = O.plv_family(x.astype(np.float64), input_kind="real", amp_floor=floor)
        res = C.plv_family(x, input_kind="real", precision="split", amp_floor=floor)
        check(res, ref, "split", f"four-step floor={floor}")
        m = O.normalize_phasors(O.analytic_signal(x.astype(np.float64), axis=1), amp_floor=floor)[1]
        assert res["plv"].meta["n_masked_samples"] == int(m.sum())


def test_float32_trial_fastest_layout_copies():
    # reference layout [N, T, R] row-major: samples are strided -> packing copy
    rng = np.random.default_rng(5)
    x = rng.standard_normal((90, 1500, 3)).astype(np.float32)
    ref = O.plv_family(x, input_kind="real")
    res = C.plv_family(x, precision="split")
    check(res, ref, "split", "f32 [N,T,R] contiguous")
    assert res["plv"].meta["input_copied"]


def test_combinations_bands_with_bandpass_over_trials_and_pipelined_bandpass():
    import torch

    rng = np.random.default_rng(62)
    f = _fir(order=60, lo=0.2, hi=0.5)
    # band-pass front end with a band axis (device and host paths)
    x = rng.standard_normal((2, 40, 700, 3)).astype(np.float32)        # [B, N, T, R]
    res = C.plv_family(x, input_kind="real", bands=True, fir=f, pad_samples=80)
    for b in range(2):
        ref = O.plv_family(x[b].astype(np.float64), input_kind="real", fir=(f.taps, 80))
        for m in METRICS:
            assert maxerr(res[m].values[b], ref[m]) <= TOL["split"], (b, m)
    # time-resolved mode with a band axis
    z = np.exp(1j * rng.uniform(0, 6.3, (2, 30, 20, 9)))                # [B, N, T, R]
    tr = C.plv_family(z, input_kind="phasor", bands=True, mode="over_trials", precision="fp64")
    assert tr["plv"].values.shape == (2, 30, 30, 20)
    for b in range(2):
        zz, mk = O.phasors_from_unit(z[b])
        ref = O.plv_family_over_trials(zz, mk)
        for m in METRICS:
            assert maxerr(tr[m].values[b], ref[m]) <= TOL["fp64"], (b, m)
    # band-pass on the pipelined host path (N >= 2048 and >= 148 tiles)
    N = 3072
    xp = rng.standard_normal((N, 400)).astype(np.float32)
    h = C.plv_family(xp, input_kind="real", fir=f, pad_samples=100)
    d = C.plv_family(torch.from_numpy(xp).cuda(), input_kind="real", fir=f, pad_samples=100)
    for m in METRICS:
        assert np.array_equal(h[m].values, d[m].values.cpu().numpy()), m
    idx = np.sort(rng.choice(N, size=40, replace=False))
    ref = O.plv_family(xp[idx][:, :, None], input_kind="real", fir=(f.taps, 100))
    for m in METRICS:
        assert maxerr(h[m].values[np.ix_(idx, idx)], ref[m]) <= TOL["split"], m


@pytest.mark.parametrize("reduce_", ["mean", "none"])
def test_heavy_zero_lag_leakage_split_accuracy(reduce_):
    # clusters of signals sharing one source at zero lag (|Re| -> 1 for every
    # within-cluster pair): tens of thousands of ill-conditioned ciPLV pairs,
    # all refined in FP64 on the device; split results within 1e-5
    rng = np.random.default_rng(61)
    N, T, R, K = 512, 2048, 2, 32
    src = rng.standard_normal((N // K, T, R)) + 1j * rng.standard_normal((N // K, T, R))
    a = src[np.arange(N) // K] + 0.05 * (rng.standard_normal((N, T, R)) + 1j * rng.standard_normal((N, T, R)))
    a = a.astype(np.complex64)
    ref = O.plv_family(a, input_kind="analytic", trial_reduce=reduce_)
    res = C.plv_family(a, input_kind="analytic", precision="split", trial_reduce=reduce_)
    check(res, ref, "split", f"leakage {reduce_}")
    assert res["plv"].meta["n_refined_pairs"] > 10000
    # accurate after refinement: none may be reported indeterminate
    assert res["plv"].meta["n_indeterminate_ciplv"] == 0


def test_signed_coherency_outputs():
    z = O.make_surrogate(40, 500, 1, seed=8)
    raw = O.plv_family(z, input_kind="phasor", raw=True)["cgram"][:, :, 0]
    res = C.plv_family(z, input_kind="phasor", precision="fp64", metrics=("cre", "cim"))
    re = raw.real.copy()
    im = raw.imag.copy()
    np.fill_diagonal(re, 1.0)
    np.fill_diagonal(im, 0.0)
    assert maxerr(res["cre"].values, re) < 1e-12
    assert maxerr(res["cim"].values, im) < 1e-12


# ------------------------------------------------------------ masks / errors
@pytest.mark.parametrize("prec", ["split", "fp64"])
def test_masked_samples_effective_T(prec):
    rng = np.random.default_rng(3)
    a = (rng.standard_normal((20, 400, 2)) + 1j * rng.standard_normal((20, 400, 2)))
    a[2, 10:50, 0] = 0
    a[5, 30:90, 0] = 0
    a[5, :5, 1] = 1e-9  # below 1e-6 x median amplitude -> masked
    ref = O.plv_family(a, input_kind="analytic")
    res = C.plv_family(a, input_kind="analytic", precision=prec)
    check(res, ref, prec, "masked")
    assert res["plv"].meta["n_masked_samples"] == 40 + 60 + 5


def test_all_masked_raises():
    a = np.ones((4, 64, 1), np.complex128)
    a[2] = 0
    with pytest.raises(errors.AllSamplesMaskedError):
        C.plv_family(a, input_kind="analytic")


def test_empty_effective_window_raises():
    z = O.make_surrogate(3, 8, 1, seed=5)
    z[0, :4, 0] = 0
    z[1, 4:, 0] = 0
    with pytest.raises(errors.EmptyEffectiveWindowError):
        C.plv_family(z, input_kind="phasor")


def test_shape_error():
    with pytest.raises(errors.ShapeError):
        C.plv_family(np.zeros((4,)))
    with pytest.raises(errors.ShapeError):
        C.plv_family(np.zeros((4, 1, 1)))


# ------------------------------------------------------------ signalprep
@pytest.mark.parametrize("T", [2000, 2001, 4096])
def test_analytic_signal_matches_oracle(T):
    rng = np.random.default_rng(T)
    x = rng.standard_normal((7, T, 2))
    a = signalprep.analytic_signal(x).data
    ref = O.analytic_signal(x)
    assert np.array_equal(a.real, x)
    assert np.max(np.abs(a.imag - ref.imag)) < 1e-12 * np.sqrt(T) * 10
    x32 = x.astype(np.float32)
    a32 = signalprep.analytic_signal(x32).data
    assert a32.dtype == np.complex64 and np.array_equal(a32.real, x32)
    assert np.max(np.abs(a32.imag - ref.imag)) < 1e-4


def test_normalize_phasors_matches_oracle():
    rng = np.random.default_rng(4)
    a = rng.standard_normal((9, 300, 2)) + 1j * rng.standard_normal((9, 300, 2))
    a[1, 4, 0] = 0
    a[3, 7, 1] = 1e-12
    p = signalprep.normalize_phasors(a)
    z, m = O.normalize_phasors(a)
    assert np.array_equal(np.asarray(p.mask), m)
    assert np.max(np.abs(p.data - z)) < 1e-15


# ------------------------------------------------------------ full-size configs
def subset_check(x, res, idx, input_kind, prec, label, trial_reduce="mean"):
    xs = x[idx]
    ref = O.plv_family(xs, input_kind=input_kind, trial_reduce=trial_reduce)
    sub = {m: np.asarray(res[m].values[np.ix_(idx, idx)], dtype=np.float64) for m in METRICS}
    errs = {m: maxerr(sub[m], ref[m]) for m in METRICS}
    print(f"[parity] {label} {prec} subset={len(idx)} " + " ".join(f"{m}={e:.3e}" for m, e in errs.items()))
    return errs


def props(res, N):
    p = res["plv"].values
    for m in METRICS:
        v = res[m].values
        assert float(v.max()) <= 1.0 + 1e-9 and float(v.min()) >= 0.0
        # symmetric (each pair written once with its mirror)
        k = np.random.default_rng(0).integers(0, N, size=(2000, 2))
        vv = np.asarray(v)
        assert np.array_equal(vv[k[:, 0], k[:, 1]], vv[k[:, 1], k[:, 0]])
    dg = np.asarray(p)[np.arange(N), np.arange(N)]
    assert np.all(dg == 1.0)


# full-size configs: tests/test_gpu_scale_parity.py (structured row subsets, both precisions)


# ------------------------------------------------------------ CLI (acceptance #9)
def test_cli_matches_library_bit_exactly(tmp_path):
    from paper_1710_08037_b200 import bindings, cli

    rng = np.random.default_rng(20)
    x = rng.standard_normal((20, 700, 2))
    x[7] = x[3]  # duplicated channel: PLV 1, ciPLV 0
    cli.write_bundle(tmp_path / "in", x, axes=["signal", "sample", "trial"])
    for metric in ("plv", "iplv", "ciplv"):
        out = tmp_path / metric
        assert cli.entrypoint(["connectivity", str(tmp_path / "in"), "--metric", metric, "-o", str(out)]) == 0
        got, hdr = cli.read_bundle(out)
        lib = bindings.py_plv(x) if metric == "plv" else (
            bindings.py_iplv(x) if metric == "iplv" else bindings.py_ciplv(x))
        assert np.array_equal(got, np.asarray(lib, dtype=np.float64)), metric
        assert (out.with_suffix(".csv")).exists() and (out.with_suffix(".manifest.json")).exists()
        if metric == "plv":
            assert abs(got[3, 7] - 1.0) < 1e-5
        if metric == "ciplv":
            assert got[3, 7] == 0.0


def test_cli_band_pass_matches_library(tmp_path):
    # cmd_connectivity with --band runs the band-pass front end
    from paper_1710_08037_b200 import cli

    rng = np.random.default_rng(22)
    x = rng.standard_normal((10, 900, 2))
    cli.write_bundle(tmp_path / "in", x, axes=["signal", "sample", "trial"])
    out = tmp_path / "bp"
    argv = ["connectivity", str(tmp_path / "in"), "--metric", "plv", "--band", "0.3", "0.5", "--order", "200",
            "--pad", "300", "-o", str(out)]
    assert cli.entrypoint(argv) == 0
    got, _ = cli.read_bundle(out)
    f = signalprep.design_bandpass_fir((0.3, 0.5), 200)
    lib = C.plv_family(x, input_kind="real", metrics=("plv",), fir=f, pad_samples=300)["plv"].values
    assert np.array_equal(got, np.asarray(lib, dtype=np.float64))
    ref = O.plv_family(x, input_kind="real", fir=(f.taps, 300))["plv"]
    assert maxerr(got, ref) <= TOL["split"]


@pytest.mark.parametrize("metric", ["coh_max", "coh_mean"])
def test_cli_coherence_matches_oracle(tmp_path, metric):
    from paper_1710_08037_b200 import cli

    rng = np.random.default_rng(23)
    x = rng.standard_normal((12, 2000, 2))
    x[4] = x[1]  # duplicated channel: coherence 1
    cli.write_bundle(tmp_path / "in", x, axes=["signal", "sample", "trial"])
    out = tmp_path / metric
    argv = ["connectivity", str(tmp_path / "in"), "--metric", metric, "--band", "0.3", "0.8", "--window", "200",
            "--overlap", "100", "--precision", "fp64", "-o", str(out)]
    assert cli.entrypoint(argv) == 0
    got, hdr = cli.read_bundle(out)
    ref = O.coherence_matrix(x, 200, 100, 0.3, 0.8, metric.split("_")[1])["coh"]
    assert maxerr(got, ref) <= TOL["fp64"]
    assert abs(got[1, 4] - 1.0) < 1e-12 and hdr["meta"]["metric"] == metric.upper()
