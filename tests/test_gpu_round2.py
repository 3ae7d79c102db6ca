"""GPU tests of the round-2 pieces on one B200:
  * (band, trial) unit sharding: two unit shards' trial SUMS combined by
    ps_reduce_partials (fixed order) equal the unsharded trial mean within
    float order; ps_reduce_partials equals a left-to-right fp64 sum;
  * the all-gather of owned tiles: ps_shard_pack / ps_shard_unpack move the
    tiles of shard s exactly (both layouts, antisymmetric cim);
  * a sharded host-output call in the 'full' layout must
    not leak another shard's values through the reused staging buffer;
  * a ~1e-4 rad constant offset (|Re| rounds to 1 in fp32)
    gives ciPLV ~ 1 or an explicit CiplvIndeterminateWarning;
  * the py_coherence binding equals `phasesync connectivity --metric coh_max`
    bit-exactly (acceptance #9 analogue);
  * concurrent host-output calls on one context.
"""
import ctypes
import threading
import warnings

import numpy as np
import pytest

from oracle import plv_oracle as O
from paper_1710_08037_b200 import _native, errors, sharding
from paper_1710_08037_b200 import connectivity as C

pytestmark = pytest.mark.gpu
METRICS = ("plv", "iplv", "ciplv")


def _reduce(parts, n_parts, stride, n, divisor, out):
    sharding._native_reduce(parts, n_parts, stride, n, divisor, out)


@pytest.mark.parametrize("prec", ["split", "fp64"])
def test_unit_shards_sum_then_reduce_equals_mean(prec):
    import torch

    B, N, T, R = 2, 300, 900, 5
    rng = np.random.default_rng(90)
    x = rng.standard_normal((B, R, N, T)).astype(np.float32)           # [B, R, N, T] memory
    xd = torch.from_numpy(x).cuda()
    full = C.plv_family(xd.permute(0, 2, 3, 1), input_kind="real", precision=prec, bands=True)
    world = 3
    parts = []
    for r in range(world):
        frags = [(b, xd[b, t0:t1].permute(1, 2, 0)) for b, t0, t1 in sharding.unit_ranges(B, R, world, r)]
        p, _ = sharding.unit_partial_sums(frags, B, N, input_kind="real", precision=prec)
        parts.append(p)
    for m in METRICS:
        stacked = torch.stack([p[m] for p in parts]).contiguous()     # [P, B, N, N] as after the all-to-all
        out = torch.empty_like(stacked[0])
        n = stacked[0].numel()
        _reduce(stacked.reshape(-1), world, n, n, float(R), out.reshape(-1))
        want = full[m].values
        err = (out - want).abs().max().item()
        assert err <= (2e-6 if prec == "split" else 1e-14), (m, err)
        # fixed order: left-to-right in fp64 of the same partials, then / R
        ref = stacked[0].double()
        for s in range(1, world):
            ref = ref + stacked[s].double()
        if prec == "fp64":
            assert torch.equal(out, ref / torch.full_like(ref, float(R))), m
        else:
            lr = stacked[0].clone()
            for s in range(1, world):
                lr = lr + stacked[s]
            assert torch.equal(out, lr / torch.full_like(lr, float(R))), m  # (torch scalar division is a reciprocal multiply)


def test_reduce_partials_unaligned_and_errors():
    import torch

    lib = _native.lib()
    ctx = _native.context(0)
    for n, stride in ((1001, 1003), (4096, 4096)):
        parts = torch.randn(3 * stride, dtype=torch.float32, device="cuda")
        out = torch.empty(n, dtype=torch.float32, device="cuda")
        _native.check(lib.ps_reduce_partials(ctx.handle, parts.data_ptr(), 3, stride, n, 7.0, 0, out.data_ptr(),
                                             None))
        torch.cuda.synchronize()
        s3 = parts[:n] + parts[stride:stride + n] + parts[2 * stride:2 * stride + n]
        want = s3 / torch.full_like(s3, 7.0)
        assert torch.equal(out, want)
    with pytest.raises(ValueError):
        _native.check(lib.ps_reduce_partials(ctx.handle, parts.data_ptr(), 3, 10, 20, 1.0, 0, out.data_ptr(), None))


@pytest.mark.parametrize("prec,layout", [("split", "full"), ("split", "upper"), ("fp64", "full")])
def test_shard_pack_unpack_reassembles(prec, layout):
    import torch

    N, P = 700, 3
    z = O.make_surrogate(N, 400, 1, seed=91)
    x = torch.from_numpy(z).cuda()
    ms = ("plv", "cim")
    full = C.plv_family(x, input_kind="phasor", precision=prec, metrics=ms, layout=layout)
    shards = [C.plv_family(x, input_kind="phasor", precision=prec, metrics=ms, layout=layout, shard=(r, P))
              for r in range(P)]
    lib = _native.lib()
    ctx = _native.context(0)
    for m in ms:
        dst = shards[0][m].values.clone()
        for s in range(1, P):
            n, bm, bn = _native.shard_tiles(N, prec, P, s)
            packed = torch.zeros(n * bm * bn, dtype=dst.dtype, device="cuda")
            _native.check(lib.ps_shard_pack(ctx.handle, N, _native.PRECISIONS[prec], P, s,
                                            shards[s][m].values.data_ptr(), packed.data_ptr(), None))
            mirror = 0 if layout == "upper" else (-1 if m == "cim" else 1)
            _native.check(lib.ps_shard_unpack(ctx.handle, N, _native.PRECISIONS[prec], P, s, packed.data_ptr(),
                                              dst.data_ptr(), mirror, None))
        torch.cuda.synchronize()
        assert torch.equal(dst, full[m].values), (m, (dst - full[m].values).abs().max().item())


@pytest.mark.parametrize("prec", ["split", "fp64"])
def test_sharded_host_call_full_layout_no_stale_entries(prec):
    # numpy input, shard=(r, 2), layout 'full', one context reused
    z = O.make_surrogate(500, 600, 1, seed=92)
    ref = C.plv_family(z, input_kind="phasor", precision=prec)
    got = [C.plv_family(z, input_kind="phasor", precision=prec, shard=(r, 2)) for r in (0, 1)]
    own = sharding.owner_matrix(500, prec, 2)
    for m in METRICS:
        s = got[0][m].values + got[1][m].values
        assert np.array_equal(s, ref[m].values), m
        assert not np.any(got[1][m].values[own != 1]), m  # other shard's entries are 0, not shard 0's values


def test_small_offset_ciplv_is_one_or_flagged():
    # constant offset 1e-4 rad -> true ciPLV = 1 (|Re| = cos 1e-4
    # rounds to 1 in fp32); split must return ~1 or warn
    T = 4000
    rng = np.random.default_rng(93)
    ph = np.cumsum(rng.normal(0, 0.3, size=T))
    z = np.zeros((3, T, 1), dtype=np.complex128)
    z[0, :, 0] = np.exp(1j * ph)
    z[1, :, 0] = np.exp(1j * (ph + 1e-4))
    z[2, :, 0] = np.exp(1j * rng.uniform(0, 2 * np.pi, T))
    ref = O.plv_family(z, input_kind="phasor")
    assert abs(ref["ciplv"][0, 1] - 1.0) < 1e-6
    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always")
        res = C.plv_family(z, input_kind="phasor", precision="split")
    v = float(res["ciplv"].values[0, 1])
    flagged = any(issubclass(w.category, errors.CiplvIndeterminateWarning) for w in rec)
    assert abs(v - 1.0) <= 1e-5 or (flagged and res["plv"].meta["n_indeterminate_ciplv"] >= 1), (v, flagged)
    # FP64: 1 - Re^2 = 1e-8 amplifies fp64 rounding (~1e-15 in Re) by ~1e8 in
    # ciPLV -- the oracle and the DMMA path agree to that conditioning limit,
    # and the value stays inside the SPEC.md:150 bound
    f64 = C.plv_family(z, input_kind="phasor", precision="fp64")
    v64 = float(f64["ciplv"].values[0, 1])
    assert abs(v64 - ref["ciplv"][0, 1]) <= 1e-6 and v64 <= 1.0
    # duplicated channel (exactly singular): 0 without a warning
    zd = z.copy()
    zd[1] = zd[0]
    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always")
        rd = C.plv_family(zd, input_kind="phasor", precision="split")
    assert float(rd["ciplv"].values[0, 1]) == 0.0
    assert not any(issubclass(w.category, errors.CiplvIndeterminateWarning) for w in rec)


def test_py_coherence_equals_cli_bit_exactly(tmp_path):
    from paper_1710_08037_b200 import bindings, cli

    rng = np.random.default_rng(94)
    x = rng.standard_normal((14, 3000, 2))
    x[5] = x[2]
    cli.write_bundle(tmp_path / "in", x, axes=["signal", "sample", "trial"])
    for metric, mode in (("coh_max", "max"), ("coh_mean", "mean")):
        out = tmp_path / metric
        argv = ["connectivity", str(tmp_path / "in"), "--metric", metric, "--band", "0.2", "0.7", "--window", "256",
                "--overlap", "128", "-o", str(out)]
        assert cli.entrypoint(argv) == 0
        got, _ = cli.read_bundle(out)
        lib = bindings.py_coherence(x, {"window_len": 256, "overlap": 128, "band": (0.2, 0.7), "mode": mode})
        assert np.array_equal(got, np.asarray(lib, dtype=np.float64)), metric
        assert abs(lib[2, 5] - 1.0) < 1e-5
    spec = bindings.py_coherence(x[:2], {"window_len": 256, "overlap": 128, "precision": "fp64"})
    ref = O.coherence_welch(x[:2], 256, 128)
    assert spec.shape == (2, 2, 129) and np.max(np.abs(spec[0, 1] - ref)) <= 1e-12


def test_concurrent_host_calls_one_context():
    # two threads, one context (ctypes releases the GIL)
    import torch

    zs = [O.make_surrogate(400, 500, 1, seed=s) for s in (95, 96)]
    refs = [C.plv_family(z, input_kind="phasor")["plv"].values for z in zs]
    ctx = _native.context(0)
    errs = []

    def run(k):
        try:
            for _ in range(5):
                z = zs[k]
                a = _native.PlvArgs()
                a.input = z.ctypes.data
                a.dtype = _native.DTYPES["c128"]
                a.input_kind = _native.INPUT_KINDS["phasor"]
                a.n_bands, a.n_signals, a.n_samples, a.n_trials = 1, 400, 500, 1
                a.stride_band, a.stride_signal, a.stride_sample, a.stride_trial = 400 * 500, 500, 1, 1
                a.amp_floor = 1e-6
                a.metrics = 1
                a.precision = 0
                a.shard_count = 1
                out = np.zeros((400, 400), dtype=np.float32)
                a.out_plv = out.ctypes.data
                res = _native.PlvResult()
                _native.check(_native.lib().ps_plv_family_host(ctx.handle, ctypes.byref(a), ctypes.byref(res)))
                if not np.array_equal(out, refs[k]):
                    errs.append(k)
        except Exception as exc:  # pragma: no cover
            errs.append(repr(exc))

    th = [threading.Thread(target=run, args=(k,)) for k in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not errs, errs


@pytest.mark.parametrize("R,groups", [(41, None), (41, "1"), (47, "47")])
def test_trial_mean_diagonal_exact_and_symmetric(R, groups, monkeypatch):
    """Trial means over R trials where R * fl(1/R) != 1 in fp32: the self-pair
    PLV stays exactly 1 and iPLV / ciPLV exactly 0, both
    triangles are bit-identical mirrors, and the values match the oracle --
    through the trial-group partial sums (upper-triangle slots + tiled
    reduce) and through the single-group path (mean at the last round)."""
    import subprocess
    import sys

    if groups is not None:
        # PS_GROUPS is read once per process: run the check in a child
        code = f"""
import sys; sys.path.insert(0, {repr(str(__import__('pathlib').Path(__file__).resolve().parents[1]))})
import numpy as np, torch
from oracle import plv_oracle as O
from paper_1710_08037_b200 import connectivity as C
z = O.make_surrogate(320, 64, {R}, seed=91)
r = C.plv_family(torch.from_numpy(z).cuda(), input_kind="phasor")
ref = O.plv_family(z, input_kind="phasor")
for m in ("plv", "iplv", "ciplv"):
    v = r[m].values[0].cpu().numpy() if r[m].values.dim() == 3 else r[m].values.cpu().numpy()
    d = np.diag(v)
    assert np.all(d == (1.0 if m == "plv" else 0.0)), (m, d[d != (1.0 if m == "plv" else 0.0)][:4])
    assert np.array_equal(v, v.T), m
    assert np.max(np.abs(v - ref[m])) <= 1e-5, m
print("ok")
"""
        env = dict(__import__("os").environ, PS_GROUPS=groups)
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
        return
    import torch

    z = O.make_surrogate(320, 64, R, seed=91)
    r = C.plv_family(torch.from_numpy(z).cuda(), input_kind="phasor")
    ref = O.plv_family(z, input_kind="phasor")
    for m in METRICS:
        v = r[m].values.cpu().numpy()
        v = v[0] if v.ndim == 3 else v
        want = 1.0 if m == "plv" else 0.0
        assert np.all(np.diag(v) == want), m
        assert np.array_equal(v, v.T), m
        assert np.max(np.abs(v - ref[m])) <= 1e-5, m


@pytest.mark.parametrize("N", [256, 260, 1032])
def test_diagonal_blocks_fast_path_matches_general(N):
    """Diagonal warp blocks take the predicated interior loops; the general
    per-pair path (PS_DEBUG_EPI=2048 in a child process) must give the same
    bits, per trial and for trial means, both layouts."""
    import os
    import subprocess
    import sys

    code = f"""
import sys; sys.path.insert(0, {repr(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))})
import numpy as np, torch
from oracle import plv_oracle as O
from paper_1710_08037_b200 import connectivity as C
z = torch.from_numpy(O.make_surrogate({N}, 96, 3, seed=92)).cuda()
out = []
for red in ("none", "mean"):
    for layout in ("full", "upper"):
        r = C.plv_family(z, input_kind="phasor", trial_reduce=red, layout=layout,
                         metrics=("plv", "iplv", "ciplv", "cre", "cim"))
        out += [r[m].values.cpu().numpy() for m in ("plv", "iplv", "ciplv", "cre", "cim")]
np.save(sys.argv[1], np.concatenate([o.reshape(-1) for o in out]))
"""
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        res = []
        for flag in ("0", "2048"):
            path = os.path.join(td, f"o{flag}.npy")
            env = dict(os.environ, PS_DEBUG_EPI=flag)
            out = subprocess.run([sys.executable, "-c", code, path], env=env, capture_output=True, text=True,
                                 timeout=600)
            assert out.returncode == 0, out.stderr[-2000:]
            res.append(np.load(path))
        assert np.array_equal(res[0], res[1])
