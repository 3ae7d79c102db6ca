"""GPU: PS_LAYOUT_UPPER (BASELINE configs[4]: "the upper triangle for each
metric") against PS_LAYOUT_FULL on the same inputs.

The upper entries (i <= j) must be bit-identical to the full layout's (the
same tiles, epilogue, trial-group reduction and FP64 refinement produce them;
only the mirror writes and their transfer are skipped), and the strictly lower
triangle must be left as allocated (zero here) -- on the device path, the host
non-pipelined path, the host pipelined path, the trial-group reduction, the
refine queue, time-resolved mode and Welch coherence.
"""
import numpy as np
import pytest

from oracle import plv_oracle as O
from paper_1710_08037_b200 import connectivity as C

pytestmark = pytest.mark.gpu

ALL = ("plv", "iplv", "ciplv", "cre", "cim")


def _np(v):
    return v.cpu().numpy() if hasattr(v, "cpu") else np.asarray(v)


def _same_upper(full, upper, label):
    """full / upper: arrays [..., N, N] or TimeResolved / per-trial [N, N, K]."""
    f, u = _np(full), _np(upper)
    assert f.shape == u.shape, label
    if f.shape[-1] != f.shape[-2]:  # [..., N, N, K] (per trial / sample / bin) -> [K, ..., N, N]
        f, u = np.moveaxis(f, -1, 0), np.moveaxis(u, -1, 0)
    N = f.shape[-1]
    iu = np.triu_indices(N)
    il = np.tril_indices(N, -1)
    fu, uu = f[..., iu[0], iu[1]], u[..., iu[0], iu[1]]
    assert np.array_equal(fu, uu), (label, float(np.max(np.abs(fu - uu))))
    assert not np.any(u[..., il[0], il[1]]), (label, "lower triangle written")


def _both(x, label, **kw):
    full = C.plv_family(x, layout="full", **kw)
    upper = C.plv_family(x, layout="upper", **kw)
    assert upper[next(iter(upper))].meta["layout"] == "upper"
    for m in full:
        _same_upper(full[m].values, upper[m].values, f"{label}:{m}")
    return full, upper


@pytest.mark.parametrize("prec", ["split", "fp64"])
def test_device_upper_matches_full(prec):
    import torch

    z = O.make_surrogate(300, 700, 3, seed=81)
    x = torch.from_numpy(z).cuda()
    _both(x, f"device-{prec}", input_kind="phasor", precision=prec, metrics=ALL)
    _both(x, f"device-{prec}-none", input_kind="phasor", precision=prec, metrics=ALL, trial_reduce="none")
    _both(x, f"device-{prec}-pool", input_kind="phasor", precision=prec, metrics=ALL, trial_reduce="pool")


def test_device_upper_leaves_caller_lower_untouched():
    import torch

    z = O.make_surrogate(200, 400, 1, seed=82)
    x = torch.from_numpy(z).cuda()
    out = {m: torch.full((1, 200, 200), 7.0, dtype=torch.float32, device="cuda") for m in ("plv", "ciplv")}
    C.plv_family(x, input_kind="phasor", metrics=("plv", "ciplv"), layout="upper", out=out)
    ref = C.plv_family(x, input_kind="phasor", metrics=("plv", "ciplv"))
    il = np.tril_indices(200, -1)
    iu = np.triu_indices(200)
    for m in out:
        o = out[m][0].cpu().numpy()
        assert np.all(o[il] == 7.0), m
        assert np.array_equal(o[iu], ref[m].values.cpu().numpy()[iu]), m


def test_host_paths_upper_match_full():
    rng = np.random.default_rng(83)
    # non-pipelined host path (small N)
    x = rng.standard_normal((256, 900, 2)).astype(np.float32)
    _both(x, "host-small", input_kind="real", metrics=ALL)
    # pipelined host path (N >= 2048, >= 148 tiles): growing stages, diagonal blocks
    xp = rng.standard_normal((4100, 300)).astype(np.float32)
    full, upper = _both(xp, "host-pipelined", input_kind="real", metrics=("plv", "iplv", "ciplv"))
    assert upper["plv"].meta["d2h_bytes"] < 0.7 * full["plv"].meta["d2h_bytes"]
    # pipelined, FP64
    _both(xp[:2304].astype(np.float64), "host-pipelined-fp64", input_kind="real", precision="fp64",
          metrics=("plv", "cim"))


def test_upper_with_trial_groups_and_refinement():
    # zero-lag clusters: many ill-conditioned ciPLV pairs refined in FP64 (the
    # refine writes must respect the layout too); R = 6 small N -> the trial-
    # group reduction path
    rng = np.random.default_rng(84)
    N, T, R, K = 384, 1024, 6, 32
    src = rng.standard_normal((N // K, T, R)) + 1j * rng.standard_normal((N // K, T, R))
    a = src[np.arange(N) // K] + 0.05 * (rng.standard_normal((N, T, R)) + 1j * rng.standard_normal((N, T, R)))
    a = a.astype(np.complex64)
    full, upper = _both(a, "refine-mean", input_kind="analytic", metrics=ALL)
    assert upper["ciplv"].meta["n_refined_pairs"] > 1000
    _both(a[:, :, :2], "refine-none", input_kind="analytic", metrics=ALL, trial_reduce="none")
    ref = O.plv_family(a.astype(np.complex128), input_kind="analytic")
    iu = np.triu_indices(N)
    for m in ("plv", "iplv", "ciplv"):
        assert np.max(np.abs(upper[m].values[iu] - ref[m][iu])) <= 1e-5, m


@pytest.mark.parametrize("R,reduce", [(1, "mean"), (3, "mean"), (2, "none")])
def test_host_pipelined_upper_streamed_with_refinement(R, reduce):
    # pipelined host path (N >= 2048, >= 148 tiles) with the upper layout: the
    # output sub-blocks are shipped while the Gram kernel still runs, and the
    # refined ciPLV entries (FP64, after their stage) come back as (index,
    # value) pairs that patch the received blocks -- upper entries bit-
    # identical to the full layout (which ships whole stage blocks after the
    # refinement), lower triangle zero
    rng = np.random.default_rng(87)
    N, T, K = 3072, 192, 48
    src = rng.standard_normal((N // K, T, R)) + 1j * rng.standard_normal((N // K, T, R))
    a = src[np.arange(N) // K] + 0.05 * (rng.standard_normal((N, T, R)) + 1j * rng.standard_normal((N, T, R)))
    # trials-first storage ([R, N, T] contiguous, viewed as [N, T, R]): unit
    # sample stride, the layout the pipelined host path requires
    a = np.transpose(np.ascontiguousarray(np.transpose(a, (2, 0, 1)).astype(np.complex64)), (1, 2, 0))
    full, upper = _both(a, f"host-stream-{R}-{reduce}", input_kind="analytic", trial_reduce=reduce,
                        metrics=("plv", "iplv", "ciplv", "cim"))
    assert upper["ciplv"].meta["n_refined_pairs"] > 1000
    # only the upper triangle (+ the strictly-lower corners of the 256-row
    # strips crossing the diagonal: 255 / N of it) and 12 B per refined entry
    # cross the link
    slots = R if reduce == "none" else 1
    exact = 4 * slots * N * (N + 1) // 2 * 4
    patch = 12 * upper["ciplv"].meta["n_refined_pairs"]
    assert exact <= upper["plv"].meta["d2h_bytes"] <= (1 + 256 / N) * exact + patch
    ref = O.plv_family(a[:300].astype(np.complex128), input_kind="analytic", trial_reduce=reduce)
    iu = np.triu_indices(300)
    for m in ("plv", "iplv", "ciplv"):
        v = upper[m].values
        v = v[:300, :300] if v.ndim == 2 else v[:300, :300, :]
        r = ref[m]
        assert np.max(np.abs(v[iu] - r[iu])) <= 1e-5, m


def test_upper_over_trials():
    z = np.exp(1j * np.random.default_rng(85).uniform(0, 6.3, (2, 40, 25, 11)))  # [B, N, T, R]
    _both(z, "over-trials", input_kind="phasor", bands=True, mode="over_trials", metrics=ALL)
    _both(z[0], "over-trials-fp64", input_kind="phasor", mode="over_trials", precision="fp64")


@pytest.mark.parametrize("mode", ["max", "mean", "none"])
def test_upper_coherence(mode):
    rng = np.random.default_rng(86)
    x = rng.standard_normal((70, 1024, 2))
    cfg = C.WelchConfig(window_len=128, overlap=64)
    full = C.coherence_matrix(x, cfg, (0.3, 0.9), mode=mode, metrics=("coh", "icoh", "cim"))
    upper = C.coherence_matrix(x, cfg, (0.3, 0.9), mode=mode, metrics=("coh", "icoh", "cim"), layout="upper")
    for m in full:
        _same_upper(full[m].values, upper[m].values, f"coh-{mode}:{m}")


def test_bad_layout_rejected():
    with pytest.raises(ValueError):
        C.plv_family(np.zeros((4, 16), np.float32), layout="lower")


def test_host_pipelined_upper_sharded_row_bands():
    # sharded calls on the streamed host path: each shard owns whole row bands
    # (dealt by work) and ships only those rows; the shards together give the
    # unsharded upper triangle bit for bit, each entry from exactly one shard
    rng = np.random.default_rng(88)
    N, T = 3200, 160
    x = rng.standard_normal((N, T)).astype(np.float32)
    ref = C.plv_family(x, input_kind="real", layout="upper", metrics=("plv", "ciplv"))
    P = 3
    parts = [C.plv_family(x, input_kind="real", layout="upper", metrics=("plv", "ciplv"), shard=(r, P))
             for r in range(P)]
    for m in ("plv", "ciplv"):
        owned = np.zeros((N, N), dtype=np.int32)
        acc = np.zeros((N, N), dtype=np.float32)
        for p in parts:
            v = p[m].values
            nz = np.any(v != 0, axis=1)  # rows this shard wrote
            owned[nz] += 1
            acc[nz] = v[nz]
            assert p[m].meta["d2h_bytes"] < 0.7 * ref[m].meta["d2h_bytes"]
        iu = np.triu_indices(N)
        assert np.array_equal(acc[iu], ref[m].values[iu]), m
        assert np.all(owned[np.arange(N - 1)] == 1), m  # every row (with an off-diagonal entry) from one shard


@pytest.mark.parametrize("layout", ["upper", "full"])
def test_device_input_host_outputs(layout):
    # ps_plv_family_to_host: CUDA input, numpy outputs -- same values as the
    # host path (streamed row bands for 'upper', column stages for 'full'),
    # sharded calls write only their rows; small N takes the unpipelined path
    import torch

    rng = np.random.default_rng(89)
    for N, T in ((3200, 160), (300, 200)):
        x = rng.standard_normal((N, T)).astype(np.float32)
        ref = C.plv_family(x, input_kind="real", layout=layout, metrics=("plv", "iplv", "ciplv"))
        xd = torch.from_numpy(x).cuda()
        outs = {m: np.zeros((1, N, N), np.float32) for m in ("plv", "iplv", "ciplv")}
        got = C.plv_family(xd, input_kind="real", layout=layout, out=outs)
        for m in outs:
            assert isinstance(got[m].values, np.ndarray)
            assert np.array_equal(got[m].values, ref[m].values), (N, layout, m)
        assert got["plv"].meta["h2d_bytes"] == 0
        if layout == "upper" and N >= 2048:
            acc = {m: np.zeros((N, N), np.float32) for m in outs}
            for r in range(2):
                o = {m: np.zeros((1, N, N), np.float32) for m in outs}
                C.plv_family(xd, input_kind="real", layout=layout, out=o, shard=(r, 2))
                for m in o:
                    rows = np.any(o[m][0] != 0, axis=1)
                    acc[m][rows] = o[m][0][rows]
            for m in outs:
                assert np.array_equal(acc[m][:-1], ref[m].values[:-1]), m


def test_all_gather_rows_nccl_single_rank():
    # the multi-GPU host-input path of bench.py (per-rank row slice -> NCCL
    # all-gather -> ps_plv_family_to_host) on a one-rank NCCL group
    import os

    import torch
    import torch.distributed as dist

    from paper_1710_08037_b200 import sharding

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(90)
        N, T = 2600, 128
        a = (rng.standard_normal((N, T)) + 1j * rng.standard_normal((N, T))).astype(np.complex64)
        r0, r1 = sharding.row_slice(N, 0, 1)
        loc = torch.view_as_real(torch.from_numpy(a[r0:r1]).pin_memory())
        xg = torch.view_as_complex(sharding.all_gather_rows(loc, N))
        outs = {m: np.zeros((1, N, N), np.float32) for m in ("plv", "iplv", "ciplv")}
        got = C.plv_family(xg, input_kind="analytic", layout="upper", out=outs, shard=(0, 1))
        ref = C.plv_family(a, input_kind="analytic", layout="upper")
        for m in outs:
            assert np.array_equal(got[m].values, ref[m].values), m
    finally:
        if own:
            dist.destroy_process_group()


@pytest.mark.parametrize("prec,dt,R", [("split", np.float32, 40), ("fp64", np.float64, 20)])
def test_host_trial_group_pipeline(prec, dt, R):
    # multi-trial trial means with >= 512 MB of host input (C2 / C4 shape):
    # the host path pipelines copy-in + normalise of trial group g+1 with the
    # Gram of group g; same values as the device path (up to the trial-group
    # summation order) and as the oracle, upper layout with a zero lower triangle
    import torch

    rng = np.random.default_rng(91)
    B, N, T = 2, 1024, 2048
    x = rng.standard_normal((B, R, N, T)).astype(dt)  # trials-outer storage, unit sample stride
    xv = np.transpose(x, (0, 2, 3, 1))                 # [B, N, T, R] view
    assert x.nbytes >= 512 << 20
    tol = 1e-5 if prec == "split" else 1e-12
    for layout in ("full", "upper"):
        host = C.plv_family(xv, input_kind="real", bands=True, precision=prec, layout=layout)
        assert host["plv"].meta["h2d_bytes"] == x.nbytes
        dev = C.plv_family(torch.from_numpy(x).cuda().permute(0, 2, 3, 1), input_kind="real", bands=True,
                           precision=prec, layout=layout)
        for m in ("plv", "iplv", "ciplv"):
            h = host[m].values
            d = dev[m].values.cpu().numpy()
            assert np.max(np.abs(h - d)) <= (2e-6 if prec == "split" else 1e-13), (layout, m)
            if layout == "upper":
                il = np.tril_indices(N, -1)
                assert not np.any(h[:, il[0], il[1]]), m
    sub = np.ascontiguousarray(xv[1, :64]).astype(np.float64)
    ref = O.plv_family(sub, input_kind="real")
    for m in ("plv", "iplv", "ciplv"):
        assert np.max(np.abs(host[m].values[1, :64, :64] - np.triu(ref[m]))) <= tol, m


def test_host_pipelined_upper_bands_and_trials():
    # streamed row-band copy-out with several bands and a trial mean (one
    # output slot per band): upper entries bit-identical to the full layout
    rng = np.random.default_rng(92)
    B, N, T, R = 2, 2304, 96, 3
    x = rng.standard_normal((B, R, N, T)).astype(np.float32)
    xv = np.transpose(x, (0, 2, 3, 1))  # [B, N, T, R], unit sample stride
    full, upper = _both(xv, "host-stream-bands", input_kind="real", bands=True,
                        metrics=("plv", "iplv", "ciplv"))
    exact = 3 * B * N * (N + 1) // 2 * 4
    assert upper["plv"].meta["d2h_bytes"] <= (1 + 256 / N) * exact


_UNIT_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_1710_08037_b200 import connectivity as C
rng = np.random.default_rng(93)
worst = 0.0
for B, R, N, T, prec, layout in ((2, 6, 300, 512, "split", "full"), (1, 7, 520, 256, "fp64", "upper"),
                                 (3, 5, 129, 300, "split", "upper")):
    x = rng.standard_normal((B, R, N, T)).astype(np.float32 if prec == "split" else np.float64)
    xv = np.transpose(x, (0, 2, 3, 1))
    host = C.plv_family(xv, input_kind="real", bands=True, precision=prec, layout=layout)
    assert host["plv"].meta["h2d_bytes"] == x.nbytes
    dev = C.plv_family(torch.from_numpy(x).cuda().permute(0, 2, 3, 1), input_kind="real", bands=True,
                       precision=prec, layout=layout)
    for m in ("plv", "iplv", "ciplv"):
        worst = max(worst, float(np.max(np.abs(host[m].values - dev[m].values.cpu().numpy()))))
print(worst)
"""


def test_host_trial_group_pipeline_small_shapes():
    # the trial-group host pipeline forced onto small inputs (PS_UNIT_PIPE_MIN_MB=1,
    # read once per process, hence the subprocess): uneven tile counts, prime
    # trial counts, fp64 upper layout -- same values as the device path
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PS_UNIT_PIPE_MIN_MB="1")
    out = subprocess.run([sys.executable, "-c", _UNIT_SCRIPT, root], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) <= 2e-6


def test_host_pipelined_growing_stage_counts_reuse_context():
    # Regression: a streamed host call that needs more pipeline stages than any
    # earlier call on the same context regrows the per-stage counters; the
    # sub-block flag buffer (mapped pinned memory) must survive that -- it was
    # freed there without being reset (later calls then wrote their flags
    # into freed memory or freed it twice).  Small -> large -> small -> large
    # again, each bit-identical to the device path.
    import torch

    rng = np.random.default_rng(91)
    for N in (3072, 9216, 3328, 12288):
        z = np.exp(1j * rng.uniform(0, 2 * np.pi, (N, 64))).astype(np.complex64)
        host = C.plv_family(z, input_kind="phasor", layout="upper")
        dev = C.plv_family(torch.from_numpy(z).cuda(), input_kind="phasor", layout="upper")
        iu = np.triu_indices(N)
        for m in ("plv", "iplv", "ciplv"):
            assert np.array_equal(host[m].values[iu], dev[m].values.cpu().numpy()[iu]), (N, m)
