"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/phasesync.h declares; host-only helpers work without a GPU.  No
compute call is made here."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1710_08037_b200 import _native, errors, sharding

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "phasesync.h")).read()
    return sorted(set(re.findall(r"^\s*(?:ps_status|int|int32_t|int64_t|const char\*)\s+(ps_\w+)\s*\(", txt, re.M)))


def test_library_exports_header_symbols():
    lib = _native.lib()
    syms = header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _native._SIGNATURES, f"binding lacks a signature for {s}"
    assert lib.ps_abi_version() == _native.ABI_VERSION


def test_struct_layout_matches_header():
    # ps_plv_args: 8 + 2*4 + 8*8 + 8 + 3*4 (+4 pad) + 5*8 + 2*4 + 8 + 2*4 + 8 (fir)
    assert ctypes.sizeof(_native.PlvArgs) == 8 + 8 + 64 + 8 + 16 + 40 + 8 + 8 + 8 + 8
    assert _native.PlvArgs.fir.offset == ctypes.sizeof(_native.PlvArgs) - 8
    assert ctypes.sizeof(_native.PlvResult) == 3 * 8 + 2 * 4 + 4 * 4 + 2 * 8 + 2 * 4
    assert ctypes.sizeof(_native.Fir) == 24


def test_fir_design_host_matches_oracle_and_validates():
    import warnings

    import numpy as np

    from oracle import plv_oracle as O
    from paper_1710_08037_b200 import signalprep as S

    f = S.design_bandpass_fir((0.57 * np.pi, 0.6 * np.pi), 2000)
    assert f.order == 2000 and f.taps.shape == (2001,)
    assert np.array_equal(f.taps, O.design_bandpass_fir(0.57 * np.pi, 0.6 * np.pi, 2000))
    with pytest.raises(errors.InvalidBandError):
        S.design_bandpass_fir((0.6, 0.5), 100)
    with pytest.raises(errors.InvalidBandError):
        S.design_bandpass_fir((0.5, 4.0), 100)
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        S.design_bandpass_fir((0.25 * np.pi, 0.75 * np.pi), 10)
    assert any(issubclass(x.category, errors.OrderTooSmallWarning) for x in w)
    assert _native.STATUS_EXC[10] is errors.SignalTooShortError


def test_welch_bins_host_helper_matches_oracle():
    import numpy as np

    from oracle import plv_oracle as O
    from paper_1710_08037_b200 import connectivity as C

    assert ctypes.sizeof(_native.Welch) == 40
    assert _native.STATUS_EXC[11] is errors.WindowTooLongError
    assert _native.STATUS_EXC[12] is errors.EmptyBandError
    rng = np.random.default_rng(3)
    cases = [(200, 0.57 * np.pi, 0.6 * np.pi), (100, 0.0, np.pi), (400, 0.1, 0.1), (7, 0.5, 2.0)]
    for _ in range(50):
        lo, hi = sorted(rng.uniform(0, np.pi, 2))
        cases.append((int(rng.integers(2, 600)), lo, hi))
    for W, lo, hi in cases:
        assert C.welch_bins(W, (lo, hi)) == O.welch_bins(W, lo, hi), (W, lo, hi)


def test_ctx_create_fails_cleanly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    with pytest.raises((errors.CudaError, errors.UnsupportedError, ValueError)):
        _native.Context(0)


def test_status_map_is_the_reference_taxonomy():
    assert _native.STATUS_EXC[1] is errors.ShapeError
    assert _native.STATUS_EXC[2] is errors.AllSamplesMaskedError
    assert _native.STATUS_EXC[3] is errors.EmptyEffectiveWindowError
    assert issubclass(errors.ShapeError, ValueError)
    assert issubclass(errors.OutputMismatchError, RuntimeError)


@pytest.mark.parametrize("prec", ["split", "fp64"])
@pytest.mark.parametrize("N", [1, 2, 63, 64, 127, 128, 129, 255, 256, 257, 1200, 2500])
def test_tile_enumeration_matches_library(N, prec):
    assert _native.tile_count(N, prec) == len(sharding.tiles(N, prec))


@pytest.mark.parametrize("prec", ["split", "fp64"])
@pytest.mark.parametrize("N,W", [(300, 2), (1200, 4), (700, 8), (5, 3)])
def test_every_pair_owned_exactly_once(N, W, prec):
    own = sharding.owner_matrix(N, prec, W)
    assert own.min() >= 0 and own.max() < W
    assert np.array_equal(own, own.T)
    rng = np.random.default_rng(N * W)
    for i, j in rng.integers(0, N, size=(200, 2)):
        assert _native.pair_shard(N, prec, W, int(i), int(j)) == own[i, j]
