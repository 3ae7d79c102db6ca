"""SPEC.md:94-111 examples for the elementwise signal-prep operations
(instantaneous_phase, downsample).  They run on the input's own device and
need no GPU for host arrays."""
import math
import warnings

import numpy as np
import pytest

from phasesync import errors, signalprep as S


def test_instantaneous_phase_examples():
    # e^{i pi/4} -> pi/4; -1 + 0i -> pi (branch (-pi, pi]); 0 -> 0
    ph = S.instantaneous_phase(np.array([np.exp(1j * np.pi / 4), -1 + 0j, complex(-1.0, -0.0), 0j]))
    assert ph[0] == pytest.approx(np.pi / 4, abs=1e-15)
    assert ph[1] == np.pi and ph[2] == np.pi and ph[3] == 0.0


def test_instantaneous_phase_slope_of_analytic_cosine():
    # unwrapped phase of analytic cos(w0 t) has slope w0 (interior samples)
    w0 = 2 * np.pi * 50 / 1000
    t = np.arange(2000)
    a = np.cos(w0 * t) + 1j * np.sin(w0 * t)
    ph = np.unwrap(S.instantaneous_phase(S.AnalyticEpochs(a[None, :])))[0, 100:-100]
    slope = np.polyfit(np.arange(ph.size), ph, 1)[0]
    assert abs(slope - w0) < 1e-6


def test_instantaneous_phase_amplitude_invariant():
    # phase of z = a / |a| equals the phase of a
    rng = np.random.default_rng(3)
    a = rng.standard_normal((4, 64, 2)) + 1j * rng.standard_normal((4, 64, 2))
    np.testing.assert_allclose(S.instantaneous_phase(a / np.abs(a)), S.instantaneous_phase(a), atol=1e-12)


def test_instantaneous_phase_torch_tensor():
    torch = pytest.importorskip("torch")
    a = torch.tensor([complex(-1.0, -0.0), 1j, 0j], dtype=torch.complex128)
    ph = S.instantaneous_phase(a)
    assert isinstance(ph, torch.Tensor)
    assert ph.tolist() == [math.pi, math.pi / 2, 0.0]


def test_downsample_examples():
    # SPEC.md:109-111
    x = np.zeros((3, 4000, 2))
    assert S.downsample(x, 10).shape == (3, 400, 2)
    y = np.random.default_rng(0).standard_normal((2, 50))
    assert np.array_equal(S.downsample(y, 1), y)
    s = np.cos(0.05 * np.pi * np.arange(4000))[None, :, None]
    r = S.downsample(S.RealEpochs(s, fs=1000.0), 10)
    assert r.fs == 100.0
    k = np.arange(400)
    np.testing.assert_allclose(r.data[0, :, 0], np.cos(0.5 * np.pi * k), atol=1e-12)


def test_downsample_errors_and_aliasing_warning():
    with pytest.raises(errors.FactorTooLargeError):
        S.downsample(np.zeros((2, 10)), 10)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        S.downsample(np.cos(0.05 * np.pi * np.arange(4000))[None, :], 10)  # band-limited: silent
    with pytest.warns(errors.AliasingWarning):
        S.downsample(np.random.default_rng(0).standard_normal((2, 4000)), 10)


def test_reference_module_names_resolve():
    # reference code importing the simulator / bench modules finds them
    import numpy as np
    from phasesync import bench, chaossim

    z = bench.make_surrogate(5, 40, 2, seed=1)
    assert z.data.shape == (5, 40, 2) and np.allclose(np.abs(z.data), 1.0, atol=1e-12)
    assert np.array_equal(bench.make_surrogate(5, 40, 2, seed=1).data, z.data)
    with pytest.raises(NotImplementedError, match="SPEC.md:281-377"):
        chaossim.integrate_coupled(None)
    with pytest.raises(NotImplementedError, match="SPEC.md:379-433"):
        bench.run_benchmark(None)
