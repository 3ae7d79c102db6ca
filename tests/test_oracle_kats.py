"""Pins the CPU oracle against every closed-form known answer and invariant
the reference SPEC states for the hot path (the reference ships no tests or
golden vectors -- SURVEY 8(c)).  CPU only."""
import numpy as np
import pytest
import scipy.signal

from oracle import plv_oracle as O

RNG = np.random.default_rng(1234)


# ---------------------------------------------------------------- analytic
def test_analytic_cosine_unit_modulus():
    # SPEC.md:82 x = cos(w0 t), w0 = 0.25 pi -> |analytic| ~ 1 (edges excluded)
    T = 64  # 8 whole cycles: the discrete construction is exact everywhere
    t = np.arange(T)
    a = O.analytic_signal(np.cos(0.25 * np.pi * t)[None, :, None])
    assert np.max(np.abs(np.abs(a) - 1.0)) < 1e-12
    T = 1000  # non-periodic: interior samples only
    a = O.analytic_signal(np.cos(0.25 * np.pi * np.arange(T))[None, :, None])
    assert np.max(np.abs(np.abs(a[0, 100:-100, 0]) - 1.0)) < 2e-2


def test_analytic_sine_phase():
    # phase of analytic(sin(w0 t)) = w0 t - pi/2 (mod 2 pi)
    T = 64
    t = np.arange(T)
    a = O.analytic_signal(np.sin(0.25 * np.pi * t)[None, :, None])[0, :, 0]
    d = np.angle(a * np.exp(-1j * (0.25 * np.pi * t - np.pi / 2)))
    assert np.max(np.abs(d)) < 1e-12


def test_analytic_real_part_bit_exact():
    # SPEC.md:84
    x = RNG.standard_normal((5, 333, 2))
    a = O.analytic_signal(x)
    assert np.array_equal(a.real, x)


@pytest.mark.parametrize("T", [2, 3, 64, 2000, 2001, 4096])
def test_analytic_matches_scipy_hilbert(T):
    # SPEC.md:124 weights == scipy.signal.hilbert's construction (even and odd T)
    x = RNG.standard_normal((3, T))
    a = O.analytic_signal(x, axis=1)
    ref = scipy.signal.hilbert(x, axis=1)
    assert np.max(np.abs(a.imag - ref.imag)) < 1e-12 * max(1.0, np.abs(x).max() * np.sqrt(T))


def test_analytic_linear_and_equal_energy():
    # SPEC.md:115-116
    T = 4096
    x = RNG.standard_normal((4, T, 1))
    y = RNG.standard_normal((4, T, 1))
    al, be = 0.7, -1.3
    lhs = O.analytic_signal(al * x + be * y)
    rhs = al * O.analytic_signal(x) + be * O.analytic_signal(y)
    assert np.max(np.abs(lhs - rhs)) < 1e-10
    X = np.fft.rfft(RNG.standard_normal((4, T)), axis=1)
    f = np.arange(T // 2 + 1) * 1000.0 / T
    X[:, (f < 8) | (f > 12)] = 0
    bl = np.fft.irfft(X, T, axis=1)[:, :, None]
    a = O.analytic_signal(bl)
    er, ei = np.mean(a.real ** 2, axis=1), np.mean(a.imag ** 2, axis=1)
    assert np.all(np.abs(er / ei - 1) < 0.05)


# ---------------------------------------------------------------- normalise
def test_normalize_kats():
    # SPEC.md:91-93
    a = np.full((1, 8, 1), 3 * np.exp(1j * 1.2))
    z, m = O.normalize_phasors(a)
    assert np.allclose(z, np.exp(1j * 1.2), atol=1e-15) and not m.any()
    a = np.exp(1j * RNG.uniform(-np.pi, np.pi, (2, 16, 1)))
    a[0, 3, 0] = 0
    z, m = O.normalize_phasors(a)
    assert z[0, 3, 0] == 0 and m[0, 3, 0] and m.sum() == 1
    c = 2.5 * np.exp(1j * RNG.uniform(-np.pi, np.pi, (3, 10, 2)))
    z, m = O.normalize_phasors(c)
    assert not m.any() and np.max(np.abs(z - c / np.abs(c))) < 1e-15


def test_normalize_all_masked_raises():
    a = np.ones((2, 8, 1), complex)
    a[1] = 0
    with pytest.raises(O.AllSamplesMaskedError):
        O.normalize_phasors(a)


def test_normalize_median_floor_even_T():
    # numpy median of an even row is the mean of the two middle values
    amp = np.array([1e-9, 1.0, 3.0, 5.0])
    a = amp[None, :, None].astype(complex)
    z, m = O.normalize_phasors(a, amp_floor=0.5)  # median 2.0 -> floor 1.0
    assert list(m[0, :, 0]) == [True, False, False, False]
    z, m = O.normalize_phasors(a, amp_floor=0.6)  # floor 1.2 masks 1.0 too
    assert list(m[0, :, 0]) == [True, True, False, False]


def test_phase_amplitude_invariance():
    # SPEC.md:117
    a = RNG.standard_normal((3, 50, 2)) + 1j * RNG.standard_normal((3, 50, 2))
    z, m = O.normalize_phasors(a)
    assert np.max(np.abs(np.angle(z) - np.angle(a))) < 1e-12


# ---------------------------------------------------------------- PLV family
def test_plv_reference_kats():
    # SPEC.md:176-178
    ph = RNG.uniform(-np.pi, np.pi, (1, 100, 1))
    ph2 = np.concatenate([ph, ph + 0.77], axis=0)
    ph2 = np.angle(np.exp(1j * ph2))
    assert abs(O.plv_reference(ph2)[0, 1, 0] - 1) < 1e-12
    canc = np.array([[[0.0], [0.0], [0.0], [0.0]], [[0.0], [np.pi / 2], [np.pi], [3 * np.pi / 2]]])
    assert O.plv_reference(np.angle(np.exp(1j * canc)))[0, 1, 0] < 1e-12


def test_random_phase_floor():
    # SPEC.md:177,574 (acceptance #8): mean PLV of independent uniform phases
    T = 10_000
    d = RNG.uniform(-np.pi, np.pi, (1000, T)) - RNG.uniform(-np.pi, np.pi, (1000, T))
    v = np.abs(np.mean(np.exp(1j * d), axis=1))
    assert abs(v.mean() - np.sqrt(np.pi / (4 * T))) < 0.005


def test_vectorized_equals_reference():
    # SPEC.md:183
    ph = RNG.uniform(-np.pi, np.pi, (20, 256, 3))
    assert np.max(np.abs(O.plv_vectorized(ph) - O.plv_reference(ph))) < 1e-10


def test_matrix_equals_reference():
    # SPEC.md:192
    z = O.make_surrogate(20, 512, 5, seed=7)
    ph = np.angle(z)
    ref = O.plv_reference(ph)
    got = O.plv_family(z, input_kind="phasor", trial_reduce="none")["plv"]
    assert np.max(np.abs(got - ref)) < 1e-9


def test_oracle_equivalence_grid():
    # SPEC.md:249 / acceptance #1: >= 30 random shapes in {2-50} x {16-1024} x {1-8}
    rng = np.random.default_rng(2024)
    for _ in range(30):
        N = int(rng.integers(2, 51))
        T = int(rng.integers(16, 1025))
        R = int(rng.integers(1, 9))
        if N * N * T * R > 3_000_000:
            T = max(16, 3_000_000 // (N * N * R))
        z = O.make_surrogate(N, T, R, seed=int(rng.integers(1 << 30)))
        ph = np.angle(z)
        got = O.plv_family(z, input_kind="phasor", trial_reduce="none")["plv"]
        vec = O.plv_vectorized(ph) if N * T * R < 40_000 else None
        ref = O.plv_reference(ph)
        assert np.max(np.abs(got - ref)) < 1e-9, (N, T, R)
        if vec is not None:
            assert np.max(np.abs(vec - ref)) < 1e-9


@pytest.mark.parametrize("phi", [np.pi / 6, np.pi / 4, np.pi / 2, 3 * np.pi / 4])
def test_constant_offset_exactness(phi):
    # SPEC.md:202-203,210 / acceptance #3
    z0 = np.exp(1j * RNG.uniform(-np.pi, np.pi, (1, 1000, 1)))
    z = np.concatenate([z0, z0 * np.exp(-1j * phi)], axis=0)
    r = O.plv_family(z, input_kind="phasor")
    assert abs(r["plv"][0, 1] - 1) < 1e-9
    assert abs(r["iplv"][0, 1] - abs(np.sin(phi))) < 1e-9
    assert abs(r["ciplv"][0, 1] - 1) < 1e-9


def test_zero_lag_kats():
    z0 = np.exp(1j * RNG.uniform(-np.pi, np.pi, (1, 500, 1)))
    z = np.concatenate([z0, z0], axis=0)
    r = O.plv_family(z, input_kind="phasor")
    assert abs(r["plv"][0, 1] - 1) < 1e-12
    assert r["iplv"][0, 1] < 1e-12
    assert r["ciplv"][0, 1] == 0.0  # singularity rule SPEC.md:211,259
    assert r["plv"][0, 0] == 1.0 and r["iplv"][1, 1] == 0.0 and r["ciplv"][0, 0] == 0.0


def test_ciplv_random_small():
    # SPEC.md:212
    z = O.make_surrogate(2, 10_000, 50, seed=3)
    c = O.plv_family(z, input_kind="phasor", trial_reduce="none")["ciplv"][0, 1, :]
    assert np.mean(c < 0.05) > 0.99 - 1e-12 or np.all(c < 0.05)


def test_bounds_and_invariances():
    # SPEC.md:250-253
    z = O.make_surrogate(12, 300, 2, seed=11)
    r = O.plv_family(z, input_kind="phasor", trial_reduce="none")
    p, i, c = r["plv"], r["iplv"], r["ciplv"]
    assert np.all(i <= p + 1e-12) and np.all(i <= c + 1e-12) and np.all(p <= 1 + 1e-9) and np.all(c <= 1 + 1e-9)
    for k in range(2):
        assert np.max(np.abs(p[:, :, k] - p[:, :, k].T)) < 1e-12
    rot = z.copy()
    rot[3] *= np.exp(1j * 0.9)
    assert np.max(np.abs(O.plv_family(rot, input_kind="phasor", trial_reduce="none")["plv"] - p)) < 1e-12
    perm = RNG.permutation(12)
    rp = O.plv_family(z[perm], input_kind="phasor", trial_reduce="none")
    for m in ("plv", "iplv", "ciplv"):
        assert np.max(np.abs(rp[m] - r[m][np.ix_(perm, perm)])) < 1e-12
    a = z * RNG.uniform(0.5, 3.0, (12, 1, 1))
    ra = O.plv_family(a, input_kind="analytic", trial_reduce="none")
    for m in ("plv", "iplv", "ciplv"):
        assert np.max(np.abs(ra[m] - r[m])) < 1e-12


def test_masked_pairs_effective_T():
    # SPEC.md:260
    z = O.make_surrogate(4, 40, 1, seed=5)
    z[0, :10, 0] = 0
    z[1, 5:15, 0] = 0
    zz, m = O.phasors_from_unit(z)
    r = O.plv_family_from_phasors(zz, m, "none", raw=True)
    both = ~m[0, :, 0] & ~m[1, :, 0]
    g = np.sum(z[0, :, 0] * np.conj(z[1, :, 0])) / both.sum()
    assert abs(r["plv"][0, 1, 0] - abs(g)) < 1e-12
    z[2, :, 0] = 0
    with pytest.raises(O.AllSamplesMaskedError):
        O.plv_family(z, input_kind="phasor")
    z = O.make_surrogate(2, 8, 1, seed=5)
    z[0, :4, 0] = 0
    z[1, 4:, 0] = 0
    with pytest.raises(O.EmptyEffectiveWindowError):
        O.plv_family(z, input_kind="phasor")


def test_von_mises_monotone():
    # SPEC.md:255
    rng = np.random.default_rng(9)
    vals = []
    for kappa in (0.0, 1.0, 4.0, 16.0):
        d = rng.vonmises(0.0, kappa, size=100_000) if kappa > 0 else rng.uniform(-np.pi, np.pi, 100_000)
        z = np.stack([np.ones(100_000), np.exp(-1j * d)])[:, :, None]
        vals.append(O.plv_family(z, input_kind="phasor")["plv"][0, 1])
    assert all(b > a + 3 * 0.01 for a, b in zip(vals, vals[1:]))


def test_over_trials_mode():
    # Eq 8: PLV_ij(t) = |mean over trials of exp(i (phi_i(t,n) - phi_j(t,n)))|
    z = O.make_surrogate(5, 12, 9, seed=4)
    ph = np.angle(z)
    got = O.plv_matrix(z, mode="over_trials")
    for t in range(12):
        for a in range(5):
            for b in range(5):
                ref = 1.0 if a == b else abs(np.mean(np.exp(1j * (ph[a, t] - ph[b, t]))))
                assert abs(got[a, b, t] - ref) < 1e-12
    fam = O.plv_family_over_trials(*O.phasors_from_unit(z))
    assert np.all(fam["iplv"] <= fam["plv"] + 1e-12)


def test_trial_reduce_modes():
    z = O.make_surrogate(6, 64, 3, seed=21)
    none = O.plv_family(z, input_kind="phasor", trial_reduce="none")
    mean = O.plv_family(z, input_kind="phasor", trial_reduce="mean")
    pool = O.plv_family(z, input_kind="phasor", trial_reduce="pool")
    assert np.allclose(mean["plv"], none["plv"].mean(axis=2), atol=1e-15)
    zz = np.transpose(z, (0, 2, 1)).reshape(6, -1)
    g = zz @ zz.conj().T / zz.shape[1]
    p = np.abs(g)
    np.fill_diagonal(p, 1)
    assert np.allclose(pool["plv"], p, atol=1e-14)


# ----------------------------------------- band-pass front end
def _dtft(h, w):
    return np.sum(h * np.exp(-1j * w * np.arange(h.size)))


def test_fir_design_kats():
    # [0.570pi, 0.600pi], order 2000 -> |H(0.585pi)| within +-1 dB
    h = O.design_bandpass_fir(0.570 * np.pi, 0.600 * np.pi, 2000)
    assert h.size == 2001
    assert abs(20 * np.log10(abs(_dtft(h, 0.585 * np.pi)))) < 1.0
    assert np.max(np.abs(h - h[::-1])) < 1e-16  # linear phase (to rounding)
    # [0.25pi, 0.75pi], order 10 -> centre response ~ 1
    h10 = O.design_bandpass_fir(0.25 * np.pi, 0.75 * np.pi, 10)
    assert abs(abs(_dtft(h10, 0.5 * np.pi)) - 1.0) < 1e-12
    # low >= high -> InvalidBand
    with pytest.raises(O.InvalidBandError):
        O.design_bandpass_fir(0.6 * np.pi, 0.5 * np.pi, 100)
    with pytest.raises(O.InvalidBandError):
        O.design_bandpass_fir(0.5, 3.5, 100)


def test_fir_design_pinned_to_scipy_firwin():
    # the SPEC's design decision (windowed sinc, Hamming) is
    # scipy.signal.firwin(..., window='hamming', scale=True): pin the restatement
    for lo, hi, order in [(0.57, 0.6, 2000), (0.25, 0.75, 10), (0.016, 0.024, 800)]:
        h = O.design_bandpass_fir(lo * np.pi, hi * np.pi, order)
        ref = scipy.signal.firwin(order + 1, [lo, hi], pass_zero=False, window="hamming", scale=True)
        assert np.max(np.abs(h - ref)) < 1e-14


def test_two_pass_matches_lfilter_definition():
    # forward, reverse, forward, reverse with zero initial state
    rng = np.random.default_rng(11)
    x = rng.standard_normal((3, 700, 2))
    h = O.design_bandpass_fir(0.2 * np.pi, 0.4 * np.pi, 60)
    pad = 100
    xp = np.pad(x, ((0, 0), (pad, pad), (0, 0)), mode="reflect")
    y = scipy.signal.lfilter(h, [1.0], xp, axis=1)
    y = scipy.signal.lfilter(h, [1.0], y[:, ::-1], axis=1)[:, ::-1]
    assert np.max(np.abs(O.two_pass_padded(x, h, pad) - y)) < 1e-13
    assert np.max(np.abs(O.filter_two_pass(x, h, pad) - y[:, pad:pad + 700])) < 1e-13


def test_two_pass_zero_phase_and_attenuation():
    h = O.design_bandpass_fir(0.2 * np.pi, 0.3 * np.pi, 200)
    T, pad = 4000, 1000
    t = np.arange(T)
    # band-centre sinusoid -> zero phase shift (xcorr peak at lag 0)
    x = np.cos(0.25 * np.pi * t)
    y = O.filter_two_pass(x[None, :, None], h, pad)[0, :, 0]
    mid = slice(500, T - 500)
    lags = np.arange(-5, 6)
    xc = [np.dot(x[mid], np.roll(y, k)[mid]) for k in lags]
    assert lags[int(np.argmax(xc))] == 0
    # single-pass -10 dB -> two-pass -20 dB +- 1 dB
    w = np.linspace(0.05 * np.pi, 0.2 * np.pi, 20000)
    mag = 20 * np.log10(np.abs(np.exp(-1j * np.outer(w, np.arange(h.size))) @ h))
    w10 = w[np.argmin(np.abs(mag + 10.0))]
    s = np.cos(w10 * t)
    ys = O.filter_two_pass(s[None, :, None], h, pad)[0, :, 0]
    gain = 20 * np.log10(np.std(ys[mid]) / np.std(s[mid]))
    assert abs(gain + 20.0) < 1.0


def test_two_pass_white_noise_band_limited():
    # power outside [low - tw, high + tw] < 1% of total
    rng = np.random.default_rng(12)
    lo, hi, order = 0.2 * np.pi, 0.3 * np.pi, 400
    h = O.design_bandpass_fir(lo, hi, order)
    x = rng.standard_normal((1, 20000, 1))
    y = O.filter_two_pass(x, h, 2000)[0, :, 0]
    f, p = scipy.signal.periodogram(y)
    w = 2 * np.pi * f
    tw = 3.3 * 2 * np.pi / order  # Hamming transition width
    out = (w < lo - tw) | (w > hi + tw)
    assert p[out].sum() < 0.01 * p.sum()


def test_two_pass_too_short_and_bandpass_analytic_trim():
    h = O.design_bandpass_fir(0.2 * np.pi, 0.4 * np.pi, 60)
    with pytest.raises(O.SignalTooShortError):
        O.filter_two_pass(np.zeros((1, 61, 1)), h, 10)
    rng = np.random.default_rng(13)
    x = rng.standard_normal((2, 500, 1))
    a = O.bandpass_analytic(x, h, 120)
    assert a.shape == x.shape
    # Re is the filtered record bit-exactly; H comes from the padded record
    assert np.array_equal(a.real, O.filter_two_pass(x, h, 120))
    full = O.analytic_signal(O.two_pass_padded(x, h, 120))
    assert np.array_equal(a, full[:, 120:620])


# ---------------------------------------- Welch coherence
def test_coherence_pinned_to_scipy():
    # magnitude coherence = sqrt(scipy's magnitude-squared coherence) with the
    # same Hamming segments and no detrending
    rng = np.random.default_rng(40)
    x = rng.standard_normal((2, 5000))
    for W, ov in [(400, 200), (100, 50), (128, 0)]:
        c = O.coherence_welch(x[:, :, None], W, ov)
        _, c2 = scipy.signal.coherence(x[0], x[1], window=np.hamming(W), nperseg=W, noverlap=ov, detrend=False)
        assert np.max(np.abs(np.sqrt(c2) - c)) < 1e-12


def test_coherence_kats():
    rng = np.random.default_rng(41)
    W, ov = 100, 50
    # identical signals -> 1 at every bin with power
    x = rng.standard_normal((1, 3000, 2))
    c = O.coherence_welch(np.concatenate([x, x]), W, ov)
    assert np.max(np.abs(c - 1.0)) < 1e-12
    # equal-frequency tones, constant offset, -20 dB independent noise -> > 0.95 at the tone bin
    T = 50 * 50 + 50
    t = np.arange(T)
    k = 12
    w0 = 2 * np.pi * k / W
    s = np.stack([np.cos(w0 * t), np.cos(w0 * t + 0.7)]) + 0.1 * rng.standard_normal((2, T))
    assert O.coherence_welch(s[:, :, None], W, ov)[k] > 0.95
    # independent white noise, 99 segments -> mean ~ sqrt(pi / (4 * 99)) +- 0.03
    T = 98 * 50 + 100
    x = rng.standard_normal((2, T, 1))
    assert abs(O.coherence_welch(x, W, ov).mean() - np.sqrt(np.pi / (4 * 99))) < 0.03


def test_coherence_weighted_phasor_identity():
    rng = np.random.default_rng(42)
    x = rng.standard_normal((2, 4000, 3))
    assert np.max(np.abs(O.coherence_weighted_phasor(x, 200, 100) - O.coherence_welch(x, 200, 100))) < 1e-10
    # one segment dominating the amplitude by 1e3 -> ~1
    y = rng.standard_normal((2, 1000, 1))
    y[:, :100] *= 1e3
    c = O.coherence_weighted_phasor(y, 100, 0)
    assert np.all(c[1:-1] > 0.99)


def test_imaginary_coherency_kats():
    W, ov = 100, 50
    T = 40 * 50 + 50
    t = np.arange(T)
    k = 10
    w0 = 2 * np.pi * k / W
    rng = np.random.default_rng(43)
    x = rng.standard_normal((1, T, 1))
    assert np.max(O.imaginary_coherency(np.concatenate([x, x]), W, ov)) < 1e-12
    for shift, scale in ((np.pi / 2, 1.0), (np.pi / 6, 0.5)):
        s = np.stack([np.cos(w0 * t), np.cos(w0 * t + shift)])[:, :, None]
        ic = O.imaginary_coherency(s, W, ov)[k]
        assert abs(ic - scale * O.coherence_welch(s, W, ov)[k]) < 0.02


def test_band_coherence_and_bins():
    W = 200
    assert O.welch_bins(W, 0.570 * np.pi, 0.600 * np.pi) == (57, 4)
    flat = np.full(W // 2 + 1, 0.3)
    assert O.band_coherence(flat, W, 0.5, 1.0, "max") == 0.3
    assert abs(O.band_coherence(flat, W, 0.5, 1.0, "mean") - 0.3) < 1e-15
    peak = flat.copy()
    peak[20] = 0.9
    lo, hi = 2 * np.pi * 18 / W, 2 * np.pi * 22 / W
    assert O.band_coherence(peak, W, lo, hi, "max") == 0.9
    assert O.band_coherence(peak, W, lo, hi, "mean") < 0.9
    with pytest.raises(O.EmptyBandError):
        O.band_coherence(flat, W, 0.0101, 0.0102)
    with pytest.raises(O.WindowTooLongError):
        O.coherence_welch(np.zeros((2, 50, 1)), 100, 10)


def test_coherence_matrix_matches_pairwise():
    rng = np.random.default_rng(44)
    x = rng.standard_normal((5, 1200, 2))
    x[3] = 0.6 * x[1] + 0.4 * x[3]
    W, ov, lo, hi = 100, 50, 0.3, 1.2
    for mode in ("max", "mean"):
        M = O.coherence_matrix(x, W, ov, lo, hi, mode)
        for i in range(5):
            for j in range(5):
                if i == j:
                    continue
                c = O.coherence_welch(x[[i, j]], W, ov)
                ic = O.imaginary_coherency(x[[i, j]], W, ov)
                assert abs(M["coh"][i, j] - O.band_coherence(c, W, lo, hi, mode)) < 1e-12
                assert abs(M["icoh"][i, j] - O.band_coherence(ic, W, lo, hi, mode)) < 1e-12
