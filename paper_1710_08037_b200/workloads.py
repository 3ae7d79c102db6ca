"""Seeded synthetic inputs for the five BASELINE.json configurations.

The paper's MEG recordings / beamformer sources are not
available; BASELINE.json describes synthetic stand-ins and SURVEY.md section
8(d) pins their generative details (seeds 1-5, decisions D3/D4).  Every
generator is deterministic in ``numpy.random.default_rng(seed)`` and returns
an array whose *shape* is the reference's RealEpochs / AnalyticEpochs layout
``[n_signals, n_samples, n_trials]`` (C4 adds a leading band
axis).  For multi-trial configs the *memory* order is ``[trial, signal,
sample]`` (samples contiguous, the layout the kernels consume) and the
returned array is a strided view -- the binding accepts it without a copy.

All sizes can be scaled down (``n_signals=``, ``n_samples=``, ``n_trials=``)
with the same generative process, which is how the parity tests get
oracle-sized versions of each config.
"""
from __future__ import annotations

import numpy as np

try:
    import scipy.fft as _fft

    def _rfft(x, axis=-1):
        return _fft.rfft(x, axis=axis, workers=-1)

    def _irfft(X, n, axis=-1):
        return _fft.irfft(X, n=n, axis=axis, workers=-1)

    def _ifft(X, axis=-1):
        return _fft.ifft(X, axis=axis, workers=-1)
except Exception:  # pragma: no cover
    _rfft, _irfft, _ifft = np.fft.rfft, np.fft.irfft, np.fft.ifft

CONFIGS = {
    # name: (N, T, R, B, dtype, input_kind)
    "c1": (64, 2000, 1, 1, "f64", "real"),
    "c2": (1200, 10_000, 20, 1, "f32", "real"),
    "c3": (5000, 65_536, 1, 1, "f32", "real"),
    "c4": (2500, 4096, 60, 5, "f32", "real"),
    "c5": (20_000, 16_384, 1, 1, "c64", "analytic"),
}

DESCRIPTIONS = {
    "c1": "CPU-oracle smoke: 64 real f64 signals x 2000 samples @500 Hz, 1 trial, 10 Hz + noise",
    "c2": "volume conduction: 1200 alpha sources x 10000 @1kHz x 20 trials, leakage-mixed, trial-mean",
    "c3": "dense large-T: 5000 x 65536 f32 random-walk-phase 20 Hz carriers, 1 trial",
    "c4": "many-trial/band: 2500 x 4096 x 60 trials x 5 bands f32, 5% pairs coupled, trial-mean",
    "c5": "whole-brain: 20000 x 16384 complex64 analytic alpha noise, 0.5% pairs coupled, 1 trial",
}

C4_BANDS = ((4.0, 8.0), (8.0, 12.0), (12.0, 30.0), (30.0, 45.0), (55.0, 80.0))


def pair_samples(n_signals: int, n_samples: int, n_trials: int = 1, n_bands: int = 1) -> int:
    """The headline work unit: unique pairs N(N-1)/2 x T x R x B."""
    return n_signals * (n_signals - 1) // 2 * n_samples * n_trials * n_bands


def _bandlimit(white: np.ndarray, fs: float, lo: float, hi: float) -> np.ndarray:
    """Brick-wall band-pass along the last axis, then unit variance."""
    T = white.shape[-1]
    X = _rfft(white, axis=-1)
    f = np.arange(T // 2 + 1) * fs / T
    X[..., (f < lo) | (f > hi)] = 0.0
    y = _irfft(X, T, axis=-1)
    y /= np.maximum(y.std(axis=-1, keepdims=True), 1e-30)
    return y


def c1(n_signals: int = 64, n_samples: int = 2000, seed: int = 1) -> np.ndarray:
    """BASELINE configs[0] / SURVEY 8(d) C1 (decision D4 for the lags)."""
    rng = np.random.default_rng(seed)
    fs = 500.0
    t = np.arange(n_samples) / fs
    theta = rng.uniform(0.0, 2 * np.pi, size=n_signals)
    lags = np.array([0, 0, np.pi / 8, np.pi / 8, np.pi / 4, np.pi / 4, np.pi / 2, np.pi / 2])
    k = min(8, n_signals)
    theta[:k] = theta[0] + lags[:k]
    x = np.cos(2 * np.pi * 10.0 * t[None, :] + theta[:, None])
    x += rng.normal(0.0, 0.5, size=x.shape)
    return np.ascontiguousarray(x[:, :, None], dtype=np.float64)


def c2(n_signals: int = 1200, n_samples: int = 10_000, n_trials: int = 20,
       n_coupled: int = 100, seed: int = 2) -> np.ndarray:
    """BASELINE configs[1] / SURVEY 8(d) C2: lag-coupled alpha sources mixed by
    a Gaussian leakage matrix exp(-d^2 / 2 sigma^2), sigma = 0.1 x spread."""
    rng = np.random.default_rng(seed)
    fs = 1000.0
    N, T, R = n_signals, n_samples, n_trials
    s = _bandlimit(rng.standard_normal((R, N, T)), fs, 8.0, 12.0)
    n_pairs = min(n_coupled, N * (N - 1))
    pairs = set()
    while len(pairs) < n_pairs:
        i, j = rng.integers(0, N, size=2)
        if i != j:
            pairs.add((int(i), int(j)))
    pairs = sorted(pairs)
    lag = rng.integers(5, 31, size=len(pairs))           # ms == samples at 1 kHz
    w = 0.6
    for (i, j), L in zip(pairs, lag):
        s[:, j, :] = np.sqrt(1 - w * w) * s[:, j, :] + w * np.roll(s[:, i, :], int(L), axis=-1)
    pos = rng.uniform(0.0, 1.0, size=(N, 3))
    d2 = ((pos[:, None, :] - pos[None, :, :]) ** 2).sum(-1)
    sigma = 0.1
    Lmix = np.exp(-d2 / (2 * sigma * sigma))
    x = np.empty((R, N, T), dtype=np.float32)
    for r in range(R):
        x[r] = (Lmix @ s[r]).astype(np.float32)
    return np.transpose(x, (1, 2, 0))                    # [N, T, R] view


def c3(n_signals: int = 5000, n_samples: int = 65_536, seed: int = 3,
       block: int = 500) -> np.ndarray:
    """BASELINE configs[2] / SURVEY 8(d) C3 (decision D3: fs = 1000 Hz)."""
    rng = np.random.default_rng(seed)
    fs = 1000.0
    N, T = n_signals, n_samples
    out = np.empty((N, T), dtype=np.float32)
    tt = 2 * np.pi * 20.0 * np.arange(T) / fs
    for r0 in range(0, N, block):
        n = min(block, N - r0)
        phi0 = rng.uniform(0.0, 2 * np.pi, size=(n, 1))
        walk = np.cumsum(rng.normal(0.0, 0.05, size=(n, T)), axis=1)
        x = np.cos(tt[None, :] + phi0 + walk) + rng.standard_normal((n, T))
        out[r0:r0 + n] = x
    return out[:, :, None]


def c4(n_signals: int = 2500, n_samples: int = 4096, n_trials: int = 60,
       bands=C4_BANDS, n_latent: int = 20, seed: int = 4) -> np.ndarray:
    """BASELINE configs[3] / SURVEY 8(d) C4: per band, each signal bound to one
    of 20 latent band-limited sources (fixed binding and lag across trials,
    weight 0.6) => ~1/20 of pairs coupled.  Returns [B, N, T, R] (view of
    [B, R, N, T] memory)."""
    rng = np.random.default_rng(seed)
    fs = 1000.0
    B, N, T, R = len(bands), n_signals, n_samples, n_trials
    x = np.empty((B, R, N, T), dtype=np.float32)
    w = 0.6
    for b, (lo, hi) in enumerate(bands):
        bind = rng.integers(0, n_latent, size=N)
        lag = rng.integers(5, 31, size=N)
        for r in range(R):
            own = _bandlimit(rng.standard_normal((N, T)), fs, lo, hi)
            lat = _bandlimit(rng.standard_normal((n_latent, T)), fs, lo, hi)
            shifted = np.empty((N, T))
            for k in range(n_latent):
                idx = np.nonzero(bind == k)[0]
                for L in np.unique(lag[idx]):
                    sel = idx[lag[idx] == L]
                    shifted[sel] = np.roll(lat[k], int(L))
            x[b, r] = (np.sqrt(1 - w * w) * own + w * shifted).astype(np.float32)
    return np.transpose(x, (0, 2, 3, 1))                 # [B, N, T, R] view


def c5(n_signals: int = 20_000, n_samples: int = 16_384, n_latent: int = 200,
       seed: int = 5, block: int = 2000) -> np.ndarray:
    """BASELINE configs[4] / SURVEY 8(d) C5: complex64 analytic alpha noise
    (complex Gaussian on positive 8-12 Hz bins only -> ifft), each signal bound
    to one of 200 latents with a lag tau ~ U[5, 30] ms applied as
    exp(-i 2 pi f tau), weight 0.6 (=> ~0.5% of pairs share a latent)."""
    rng = np.random.default_rng(seed)
    fs = 1000.0
    N, T = n_signals, n_samples
    f = np.arange(T) * fs / T
    band = np.nonzero((f >= 8.0) & (f <= 12.0))[0]
    nb = band.size
    lat = (rng.standard_normal((n_latent, nb)) + 1j * rng.standard_normal((n_latent, nb)))
    bind = rng.integers(0, n_latent, size=N)
    tau = rng.uniform(0.005, 0.030, size=N)
    w = 0.6
    out = np.empty((N, T), dtype=np.complex64)
    fb = f[band]
    for r0 in range(0, N, block):
        n = min(block, N - r0)
        own = rng.standard_normal((n, nb)) + 1j * rng.standard_normal((n, nb))
        spec = np.sqrt(1 - w * w) * own + w * lat[bind[r0:r0 + n]] * np.exp(
            -2j * np.pi * fb[None, :] * tau[r0:r0 + n, None])
        X = np.zeros((n, T), dtype=np.complex128)
        X[:, band] = spec
        out[r0:r0 + n] = _ifft(X, axis=-1) * np.sqrt(T)
    return out[:, :, None]


def generate(name: str, **overrides) -> np.ndarray:
    """Dispatch by config name ('c1'..'c5')."""
    fn = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}[name]
    return fn(**overrides)
