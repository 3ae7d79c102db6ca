"""CPU oracle for the PLV / iPLV / ciPLV hot path -- TEST INFRASTRUCTURE ONLY.

This module is the *checker*.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may import
it.  The product path (``paper_1710_08037_b200``) never calls into it; the
product fails loudly when its CUDA library is missing.

What it restates
----------------
The reference (``/root/reference``) ships no implementation code: its
behavioural contract is ``SPEC.md`` + the paper's Eqs 1-16 + the three Matlab
implementations in the paper's Appendix + ``pkg/src/phasesync/errors.py``.
Each function below cites the SPEC / PAPER lines it follows.

Third-party arithmetic the reference declares (``pkg/pyproject.toml:10-13``):
numpy>=1.24 (complex matmul -> BLAS zgemm) and scipy>=1.10 (FFT).  Neither is
vendored by the reference; this oracle uses the numpy/scipy installed here
(numpy 2.3, scipy 1.18) and restates the published algorithms directly.

Parity pinning -- parity unpinned by reference tests
----------------------------------------------------
There are no reference tests, fixtures or golden vectors to pin against
(``pkg/pyproject.toml:25`` names an absent ``tests/``) and no reference code to
run, so parity against reference *code* is unpinned.  The oracle is pinned
against every closed-form known-answer example and invariant the SPEC states
for this path (see ``tests/test_oracle_kats.py``) and against
``scipy.signal.hilbert`` for the analytic signal.
"""
from __future__ import annotations

import numpy as np

try:  # threaded FFT for the CPU-baseline timing; numpy fallback is equivalent
    import scipy.fft as _fft

    def _rfft(x, axis):
        return _fft.rfft(x, axis=axis, workers=-1)

    def _irfft(X, n, axis):
        return _fft.irfft(X, n=n, axis=axis, workers=-1)

except Exception:  # pragma: no cover
    def _rfft(x, axis):
        return np.fft.rfft(x, axis=axis)

    def _irfft(X, n, axis):
        return np.fft.irfft(X, n=n, axis=axis)


class OracleError(ValueError):
    """Base for the oracle's own error signalling (mirrors errors.py names)."""


class AllSamplesMaskedError(OracleError):
    """errors.py:12 -- every sample of some signal/trial fell below the floor."""


class EmptyEffectiveWindowError(OracleError):
    """errors.py:20 -- all samples are masked for at least one signal pair."""


CIPLV_SINGULAR_EPS = 1e-12
DEFAULT_AMP_FLOOR = 1e-6
ROW_BLOCK = 256


# --------------------------------------------------------------------------
# signalprep
# --------------------------------------------------------------------------
def hilbert_weights_half(n_samples: int) -> np.ndarray:
    """Multiplier on the one-sided (rfft) spectrum that yields H{x}.

    SPEC.md:79,124: DC and Nyquist kept at unit weight, strictly positive bins
    doubled, strictly negative bins zeroed.  The analytic signal is then
    a = x + i*H{x}, so H{x} = irfft(-i * sgn(k) * X_k): DC/Nyquist get 0,
    strictly positive bins get -i (odd T has no Nyquist bin, matching
    scipy.signal.hilbert's ``h[1:(N+1)//2] = 2``).
    """
    T = int(n_samples)
    w = np.zeros(T // 2 + 1, dtype=np.complex128)
    if T % 2 == 0:
        w[1:T // 2] = -1j
    else:
        w[1:(T + 1) // 2] = -1j
    return w


def analytic_signal(x, axis: int = 1) -> np.ndarray:
    """SPEC.md:76-84 (Eq 3): a = x + i*H{x}, Re(a) == x bit-exactly.

    ``x`` is RealEpochs-shaped ``[n_signals, n_samples, n_trials]`` (or any
    array with samples on ``axis``); computed in float64.  The
    real part is copied from x -- only the imaginary part
    comes from the inverse FFT.
    """
    x = np.asarray(x, dtype=np.float64)
    if x.shape[axis] < 2:
        raise ValueError("n_samples must be >= 2 (SPEC.md:31)")
    T = x.shape[axis]
    X = _rfft(x, axis)
    shape = [1] * x.ndim
    shape[axis] = T // 2 + 1
    H = _irfft(X * hilbert_weights_half(T).reshape(shape), T, axis)
    a = np.empty(x.shape, dtype=np.complex128)
    a.real = x
    a.imag = H
    return a


def normalize_phasors(a, amp_floor: float = DEFAULT_AMP_FLOOR, axis: int = 1):
    """SPEC.md:85-93 (Eq 4): z = a/|a| with the amplitude guard.

    Masked where |a| < amp_floor * median_row(|a|) (median per
    signal/trial along the sample axis, numpy semantics: mean of the two middle
    values for even T) or where |a| == 0.  Masked samples are
    exactly 0+0i.  Raises AllSamplesMaskedError if a whole
    signal/trial row is masked (errors.py:12).
    Returns (z, mask).
    """
    a = np.asarray(a)
    a = a.astype(np.complex128, copy=False)
    amp = np.abs(a)
    med = np.median(amp, axis=axis, keepdims=True)
    mask = (amp < amp_floor * med) | (amp == 0.0)
    if np.any(np.all(mask, axis=axis)):
        raise AllSamplesMaskedError("an entire signal/trial is below the amplitude floor")
    safe = np.where(mask, 1.0, amp)
    z = np.where(mask, 0.0 + 0.0j, a / safe)
    return z, mask


# --------------------------------------------------------------------------
# band-pass front end (design decisions :121-122)
# --------------------------------------------------------------------------
class InvalidBandError(OracleError):
    """errors.py InvalidBandError -- low >= high or edges outside (0, pi)."""


class SignalTooShortError(OracleError):
    """errors.py SignalTooShortError -- n_samples <= order + 1."""


def design_bandpass_fir(low: float, high: float, order: int) -> np.ndarray:
    """SPEC.md:58-66 design_bandpass_fir, with the SPEC's design decision
    (SPEC.md:121): windowed sinc with a Hamming window, order + 1 taps,
    linear phase (symmetric).  Band edges in radians per sample.  The SPEC
    asks for pass-band gain within +-1 dB of unity at the band centre; this
    restatement scales the taps so the gain there is exactly 1 (the one
    free normalisation choice; DESIGN.md section 8(f) #1).
    """
    if not (0.0 < low < high < np.pi):
        raise InvalidBandError("band edges must satisfy 0 < low < high < pi")
    if order <= 0 or order % 2:
        raise ValueError("order must be a positive even integer")
    M = int(order)
    m = np.arange(M + 1, dtype=np.float64) - M / 2.0
    h = np.empty(M + 1)
    nz = m != 0
    h[nz] = (np.sin(high * m[nz]) - np.sin(low * m[nz])) / (np.pi * m[nz])
    h[~nz] = (high - low) / np.pi
    h *= 0.54 - 0.46 * np.cos(2.0 * np.pi * np.arange(M + 1) / M)
    wc = 0.5 * (low + high)
    g = abs(np.sum(h * np.exp(-1j * wc * np.arange(M + 1))))
    return h / g


def reflect_pad(x, pad: int, axis: int = 1) -> np.ndarray:
    """reflection padding of `pad` samples on each side
    (numpy 'reflect': the edge sample is not repeated).  pad < n_samples."""
    x = np.asarray(x, dtype=np.float64)
    if pad >= x.shape[axis]:
        raise SignalTooShortError("reflection padding needs pad < n_samples")
    widths = [(0, 0)] * x.ndim
    widths[axis] = (pad, pad)
    return np.pad(x, widths, mode="reflect")


def _fir_causal(x, taps, axis):
    """Causal FIR with zero initial state: y[n] = sum_k h[k] x[n-k], len(y) = len(x)."""
    xm = np.moveaxis(x, axis, -1)
    L = xm.shape[-1]
    flat = xm.reshape(-1, L)
    out = np.empty_like(flat)
    for r in range(flat.shape[0]):
        out[r] = np.convolve(flat[r], taps)[:L]
    return np.moveaxis(out.reshape(xm.shape), -1, axis)


def two_pass_padded(x, taps, pad: int, axis: int = 1) -> np.ndarray:
    """SPEC.md:67-75 filter_two_pass on the reflection-padded record, padding
    kept: forward pass, reverse, second pass, reverse (zero phase, |H|^2)."""
    taps = np.asarray(taps, dtype=np.float64)
    T = np.asarray(x).shape[axis]
    if T <= taps.size:  # n_samples <= order + 1
        raise SignalTooShortError("n_samples must exceed order + 1")
    xp = reflect_pad(x, pad, axis)
    y = _fir_causal(xp, taps, axis)
    y = np.flip(_fir_causal(np.flip(y, axis), taps, axis), axis)
    return y


def _trim(y, pad, T, axis):
    sl = [slice(None)] * y.ndim
    sl[axis] = slice(pad, pad + T)
    return y[tuple(sl)]


def filter_two_pass(x, taps, pad: int, axis: int = 1) -> np.ndarray:
    """zero-phase two-pass FIR with reflection padding
    (SPEC.md:122), output trimmed back to the input's shape."""
    T = np.asarray(x).shape[axis]
    return np.ascontiguousarray(_trim(two_pass_padded(x, taps, pad, axis), pad, T, axis))


def bandpass_analytic(x, taps, pad: int, axis: int = 1) -> np.ndarray:
    """The real-input front end of cmd_connectivity: band-pass
    (two-pass, reflection padded) -> analytic signal of the PADDED record ->
    trim ("the analytical signal was calculated prior to the removal of the
    padding")."""
    T = np.asarray(x).shape[axis]
    a = analytic_signal(two_pass_padded(x, taps, pad, axis), axis)
    return np.ascontiguousarray(_trim(a, pad, T, axis))


# --------------------------------------------------------------------------
# Welch coherence family (Eq 12)
# --------------------------------------------------------------------------
class WindowTooLongError(OracleError):
    """errors.py WindowTooLongError -- window_len > n_samples."""


class EmptyBandError(OracleError):
    """errors.py EmptyBandError -- no spectral bin inside the band."""


def welch_spectra(x, window_len: int, overlap: int) -> np.ndarray:
    """Spectra of Hamming-tapered segments (symmetric window)
    of x [N, T, R]: segments of window_len samples advancing by
    window_len - overlap, drawn within each trial and pooled over trials
    (SPEC.md:262).  Returns X [N, R * S, window_len // 2 + 1], q = r * S + s."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 2:
        x = x[:, :, None]
    N, T, R = x.shape
    W, O = int(window_len), int(overlap)
    if not (0 <= O < W):
        raise ValueError("WelchConfig needs 0 <= overlap < window_len (SPEC.md:168)")
    if W > T:
        raise WindowTooLongError("window_len exceeds n_samples (SPEC.md:225)")
    hop = W - O
    S = (T - W) // hop + 1
    win = np.hamming(W)
    seg = np.stack([x[:, s * hop:s * hop + W, :] for s in range(S)], axis=1)  # [N, S, W, R]
    seg = np.transpose(seg, (0, 3, 1, 2)) * win                              # [N, R, S, W]
    return np.fft.rfft(seg, axis=-1).reshape(N, R * S, W // 2 + 1)


def _norm_cross(Xi, Xj):
    """Normalised cross-spectrum over segments (axis 0), 0 where a power is 0."""
    s = np.sum(Xi * np.conj(Xj), axis=0)
    p = np.sqrt(np.sum(np.abs(Xi) ** 2, axis=0) * np.sum(np.abs(Xj) ** 2, axis=0))
    return np.where(p > 0, s / np.where(p > 0, p, 1.0), 0.0)


def coherence_welch(x2, window_len: int, overlap: int) -> np.ndarray:
    """|sum X_i X_j^*| / sqrt(sum|X_i|^2 sum|X_j|^2) per bin
    (magnitude, not squared) for two signals x2 [2, T(, R)]."""
    X = welch_spectra(x2, window_len, overlap)
    return np.abs(_norm_cross(X[0], X[1]))


def coherence_weighted_phasor(x2, window_len: int, overlap: int) -> np.ndarray:
    """SPEC.md:221-228, Eq 12 second line: amplitude-weighted average of the
    per-segment unit cross-phasors, normalised by the amplitude root-product."""
    X = welch_spectra(x2, window_len, overlap)
    Ai, Aj = np.abs(X[0]), np.abs(X[1])
    dphi = np.angle(X[0]) - np.angle(X[1])
    num = np.abs(np.sum(Ai * Aj * np.exp(1j * dphi), axis=0))
    den = np.sqrt(np.sum(Ai ** 2, axis=0) * np.sum(Aj ** 2, axis=0))
    return np.where(den > 0, num / np.where(den > 0, den, 1.0), 0.0)


def imaginary_coherency(x2, window_len: int, overlap: int) -> np.ndarray:
    """|Im| of the normalised cross-spectrum per bin."""
    X = welch_spectra(x2, window_len, overlap)
    return np.abs(_norm_cross(X[0], X[1]).imag)


def welch_bins(window_len: int, low: float, high: float):
    """(first bin, n bins) with low <= 2 pi k / window_len <= high."""
    W = int(window_len)
    ks = [k for k in range(W // 2 + 1) if low <= 2 * np.pi * k / W <= high]
    return (ks[0], len(ks)) if ks else (0, 0)


def band_coherence(spec, window_len: int, low: float, high: float, mode: str = "max") -> float:
    """max or mean over the band's bins; EmptyBand if none."""
    k0, nb = welch_bins(window_len, low, high)
    if nb == 0:
        raise EmptyBandError("band contains no spectral bin (SPEC.md:239)")
    v = np.asarray(spec)[k0:k0 + nb]
    return float(v.max() if mode == "max" else v.mean())


def coherence_matrix(x, window_len: int, overlap: int, low: float, high: float, mode: str = "max"):
    """All-pairs band coherence (the N x N form of band_coherence(coherence_welch)):
    per bin, the normalised cross-spectrum over pooled segments as one complex
    Gram; returns {'coh', 'icoh', 'cre', 'cim'} as [N, N] (mode max / mean) or
    [N, N, n_bins] (mode none).  Diagonal: coh = cre = 1, icoh = cim = 0."""
    X = welch_spectra(x, window_len, overlap)
    k0, nb = welch_bins(window_len, low, high)
    if nb == 0:
        raise EmptyBandError("band contains no spectral bin (SPEC.md:239)")
    N = X.shape[0]
    per = {m: [] for m in ("coh", "icoh", "cre", "cim")}
    for k in range(k0, k0 + nb):
        Z = X[:, :, k]
        S = Z @ Z.conj().T
        p = np.sqrt(np.real(np.diag(S)))
        d = np.outer(p, p)
        C = np.where(d > 0, S / np.where(d > 0, d, 1.0), 0.0)
        for m, v in (("coh", np.abs(C)), ("icoh", np.abs(C.imag)), ("cre", C.real.copy()), ("cim", C.imag.copy())):
            np.fill_diagonal(v, 1.0 if m in ("coh", "cre") else 0.0)
            per[m].append(v)
    out = {}
    for m, vs in per.items():
        a = np.stack(vs, axis=-1)
        out[m] = a.max(axis=-1) if mode == "max" else (a.mean(axis=-1) if mode == "mean" else a)
    return out


def phasors_from_unit(z, axis: int = 1):
    """PhasorEpochs given directly (plv_matrix input): mask = (z == 0)."""
    z = np.asarray(z).astype(np.complex128, copy=False)
    mask = (z == 0)
    if np.any(np.all(mask, axis=axis)):
        raise AllSamplesMaskedError("an entire signal/trial is masked")
    return z, mask


def instantaneous_phase(a) -> np.ndarray:
    """angle in (-pi, pi]; phase of 0 is 0."""
    ph = np.angle(np.asarray(a))
    ph = np.where(ph == -np.pi, np.pi, ph)
    return ph


# --------------------------------------------------------------------------
# connectivity
# --------------------------------------------------------------------------
def _gram_blocked(zt: np.ndarray) -> np.ndarray:
    """G = Z Z^H for one trial [N, T] in row blocks of 256,
    complex128 accumulation; PAPER.md:286 (impl 3)."""
    N = zt.shape[0]
    G = np.empty((N, N), dtype=np.complex128)
    zh = zt.conj().T
    for r0 in range(0, N, ROW_BLOCK):
        G[r0:r0 + ROW_BLOCK] = zt[r0:r0 + ROW_BLOCK] @ zh
    return G


def _metrics_from_gram(G: np.ndarray, C: np.ndarray):
    """Eq 7 / Eq 13 / Eq 14 epilogue with the SPEC's
    design decisions: |Im| for iPLV, ciPLV singularity rule
    (SPEC.md:259), per-pair effective T, diagonal rules
    (SPEC.md:151,194)."""
    if np.any(C <= 0):
        raise EmptyEffectiveWindowError("all samples masked for some pair")
    re = G.real / C
    im = G.imag / C
    plv = np.abs(G) / C
    iplv = np.abs(im)
    den = 1.0 - re * re
    sing = np.abs(re) >= 1.0 - CIPLV_SINGULAR_EPS
    ciplv = np.where(sing, 0.0, np.abs(im) / np.sqrt(np.where(sing, 1.0, den)))
    # |Im|^2 <= 1 - Re^2 (Cauchy-Schwarz): rounding near the singularity can
    # push the quotient past 1; keep the output bound [0, 1]
    ciplv = np.minimum(ciplv, 1.0)
    n = G.shape[0]
    d = np.arange(n)
    plv[d, d] = 1.0
    iplv[d, d] = 0.0
    ciplv[d, d] = 0.0
    return plv, iplv, ciplv


def plv_family_from_phasors(z, mask, trial_reduce: str = "mean", raw: bool = False):
    """All three metrics from one Gram per trial.

    z, mask: [N, T, R].  trial_reduce:
      'none' -> per-trial matrices [N, N, R] (the Appendix's plv(:,:,t));
      'mean' -> mean over trials of the per-trial metrics [N, N] (default);
      'pool' -> one Gram over all R*T observations [N, N].
    Returns dict(plv=..., iplv=..., ciplv=..., n_observations=...).
    With raw=True also returns the per-trial normalized complex Gram
    ('cgram', [N, N, R]) used by the tests to separate Gram error from
    epilogue conditioning.
    """
    z = np.asarray(z)
    N, T, R = z.shape
    any_mask = bool(np.any(mask))
    if trial_reduce == "pool":
        zz = np.transpose(z, (0, 2, 1)).reshape(N, R * T)
        G = _gram_blocked(zz)
        if any_mask:
            u = (~np.transpose(mask, (0, 2, 1)).reshape(N, R * T)).astype(np.float64)
            C = u @ u.T
        else:
            C = np.full((N, N), float(R * T))
        p, i, c = _metrics_from_gram(G, C)
        out = dict(plv=p, iplv=i, ciplv=c, n_observations=R * T)
        if raw:
            out["cgram"] = (G / C)[:, :, None]
        return out
    per = []
    cg = []
    for t in range(R):
        zt = np.ascontiguousarray(z[:, :, t])
        G = _gram_blocked(zt)
        if any_mask:
            u = (~mask[:, :, t]).astype(np.float64)
            C = u @ u.T
        else:
            C = np.full((N, N), float(T))
        per.append(_metrics_from_gram(G, C))
        if raw:
            cg.append(G / C)
    if trial_reduce == "none":
        out = dict(plv=np.stack([p[0] for p in per], axis=2),
                   iplv=np.stack([p[1] for p in per], axis=2),
                   ciplv=np.stack([p[2] for p in per], axis=2),
                   n_observations=T)
    elif trial_reduce == "mean":
        out = dict(plv=np.mean([p[0] for p in per], axis=0),
                   iplv=np.mean([p[1] for p in per], axis=0),
                   ciplv=np.mean([p[2] for p in per], axis=0),
                   n_observations=T)
    else:
        raise ValueError(f"unknown trial_reduce {trial_reduce!r}")
    if raw:
        out["cgram"] = np.stack(cg, axis=2)
    return out


def plv_family(x, input_kind: str = "real", amp_floor: float = DEFAULT_AMP_FLOOR,
               trial_reduce: str = "mean", raw: bool = False, fir=None):
    """The whole hot path: [band-pass ->] [analytic ->] normalise -> Gram ->
    PLV/iPLV/ciPLV.

    x: [N, T, R] (a 2-D [N, T] array is treated as one trial).
    input_kind: 'real', 'analytic' or 'phasor'
    (SPEC.md:186).  fir: optional (taps, pad_samples) for real input -> the
    band-pass front end bandpass_analytic.
    """
    x = np.asarray(x)
    if x.ndim == 2:
        x = x[:, :, None]
    if input_kind == "real" and fir is not None:
        z, mask = normalize_phasors(bandpass_analytic(x, fir[0], int(fir[1])), amp_floor)
    elif input_kind == "real":
        z, mask = normalize_phasors(analytic_signal(x), amp_floor)
    elif input_kind == "analytic":
        z, mask = normalize_phasors(x, amp_floor)
    elif input_kind == "phasor":
        z, mask = phasors_from_unit(x)
    else:
        raise ValueError(f"unknown input_kind {input_kind!r}")
    return plv_family_from_phasors(z, mask, trial_reduce, raw=raw)


def _metrics_from_block(G: np.ndarray, C: np.ndarray, rows: np.ndarray, c0: int):
    """_metrics_from_gram for the block rows x cols [c0, c0 + G.shape[1]):
    same epilogue, diagonal rules where the
    global column equals the row."""
    if np.any(C <= 0):
        raise EmptyEffectiveWindowError("all samples masked for some pair")
    re = G.real / C
    im = G.imag / C
    plv = np.abs(G) / C
    iplv = np.abs(im)
    den = 1.0 - re * re
    sing = np.abs(re) >= 1.0 - CIPLV_SINGULAR_EPS
    ciplv = np.minimum(np.where(sing, 0.0, np.abs(im) / np.sqrt(np.where(sing, 1.0, den))), 1.0)
    r = np.nonzero((rows >= c0) & (rows < c0 + G.shape[1]))[0]
    plv[r, rows[r] - c0] = 1.0
    iplv[r, rows[r] - c0] = 0.0
    ciplv[r, rows[r] - c0] = 0.0
    return plv, iplv, ciplv


def plv_family_rows(x, rows, input_kind: str = "real", amp_floor: float = DEFAULT_AMP_FLOOR,
                    trial_reduce: str = "mean", col_block: int | None = None):
    """Rows ``rows`` (all columns) of the plv_family matrices -- the oracle at
    full config size for a row subset: every signal is normalised (row-local
    work: analytic signal, median floor) in column blocks of
    ``col_block`` signals, and G[rows, block] = z_rows z_block^H per trial in
    complex128.  x: [N, T, R].  trial_reduce
    'mean' (default) or 'none' ([len(rows), N, R]).  Returns dict of
    [len(rows), N] float64 arrays."""
    x = np.asarray(x)
    if x.ndim == 2:
        x = x[:, :, None]
    N, T, R = x.shape
    rows = np.asarray(rows, dtype=np.int64)
    if col_block is None:  # ~1 GB of complex128 phasors per column block
        col_block = max(64, (1 << 26) // (T * R))

    def prep(sel):
        xs = x[sel]
        if input_kind == "real":
            return normalize_phasors(analytic_signal(xs), amp_floor)
        if input_kind == "analytic":
            return normalize_phasors(xs, amp_floor)
        return phasors_from_unit(xs)

    zr, mr = prep(rows)
    acc = {k: np.zeros((len(rows), N, R if trial_reduce == "none" else 1)) for k in ("plv", "iplv", "ciplv")}
    for c0 in range(0, N, col_block):
        c1 = min(N, c0 + col_block)
        zc, mc = prep(slice(c0, c1))
        for t in range(R):
            G = np.ascontiguousarray(zr[:, :, t]) @ np.ascontiguousarray(zc[:, :, t]).conj().T
            if np.any(mr[:, :, t]) or np.any(mc[:, :, t]):
                C = (~mr[:, :, t]).astype(np.float64) @ (~mc[:, :, t]).astype(np.float64).T
            else:
                C = np.full(G.shape, float(T))
            p, i, c = _metrics_from_block(G, C, rows, c0)
            k = t if trial_reduce == "none" else 0
            acc["plv"][:, c0:c1, k] += p
            acc["iplv"][:, c0:c1, k] += i
            acc["ciplv"][:, c0:c1, k] += c
    if trial_reduce == "none":
        return acc
    return {k: v[:, :, 0] / R for k, v in acc.items()}


def plv_matrix(phasors, mode: str = "over_samples", trial_reduce: str = "mean"):
    """(1/T)|z_i . z_j^H| via one complex product per trial
    (mode 'over_samples', Eq 7) or per sample over trials (mode 'over_trials',
    Eq 8 -> [N, N, T])."""
    z, mask = phasors_from_unit(phasors)
    if mode == "over_samples":
        return plv_family_from_phasors(z, mask, trial_reduce)["plv"]
    if mode == "over_trials":
        return plv_over_trials(z, mask)
    raise ValueError(mode)


def plv_over_trials(z, mask):
    """Eq 8: per sample t, Gram over trials.
    Returns PLV [N, N, T]."""
    return plv_family_over_trials(z, mask)["plv"]


def plv_family_over_trials(z, mask):
    """Time-resolved PLV / iPLV / ciPLV (Eq 8 with the Eq 13/14 epilogues; the
    trial-axis variant SPEC.md:277 makes available): per sample t the Gram is
    taken over trials and the per-pair count is the number of trials unmasked
    in both signals.  Returns dict of [N, N, T] arrays."""
    z = np.asarray(z)
    N, T, R = z.shape
    outs = {k: np.empty((N, N, T)) for k in ("plv", "iplv", "ciplv")}
    u = (~mask).astype(np.float64)
    for t in range(T):
        zt = z[:, t, :]
        G = zt @ zt.conj().T
        C = u[:, t, :] @ u[:, t, :].T
        p, i, c = _metrics_from_gram(G, C)
        outs["plv"][:, :, t] = p
        outs["iplv"][:, :, t] = i
        outs["ciplv"][:, :, t] = c
    return outs


# --------------------------------------------------------------------------
# Phase-angle implementations: the
# oracle's own oracle.  Small shapes only (pure-Python pair loop).
# --------------------------------------------------------------------------
def plv_reference(phases, mode: str = "over_samples") -> np.ndarray:
    """Appendix impl 1: two nested loops over pairs.

    phases: [N, T, R] in (-pi, pi].  Returns [N, N, R] (over_samples) with the
    symmetric part and diagonal filled per ConnectivityMatrix
    -- the Matlab code fills only c2 > c1.
    """
    ph = np.asarray(phases, dtype=np.float64)
    N, T, R = ph.shape
    if mode != "over_samples":
        raise ValueError(mode)
    plv = np.zeros((N, N, R))
    for t in range(R):
        for c1 in range(N):
            plv[c1, c1, t] = 1.0
            for c2 in range(c1 + 1, N):
                d = ph[c1, :, t] - ph[c2, :, t]
                v = abs(np.mean(np.exp(1j * d)))
                plv[c1, c2, t] = v
                plv[c2, c1, t] = v
    return plv


def plv_vectorized(phases, mode: str = "over_samples") -> np.ndarray:
    """Appendix impl 2: all pairs at once, loop over samples."""
    ph = np.asarray(phases, dtype=np.float64)
    N, T, R = ph.shape
    if mode != "over_samples":
        raise ValueError(mode)
    plv = np.zeros((N, N, R))
    for t in range(R):
        acc = np.zeros((N, N), dtype=np.complex128)
        for s in range(T):
            p = ph[:, s, t]
            acc += np.exp(1j * (p[:, None] - p[None, :]))
        plv[:, :, t] = np.abs(acc / T)
        np.fill_diagonal(plv[:, :, t], 1.0)
    return plv


def make_surrogate(n_signals: int, n_samples: int, n_trials: int, seed: int) -> np.ndarray:
    """seeded uniform phases -> unit phasors [N, T, R]."""
    rng = np.random.default_rng(seed)
    ph = rng.uniform(-np.pi, np.pi, size=(n_signals, n_samples, n_trials))
    return np.exp(1j * ph)
