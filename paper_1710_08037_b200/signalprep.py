"""signalprep -- band-pass, analytic signal and unit phasors on the GPU.

The operations on the PLV hot path and its band-pass front
end:
  design_bandpass_fir(band, order)   SPEC.md:58-66   (host: coefficient design)
  filter_two_pass(x, f, pad)         SPEC.md:67-75   zero-phase, reflection pad
  analytic_signal(x[, fir, pad])     SPEC.md:76-84   Eq 3
  normalize_phasors(a, amp_floor)    SPEC.md:85-93   Eq 4
Downsampling and instantaneous_phase stay out of scope
(they feed only the reference oracles).

All compute runs through libphasesync_cuda.so: cuFFT R2C -> one-sided Hilbert
multiplier -> C2R for H{x} (Re is copied from x bit-exactly),
then z = a/|a| with the amplitude-floor mask (exact per-row median only when
the row's min/max bound cannot rule masking out).  The two-pass FIR is
evaluated spectrally (DESIGN.md 8(f) #1).
"""
from __future__ import annotations

import ctypes
import math
import warnings
from dataclasses import dataclass

import numpy as np

from . import _native, errors
from ._arrays import describe, dtype_code


@dataclass(frozen=True)
class BandSpec:
    """SPEC.md band: edges in radians per sample, 0 < low < high < pi."""
    low: float
    high: float


@dataclass(frozen=True)
class FirFilter:
    """SPEC.md:58-66 FirFilter: linear-phase band-pass taps (order + 1)."""
    taps: np.ndarray
    band: BandSpec
    order: int


def design_bandpass_fir(band, order: int) -> FirFilter:
    """windowed-sinc band-pass, Hamming window (design decision
    SPEC.md:121), order + 1 taps, gain exactly 1 at the band centre.

    Host-side coefficient design (the reference designs on the CPU too; the
    taps then drive the GPU two-pass filter).  InvalidBandError for low >= high
    or edges outside (0, pi); OrderTooSmallWarning when order < 4 * 2pi /
    (high - low)."""
    b = band if isinstance(band, BandSpec) else BandSpec(float(band[0]), float(band[1]))
    if not (0.0 < b.low < b.high < math.pi):
        raise errors.InvalidBandError(f"band edges must satisfy 0 < low < high < pi, got {b}")
    order = int(order)
    if order <= 0 or order % 2:
        raise ValueError("order must be a positive even integer (SPEC.md:60)")
    if order < 4 * (2 * math.pi / (b.high - b.low)):
        warnings.warn(f"order {order} is small for transition width {b.high - b.low:.4g} rad/sample",
                      errors.OrderTooSmallWarning, stacklevel=2)
    m = np.arange(order + 1, dtype=np.float64) - order / 2.0
    h = np.empty(order + 1)
    nz = m != 0
    h[nz] = (np.sin(b.high * m[nz]) - np.sin(b.low * m[nz])) / (np.pi * m[nz])
    h[~nz] = (b.high - b.low) / np.pi
    h *= 0.54 - 0.46 * np.cos(2.0 * np.pi * np.arange(order + 1) / order)
    wc = 0.5 * (b.low + b.high)
    h /= abs(np.sum(h * np.exp(-1j * wc * np.arange(order + 1))))
    return FirFilter(taps=h, band=b, order=order)


def fir_struct(fir, pad_samples: int):
    """ps_fir for a FirFilter (or raw taps); keeps the taps array alive."""
    taps = np.ascontiguousarray(fir.taps if isinstance(fir, FirFilter) else fir, dtype=np.float64)
    s = _native.Fir()
    s.taps = taps.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    s.n_taps = taps.size
    s.pad_samples = int(pad_samples)
    return s, taps


@dataclass
class RealEpochs:
    """data [n_signals x n_samples x n_trials], fs optional."""
    data: object
    fs: float | None = None


@dataclass
class AnalyticEpochs:
    """SPEC.md:45-49."""
    data: object
    band: object = None


@dataclass
class PhasorEpochs:
    """unit phasors; masked entries exactly 0+0i."""
    data: object
    mask: object


def _unwrap(x):
    if isinstance(x, (RealEpochs, AnalyticEpochs, PhasorEpochs)):
        return x.data
    return x


def _to_device(x):
    """numpy -> CUDA torch tensor (device memory plumbing for the device entry points)."""
    import torch

    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            return x, False
        return x.cuda(), True
    return torch.from_numpy(np.asarray(x)).cuda(), True


def _args_for(d, kind: str) -> _native.PlvArgs:
    a = _native.PlvArgs()
    a.input = d.ptr
    a.dtype = dtype_code(d.dtype)
    a.input_kind = _native.INPUT_KINDS[kind]
    a.n_bands, a.n_signals, a.n_samples, a.n_trials = d.dims
    a.stride_band, a.stride_signal, a.stride_sample, a.stride_trial = d.strides
    a.amp_floor = 1e-6
    a.metrics = 1
    a.precision = 0
    a.trial_reduce = 0
    a.shard_index, a.shard_count = 0, 1
    return a


def filter_two_pass(x, f, pad_samples: int):
    """zero-phase two-pass FIR (forward, reverse, forward,
    reverse; zero initial state) of real epochs with reflection padding of
    pad_samples per side, trimmed back to the input shape.
    SignalTooShortError if n_samples <= order + 1.  Returns an array of the
    input's type and dtype, shape [N, T, R] (2-D input gives [N, T])."""
    import torch

    src = _unwrap(x)
    host = not (isinstance(src, torch.Tensor) and src.is_cuda)
    t, _ = _to_device(src)
    d = describe(t)
    if d.dtype not in ("f32", "f64"):
        raise ValueError("filter_two_pass expects a real-valued input (SPEC.md:67)")
    B, N, T, R = d.dims
    out = torch.empty((R, N, T), dtype=t.dtype, device=t.device)
    a = _args_for(d, "real")
    fs, keep = fir_struct(f, pad_samples)
    a.fir = ctypes.pointer(fs)
    with torch.cuda.device(t.device):
        a.stream = torch.cuda.current_stream(t.device).cuda_stream
        ctx = _native.context(t.device.index)
        _native.check(_native.lib().ps_filter_two_pass(ctx.handle, ctypes.byref(a), out.data_ptr()))
    del keep
    res = out.permute(1, 2, 0)
    if np.ndim(src) == 2 or (isinstance(src, torch.Tensor) and src.dim() == 2):
        res = res[:, :, 0]
    if host:
        res = res.cpu().numpy()
    return RealEpochs(data=res) if isinstance(x, RealEpochs) else res


def analytic_signal(x, fir=None, pad_samples: int = 0) -> AnalyticEpochs:
    """a = x + i H{x}; Re(a) == x bit-exactly.

    With `fir` (a FirFilter or taps) the band-pass front end runs first: the
    two-pass filter on the reflection-padded record, the analytic signal of
    the padded record, then the trim ("prior to the removal of the
    padding").  Output dtype follows the input (float32 -> complex64, float64
    -> complex128), shape [N, T, R] (a 2-D [N, T] input gives [N, T])."""
    import torch

    src = _unwrap(x)
    host = not (isinstance(src, torch.Tensor) and src.is_cuda)
    t, _ = _to_device(src)
    d = describe(t)
    if d.dtype not in ("f32", "f64"):
        raise ValueError("analytic_signal expects a real-valued input (SPEC.md:76)")
    B, N, T, R = d.dims
    cdt = torch.complex64 if d.dtype == "f32" else torch.complex128
    out = torch.empty((R, N, T), dtype=cdt, device=t.device)
    a = _args_for(d, "real")
    keep = None
    if fir is not None:
        fs, keep = fir_struct(fir, pad_samples)
        a.fir = ctypes.pointer(fs)
    with torch.cuda.device(t.device):
        a.stream = torch.cuda.current_stream(t.device).cuda_stream
        ctx = _native.context(t.device.index)
        _native.check(_native.lib().ps_analytic_signal(ctx.handle, ctypes.byref(a), out.data_ptr()))
    res = out.permute(1, 2, 0)
    if np.ndim(src) == 2 or (isinstance(src, torch.Tensor) and src.dim() == 2):
        res = res[:, :, 0]
    if host:
        res = res.cpu().numpy()
    return AnalyticEpochs(data=res)


def normalize_phasors(a, amp_floor: float = 1e-6) -> PhasorEpochs:
    """z = a/|a|; samples with |a| < amp_floor * median_row(|a|)
    (or |a| == 0) are masked and set to 0+0i; AllSamplesMaskedError if a whole
    signal/trial is masked.  Real input is first turned into its analytic
    signal.  Returns PhasorEpochs(data, mask)."""
    import torch

    src = _unwrap(a)
    host = not (isinstance(src, torch.Tensor) and src.is_cuda)
    t, _ = _to_device(src)
    d = describe(t)
    kind = "real" if d.dtype in ("f32", "f64") else "analytic"
    B, N, T, R = d.dims
    cdt = torch.complex64 if d.dtype in ("f32", "c64") else torch.complex128
    out = torch.empty((R, N, T), dtype=cdt, device=t.device)
    mask = torch.empty((R, N, T), dtype=torch.uint8, device=t.device)
    args = _args_for(d, kind)
    args.amp_floor = float(amp_floor)
    with torch.cuda.device(t.device):
        args.stream = torch.cuda.current_stream(t.device).cuda_stream
        ctx = _native.context(t.device.index)
        _native.check(_native.lib().ps_normalize_phasors(ctx.handle, ctypes.byref(args), out.data_ptr(),
                                                         mask.data_ptr()))
    z = out.permute(1, 2, 0)
    m = mask.permute(1, 2, 0).bool()
    if np.ndim(src) == 2 or (isinstance(src, torch.Tensor) and src.dim() == 2):
        z, m = z[:, :, 0], m[:, :, 0]
    if host:
        z, m = z.cpu().numpy(), m.cpu().numpy()
    return PhasorEpochs(data=z, mask=m)


def instantaneous_phase(a):
    """the angle of every complex sample, in (-pi, pi]; the
    phase of 0 is defined as 0.  Elementwise on the input's own
    device (torch for CUDA tensors, numpy for host arrays); accepts
    AnalyticEpochs / PhasorEpochs or a complex array of any shape."""
    import torch

    src = _unwrap(a)
    if isinstance(src, torch.Tensor):
        ph = torch.angle(src)
        return torch.where(ph == -math.pi, torch.full_like(ph, math.pi), ph)
    ph = np.angle(np.asarray(src))
    return np.where(ph == -np.pi, np.pi, ph)


def downsample(x, factor: int, alias_tol: float = 0.01):
    """keep every factor-th sample (axis 1 of [N, T(, R)]);
    RealEpochs.fs is divided by factor.  FactorTooLargeError when fewer than 2
    samples would remain.  The caller guarantees band limitation below
    pi / factor; an AliasingWarning is raised when more than `alias_tol` of the
    (mean-removed) periodogram power lies above it."""
    import torch

    factor = int(factor)
    if factor < 1:
        raise ValueError("factor must be a positive integer")
    src = _unwrap(x)
    T = int(src.shape[1])
    n_out = (T + factor - 1) // factor
    if n_out < 2:
        raise errors.FactorTooLargeError(f"downsampling {T} samples by {factor} leaves {n_out} < 2")
    if factor > 1:
        t = src if isinstance(src, torch.Tensor) else torch.from_numpy(np.asarray(src))
        v = t.movedim(1, -1).to(torch.float64)
        p = torch.fft.rfft(v - v.mean(dim=-1, keepdim=True), dim=-1).abs().square().sum(
            dim=tuple(range(v.dim() - 1)))
        k_cut = T / (2.0 * factor)  # bin of pi / factor rad/sample
        tot = float(p.sum())
        if tot > 0.0 and float(p[int(math.floor(k_cut)) + 1:].sum()) > alias_tol * tot:
            warnings.warn(f"signal has power above pi/{factor} rad/sample: downsampling aliases it",
                          errors.AliasingWarning, stacklevel=2)
    res = src[:, ::factor]
    if isinstance(x, RealEpochs):
        return RealEpochs(data=res, fs=None if x.fs is None else x.fs / factor)
    return res
