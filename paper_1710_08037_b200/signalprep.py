"""signalprep -- analytic signal and unit phasors on the GPU.

Only the two operations on the PLV hot path are built:
  analytic_signal(x)               SPEC.md:76-84   Eq 3
  normalize_phasors(a, amp_floor)  SPEC.md:85-93   Eq 4
The FIR band-pass, two-pass filtering, downsampling and instantaneous_phase
 are upstream of / beside the path and out of scope for this
build (band-pass fusion is SURVEY 8(f) row 1).

Both run through libphasesync_cuda.so: cuFFT R2C -> one-sided Hilbert
multiplier -> C2R for H{x} (Re is copied from x bit-exactly),
then z = a/|a| with the amplitude-floor mask (exact per-row median only when
the row's min/max bound cannot rule masking out).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from ._arrays import describe, dtype_code


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


def analytic_signal(x) -> AnalyticEpochs:
    """a = x + i H{x}; Re(a) == x bit-exactly.

    Output dtype follows the input (float32 -> complex64, float64 ->
    complex128), shape [N, T, R] (a 2-D [N, T] input gives [N, T])."""
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
