"""connectivity -- PLV / iPLV / ciPLV on the sm_100a path.

Mirrors the reference module's operations and types:
  plv_matrix(phasors, mode)  SPEC.md:186-194   Eq 7 / Appendix impl 3
  iplv(phasors)              SPEC.md:195-203   Eq 13
  ciplv(phasors)             SPEC.md:204-212   Eq 14
  ConnectivityMatrix
plus ``plv_family``, the fused entry point the B200 build is designed around:
one call runs [Hilbert ->] normalise -> Gram -> all requested metrics from a
single Gram per trial (north star (1)-(3)).

Every call goes through libphasesync_cuda.so (``_native``); there is no CPU
fallback.  numpy inputs take the host entry point (copies to/from the GPU
inside the call, results returned as numpy); CUDA torch tensors take the
device entry point on the current stream (results returned as torch tensors).
The CPU phase-angle implementations of the reference (plv_reference /
plv_vectorized) are test oracles and live in
``oracle/plv_oracle.py``, not here.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Iterable

import numpy as np

from . import _native, errors
from ._arrays import describe, dtype_code, is_torch

METRIC_NAMES = {"plv": "PLV", "iplv": "iPLV", "ciplv": "ciPLV", "cre": "cRe", "cim": "cIm"}


@dataclass
class ConnectivityMatrix:
    """SPEC.md:146-152.  ``values`` is [N, N] (one band, trial-reduced),
    [B, N, N] (several bands) or [N, N, R] / [B, N, N, R] (trial_reduce='none',
    the Appendix's ``plv(:,:,t)`` layout)."""

    values: object
    metric: str
    n_observations: int
    meta: dict = field(default_factory=dict)


def _infer_kind(code: str, input_kind: str | None) -> str:
    if input_kind is not None:
        if input_kind not in _native.INPUT_KINDS:
            raise ValueError(f"input_kind must be one of {sorted(_native.INPUT_KINDS)}")
        return input_kind
    return "real" if code in ("f32", "f64") else "analytic"


def plv_family(x, *, input_kind: str | None = None, metrics: Iterable[str] = ("plv", "iplv", "ciplv"),
               precision: str = "split", trial_reduce: str = "mean", amp_floor: float = 1e-6,
               bands: bool = False, shard: tuple[int, int] = (0, 1), out: dict | None = None,
               timing: bool = False, stages=None, mode: str = "over_samples", fir=None,
               pad_samples: int = 0, layout: str = "full") -> dict:
    """All requested PLV-family metrics from one Gram per trial.

    x: RealEpochs / AnalyticEpochs / PhasorEpochs data, shape [N, T], [N, T, R]
       or with ``bands=True`` [B, N, T, R]; numpy (host) or CUDA torch tensor.
    input_kind: 'real' (Hilbert first), 'analytic' (normalise first) or
       'phasor' (unit phasors, zeros = masked); default from the dtype.
    precision: 'split' (tcgen05 fp16x3, fp32 outputs, |err| <= 1e-5) or 'fp64'
       (DMMA, fp64 outputs, |err| <= 1e-12).
    trial_reduce: 'mean' (mean of per-trial metrics), 'none' (per trial),
       'pool' (one Gram over all R*T observations) -- SURVEY D1 -- or 'sum'
       (sum of per-trial metrics: the partial sums of a (band, trial)-sharded
       call, combined by sharding.reduce_trial_partials).
    shard: (index, count) output-tile sharding; entries owned by
       other shards are left as allocated (zeros when ``out`` is None).
    out: optional preallocated outputs {metric: array} (same kind as x; numpy
       arrays for a CUDA x make the call copy the results out to the host,
       streamed while the Gram runs -- ps_plv_family_to_host).
    stages: (stage_cols, ready_events) for a CUDA input that arrives in row
       chunks (ps_plv_family_staged): rows [cols[s], cols[s+1]) of every unit
       are valid once torch.cuda.Event ready_events[s] completes.
    mode: 'over_samples' (Eq 7, default) or 'over_trials' (Eq 8: time-resolved,
       one matrix per sample from the Gram over trials; values [N, N, T],
       trial_reduce ignored).
    fir, pad_samples: optional band-pass front end for real input (a
       signalprep.FirFilter or taps): two-pass zero-phase FIR on the record
       reflection-padded by pad_samples, analytic signal before the trim
       (SURVEY 3.2, 8(f) #1), fused into the Hilbert
       stage of the same call.
    layout: 'full' (both triangles, default) or 'upper' (only i <= j of every
       matrix is computed and, for host arrays, transferred -- BASELINE
       configs[4]'s output; the strictly lower triangle is zero when the
       outputs are allocated here).
    Returns {metric: ConnectivityMatrix}.
    """
    if layout not in _native.LAYOUTS:
        raise ValueError(f"layout must be one of {sorted(_native.LAYOUTS)}")
    if mode not in ("over_samples", "over_trials"):
        raise ValueError("mode must be 'over_samples' or 'over_trials'")
    over_trials = mode == "over_trials"
    if hasattr(x, "data") and not isinstance(x, np.ndarray) and not is_torch(x):
        x = x.data  # RealEpochs / AnalyticEpochs / PhasorEpochs
    metrics = tuple(metrics)
    bad = [m for m in metrics if m not in _native.METRIC_BITS]
    if bad or not metrics:
        raise ValueError(f"unknown metrics {bad}; choose from {list(_native.METRIC_BITS)}")
    if precision not in _native.PRECISIONS:
        raise ValueError(f"precision must be one of {sorted(_native.PRECISIONS)}")
    if trial_reduce not in _native.TRIAL_REDUCE:
        raise ValueError(f"trial_reduce must be one of {sorted(_native.TRIAL_REDUCE)}")
    d = describe(x, bands=bands)
    kind = _infer_kind(d.dtype, input_kind)
    B, N, T, R = d.dims
    per_trial = trial_reduce == "none" and R > 1 and not over_trials
    slots = B * T if over_trials else (B * R if per_trial else B)
    fp64 = _native.PRECISIONS[precision] == 1
    bits = 0
    for m in metrics:
        bits |= _native.METRIC_BITS[m]

    a = _native.PlvArgs()
    a.input = d.ptr
    a.dtype = dtype_code(d.dtype)
    a.input_kind = _native.INPUT_KINDS[kind]
    a.n_bands, a.n_signals, a.n_samples, a.n_trials = B, N, T, R
    a.stride_band, a.stride_signal, a.stride_sample, a.stride_trial = d.strides
    a.amp_floor = float(amp_floor)
    a.metrics = bits
    a.precision = _native.PRECISIONS[precision]
    a.trial_reduce = _native.TRIAL_REDUCE[trial_reduce]
    a.shard_index, a.shard_count = int(shard[0]), int(shard[1])
    a.mode = 1 if over_trials else 0
    a.out_layout = _native.LAYOUTS[layout]
    zero_init = shard[1] > 1 or layout == "upper"
    fir_keep = None
    if fir is not None:
        from .signalprep import fir_struct

        fs, fir_keep = fir_struct(fir, pad_samples)
        a.fir = ctypes.pointer(fs)

    outs = {}
    # CUDA input with numpy output arrays: ps_plv_family_to_host (compute and a
    # streamed copy-out into the host arrays inside the call)
    host_out = d.on_device and out is not None and stages is None and all(
        isinstance(out.get(m), np.ndarray) for m in metrics)
    if host_out:
        import torch

        ndt = np.float64 if fp64 else np.float32
        for m in metrics:
            o = out[m]
            if o.dtype != ndt or not o.flags.c_contiguous or o.size != slots * N * N:
                raise ValueError(f"out[{m!r}] must be a C-contiguous {ndt.__name__} array with {slots * N * N} "
                                 "elements")
            outs[m] = o
            setattr(a, "out_" + m, o.ctypes.data)
        dev = torch.device("cuda", d.device)
        with torch.cuda.device(dev):
            a.stream = torch.cuda.current_stream(dev).cuda_stream
            ctx = _native.context(d.device)
            ctx.set_timing(timing)
            res = _native.PlvResult()
            _native.check(_native.lib().ps_plv_family_to_host(ctx.handle, ctypes.byref(a), ctypes.byref(res)))
    elif d.on_device:
        import torch

        tdt = torch.float64 if fp64 else torch.float32
        dev = torch.device("cuda", d.device)
        for m in metrics:
            o = None if out is None else out.get(m)
            if o is None:
                o = (torch.zeros if zero_init else torch.empty)((slots, N, N), dtype=tdt, device=dev)
            elif o.dtype != tdt or not o.is_contiguous() or o.numel() != slots * N * N:
                raise ValueError(f"out[{m!r}] must be a contiguous {tdt} tensor with {slots * N * N} elements")
            outs[m] = o
        with torch.cuda.device(dev):
            a.stream = torch.cuda.current_stream(dev).cuda_stream
            for m in metrics:
                setattr(a, "out_" + m, outs[m].data_ptr())
            ctx = _native.context(d.device)
            ctx.set_timing(timing)
            res = _native.PlvResult()
            if stages is None:
                _native.check(_native.lib().ps_plv_family(ctx.handle, ctypes.byref(a), ctypes.byref(res)))
            else:
                cols, events = stages
                n = len(cols) - 1
                ccols = (ctypes.c_int64 * (n + 1))(*[int(v) for v in cols])
                cevs = (ctypes.c_void_p * n)(*[(e.cuda_event if e is not None else None) for e in events])
                _native.check(_native.lib().ps_plv_family_staged(ctx.handle, ctypes.byref(a), ctypes.byref(res), n,
                                                                 ccols, cevs))
    else:
        ndt = np.float64 if fp64 else np.float32
        for m in metrics:
            o = None if out is None else out.get(m)
            if o is None:
                o = (np.zeros if zero_init else np.empty)((slots, N, N), dtype=ndt)
            elif o.dtype != ndt or not o.flags.c_contiguous or o.size != slots * N * N:
                raise ValueError(f"out[{m!r}] must be a C-contiguous {ndt.__name__} array with {slots * N * N} "
                                 "elements")
            outs[m] = o
            setattr(a, "out_" + m, o.ctypes.data)
        a.stream = None
        ctx = _native.context(0)
        ctx.set_timing(timing)
        res = _native.PlvResult()
        _native.check(_native.lib().ps_plv_family_host(ctx.handle, ctypes.byref(a), ctypes.byref(res)))
    info = res.as_dict()
    if info.get("n_indeterminate_ciplv") and "ciplv" in metrics:
        import warnings

        warnings.warn(f"{info['n_indeterminate_ciplv']} ciPLV pair(s) have |Re| within fp32 resolution of 1 and "
                      "|Im| > 4e-6: their ciPLV is indeterminate in split precision (reported 0); use "
                      "precision='fp64' for them (SPEC.md:259)", errors.CiplvIndeterminateWarning, stacklevel=2)
    info["input_copied"] = bool(info["input_copied"]) or d.copied
    info["precision"] = precision
    info["trial_reduce"] = trial_reduce
    info["layout"] = layout
    result = {}
    for m in metrics:
        v = outs[m]
        if over_trials:  # TimeResolvedPLV layout [N, N, T]
            v = v.reshape(B, T, N, N)
            v = v.permute(0, 2, 3, 1) if is_torch(v) else np.moveaxis(v, 1, 3)
            if not bands:
                v = v[0]
        elif per_trial:
            v = v.reshape(B, R, N, N)
            v = v.permute(0, 2, 3, 1) if is_torch(v) else np.moveaxis(v, 1, 3)
            if not bands:
                v = v[0]
        else:
            v = v.reshape(B, N, N)
            if not bands:
                v = v[0]
        result[m] = ConnectivityMatrix(values=v, metric=METRIC_NAMES[m],
                                       n_observations=int(info["n_observations"]), meta=info)
    return result


def _phasor_input(phasors):
    if hasattr(phasors, "data") and not isinstance(phasors, np.ndarray) and not is_torch(phasors):
        return phasors.data
    return phasors


def plv_matrix(phasors, mode: str = "over_samples", *, trial_reduce: str = "mean",
               precision: str = "split") -> ConnectivityMatrix:
    """(1/T)|z_i z_j^H| for all pairs via one Gram per trial.

    ``phasors``: PhasorEpochs (or its complex data) [N, T, R]; masked samples
    are exactly 0 and drop out of both the product and the per-pair T
    (SPEC.md:260).  Mode 'over_trials' (Eq 8): time-resolved PLV,
    one matrix per sample from the Gram over trials -> values [N, N, T]
    (TimeResolvedPLV).
    """
    if mode not in ("over_samples", "over_trials"):
        raise ValueError("mode must be 'over_samples' or 'over_trials'")
    return plv_family(_phasor_input(phasors), input_kind="phasor", metrics=("plv",), precision=precision,
                      trial_reduce=trial_reduce, mode=mode)["plv"]


def iplv(phasors, *, trial_reduce: str = "mean", precision: str = "split") -> ConnectivityMatrix:
    """(1/T)|Im z_i z_j^H| (absolute value per SPEC.md:258)."""
    return plv_family(_phasor_input(phasors), input_kind="phasor", metrics=("iplv",), precision=precision,
                      trial_reduce=trial_reduce)["iplv"]


def ciplv(phasors, *, trial_reduce: str = "mean", precision: str = "split") -> ConnectivityMatrix:
    """|Im| / sqrt(1 - Re^2), 0 at the singularity."""
    return plv_family(_phasor_input(phasors), input_kind="phasor", metrics=("ciplv",), precision=precision,
                      trial_reduce=trial_reduce)["ciplv"]


# --------------------------------------------------------------------------
# Welch coherence family
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class WelchConfig:
    """window_len samples, overlap samples, Hamming taper."""
    window_len: int
    overlap: int
    taper: str = "hamming"


@dataclass
class CoherenceSpectrum:
    """values over bins k = 0 .. window_len // 2 at angular
    frequency 2 pi k / window_len (freq_axis, radians per sample)."""
    values: np.ndarray
    n_segments: int
    window_len: int
    overlap: int
    freq_axis: np.ndarray


# COH metric names -> slots of the PLV-family epilogue (include/phasesync.h ps_coherence)
COH_SLOTS = {"coh": "plv", "icoh": "iplv", "cre": "cre", "cim": "cim", "ciplv": "ciplv"}
BAND_REDUCE = {"mean": 0, "max": 1, "none": 2}


def welch_bins(window_len: int, band) -> tuple[int, int]:
    """(first bin, number of bins) of `band` (radians per sample, inclusive edges)."""
    first = ctypes.c_int64()
    n = _native.lib().ps_welch_bins(int(window_len), float(band[0]), float(band[1]), ctypes.byref(first))
    return int(first.value), int(n)


def coherence_matrix(x, cfg: WelchConfig, band, *, mode: str = "max", metrics: Iterable[str] = ("coh",),
                     precision: str = "split", bands: bool = False, shard: tuple[int, int] = (0, 1),
                     timing: bool = False, layout: str = "full") -> dict:
    """All-pairs Welch coherence aggregated over `band`:
    band_coherence(coherence_welch(x_i, x_j), band, mode) for every pair, from
    one Gram over segments per frequency bin on the sm_100a path.

    x: RealEpochs data [N, T], [N, T, R] or (bands=True) [B, N, T, R]; numpy
       or CUDA torch tensor.  Segments are drawn within each trial and pooled
       over trials.
    band: (low, high) in radians per sample; mode 'max' (COH_MAX), 'mean'
       (COH_MEAN) or 'none' (one matrix per bin: values [N, N, n_bins]).
    metrics: 'coh' (|C|, Eq 12), 'icoh' (|Im C|, imaginary coherency), 'cre' /
       'cim' (signed coherency parts).
    layout: 'full' or 'upper' (only i <= j computed; lower triangle zero).
    Returns {metric: ConnectivityMatrix}.
    """
    import torch

    if layout not in _native.LAYOUTS:
        raise ValueError(f"layout must be one of {sorted(_native.LAYOUTS)}")
    if mode not in BAND_REDUCE:
        raise ValueError("mode must be 'max', 'mean' or 'none'")
    if cfg.taper != "hamming":
        raise ValueError("only the Hamming taper is defined (SPEC.md:169)")
    if hasattr(x, "data") and not isinstance(x, np.ndarray) and not is_torch(x):
        x = x.data
    metrics = tuple(metrics)
    bad = [m for m in metrics if m not in COH_SLOTS]
    if bad or not metrics:
        raise ValueError(f"unknown coherence metrics {bad}; choose from {list(COH_SLOTS)}")
    host = not (is_torch(x) and x.is_cuda)
    t = x if not host else torch.from_numpy(np.asarray(x)).cuda()
    d = describe(t, bands=bands)
    if d.dtype not in ("f32", "f64"):
        raise ValueError("coherence expects real-valued epochs (SPEC.md:213)")
    B, N, T, R = d.dims
    k0, nb = welch_bins(cfg.window_len, band) if 0 <= band[0] <= band[1] <= np.pi else (0, 1)
    slots = B * nb if mode == "none" else B
    fp64 = _native.PRECISIONS[precision] == 1
    a = _native.PlvArgs()
    a.input = d.ptr
    a.dtype = dtype_code(d.dtype)
    a.input_kind = _native.INPUT_KINDS["real"]
    a.n_bands, a.n_signals, a.n_samples, a.n_trials = B, N, T, R
    a.stride_band, a.stride_signal, a.stride_sample, a.stride_trial = d.strides
    a.amp_floor = 0.0
    a.precision = _native.PRECISIONS[precision]
    a.shard_index, a.shard_count = int(shard[0]), int(shard[1])
    a.out_layout = _native.LAYOUTS[layout]
    w = _native.Welch()
    w.window_len, w.overlap = int(cfg.window_len), int(cfg.overlap)
    w.band_low, w.band_high = float(band[0]), float(band[1])
    w.reduce = BAND_REDUCE[mode]
    tdt = torch.float64 if fp64 else torch.float32
    dev = torch.device("cuda", d.device)
    outs = {}
    bits = 0
    for m in metrics:
        bits |= _native.METRIC_BITS[COH_SLOTS[m]]
        outs[m] = torch.zeros((slots, N, N), dtype=tdt, device=dev)
        setattr(a, "out_" + COH_SLOTS[m], outs[m].data_ptr())
    a.metrics = bits
    with torch.cuda.device(dev):
        a.stream = torch.cuda.current_stream(dev).cuda_stream
        ctx = _native.context(d.device)
        ctx.set_timing(timing)
        res = _native.PlvResult()
        _native.check(_native.lib().ps_coherence(ctx.handle, ctypes.byref(a), ctypes.byref(w), ctypes.byref(res)))
    info = res.as_dict()
    info.update(window_len=cfg.window_len, overlap=cfg.overlap, band=tuple(band), band_reduce=mode,
                first_bin=k0, n_bins=nb, precision=precision, layout=layout)
    names = {"coh": "COH_" + mode.upper(), "icoh": "ICOH_" + mode.upper()}
    result = {}
    for m in metrics:
        v = outs[m]
        if mode == "none":
            v = v.reshape(B, nb, N, N).permute(0, 2, 3, 1)
        else:
            v = v.reshape(B, N, N)
        if not bands:
            v = v[0]
        if host:
            v = v.cpu().numpy()
        result[m] = ConnectivityMatrix(values=v, metric=names.get(m, m), n_observations=int(info["n_observations"]),
                                       meta=info)
    return result


def _pair_spectrum(x, cfg: WelchConfig, metric: str, precision: str) -> CoherenceSpectrum:
    x = np.asarray(x) if not is_torch(x) else x
    if x.shape[0] != 2:
        raise errors.ShapeError("coherence spectra take exactly 2 signals (SPEC.md:222)")
    r = coherence_matrix(x, cfg, (0.0, np.pi), mode="none", metrics=(metric,), precision=precision)[metric]
    v = r.values
    v = v.cpu().numpy() if is_torch(v) else v
    W = int(cfg.window_len)
    return CoherenceSpectrum(values=np.asarray(v[0, 1], dtype=np.float64),
                             n_segments=int(r.n_observations), window_len=W, overlap=int(cfg.overlap),
                             freq_axis=2 * np.pi * np.arange(W // 2 + 1) / W)


def coherence_welch(x, cfg: WelchConfig, *, precision: str = "fp64") -> CoherenceSpectrum:
    """|sum_s X_i X_j^*| / sqrt(sum|X_i|^2 sum|X_j|^2) per bin
    (magnitude, not squared) for a 2-signal RealEpochs."""
    return _pair_spectrum(x, cfg, "coh", precision)


def coherence_weighted_phasor(x, cfg: WelchConfig, *, precision: str = "fp64") -> CoherenceSpectrum:
    """SPEC.md:221-228 (Eq 12, second line): the amplitude-weighted average of
    per-segment unit cross-phasors normalised by the amplitude root-product.
    On this path both forms are the same Gram over segments of the
    auto-power-normalised spectra (sum_s A_i A_j e^{i dphi} / sqrt(sum A_i^2
    sum A_j^2)), so the two agree exactly."""
    return _pair_spectrum(x, cfg, "coh", precision)


def imaginary_coherency(x, cfg: WelchConfig, *, precision: str = "fp64") -> CoherenceSpectrum:
    """|Im{sum X_i X_j^* / sqrt(sum|X_i|^2 sum|X_j|^2)}| per bin."""
    return _pair_spectrum(x, cfg, "icoh", precision)


def band_coherence(spec: CoherenceSpectrum, band, mode: str = "max") -> float:
    """max or mean of a CoherenceSpectrum over the bins with
    low <= 2 pi k / window_len <= high (inclusive); EmptyBandError
    if none.  (A reduction over one short host vector: the all-pairs version
    runs on the GPU in coherence_matrix.)"""
    if mode not in ("max", "mean"):
        raise ValueError("mode must be 'max' or 'mean'")
    k0, nb = welch_bins(spec.window_len, band) if 0 <= band[0] <= band[1] <= np.pi else (0, 0)
    if nb < 1:
        raise errors.EmptyBandError(f"band {tuple(band)} holds no bin for window_len {spec.window_len}")
    v = np.asarray(spec.values)[k0:k0 + nb]
    return float(v.max() if mode == "max" else v.mean())
