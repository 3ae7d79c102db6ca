"""Array plumbing for the C ABI: numpy (host) and torch (device) inputs.

The reference ArrayView is a contiguous row-major buffer
[n_signals x n_samples x n_trials]; copies are made -- and flagged -- when the
layout differs.  Here any strided layout is described to the
library by element strides; only dtypes the kernels do not consume natively
(ints, float16, ...) and negative-stride host views are copied.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import errors
from ._native import DTYPES

_NP_CODES = {np.dtype(np.float32): "f32", np.dtype(np.float64): "f64",
             np.dtype(np.complex64): "c64", np.dtype(np.complex128): "c128"}


def _torch():
    try:
        import torch  # noqa: F401
        return torch
    except Exception:  # pragma: no cover
        return None


def is_torch(x) -> bool:
    t = _torch()
    return t is not None and isinstance(x, t.Tensor)


@dataclass
class ArrayDesc:
    obj: object            # the (possibly converted) array kept alive for the call
    ptr: int
    dtype: str             # f32 / f64 / c64 / c128
    dims: tuple            # (B, N, T, R)
    strides: tuple         # element strides (sb, sn, st, sr)
    on_device: bool
    device: int
    copied: bool


def describe(x, bands: bool = False) -> ArrayDesc:
    """Describe an input of shape [N,T], [N,T,R] or (bands=True) [B,N,T,R]."""
    copied = False
    if is_torch(x):
        torch = _torch()
        t = x
        if t.dtype not in (torch.float32, torch.float64, torch.complex64, torch.complex128):
            t = t.to(torch.float64)
            copied = True
        code = {torch.float32: "f32", torch.float64: "f64", torch.complex64: "c64",
                torch.complex128: "c128"}[t.dtype]
        shape = tuple(t.shape)
        st = tuple(t.stride())
        on_dev = t.is_cuda
        dev = t.device.index if on_dev else 0
        if not on_dev:
            t = t.numpy() if not t.is_conj() else t.resolve_conj().numpy()
            return describe(t, bands)
        ptr = t.data_ptr()
        obj = t
    else:
        a = np.asarray(x)
        if a.dtype not in _NP_CODES:
            a = a.astype(np.float64)
            copied = True
        if any(s < 0 for s in a.strides):
            a = np.ascontiguousarray(a)
            copied = True
        code = _NP_CODES[a.dtype]
        shape = a.shape
        item = a.dtype.itemsize
        if any(s % item for s in a.strides):
            a = np.ascontiguousarray(a)
            copied = True
        st = tuple(s // a.dtype.itemsize for s in a.strides)
        ptr = a.ctypes.data
        obj = a
        on_dev = False
        dev = 0
    nd = len(shape)
    if bands:
        if nd != 4:
            raise errors.ShapeError(
                f"expected axes [n_bands x n_signals x n_samples x n_trials], got shape {shape}")
        B, N, T, R = shape
        sb, sn, ss, sr = st
    else:
        if nd == 2:
            (N, T), (sn, ss) = shape, st
            R, sr = 1, 0
        elif nd == 3:
            (N, T, R), (sn, ss, sr) = shape, st
        else:
            raise errors.ShapeError(
                f"expected axes [n_signals x n_samples x n_trials] (SPEC.md:525), got shape {shape}")
        B, sb = 1, 0
    if N < 1 or R < 1 or B < 1:
        raise errors.ShapeError(f"empty signal/trial/band axis in shape {shape}")
    if T < 2:
        raise errors.ShapeError(f"n_samples must be >= 2 (SPEC.md:31), got shape {shape}")
    return ArrayDesc(obj=obj, ptr=int(ptr), dtype=code, dims=(B, N, T, R), strides=(sb, sn, ss, sr),
                     on_device=on_dev, device=int(dev), copied=copied)


def dtype_code(code: str) -> int:
    return DTYPES[code]
