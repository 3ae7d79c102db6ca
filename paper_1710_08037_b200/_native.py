"""ctypes binding of libphasesync_cuda.so (include/phasesync.h).

This is the Python side of the drop-in boundary (SPEC.md:519-564 `bindings`):
plain pointers, sizes and strides cross the C ABI; status codes map 1:1 onto
the reference's exception classes (errors.py); ctypes.CDLL
releases the GIL for the duration of every call.

There is no CPU fallback: if the library cannot be loaded, every compute entry
point raises NativeLibraryError.
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from . import errors

LIB_PATH = Path(__file__).resolve().parent / "libphasesync_cuda.so"
if os.environ.get("PS_LIB_VARIANT"):  # A/B experiments: libphasesync_cuda.<variant>.so next to the default
    LIB_PATH = LIB_PATH.with_name(f"libphasesync_cuda.{os.environ['PS_LIB_VARIANT']}.so")
ABI_VERSION = 8
LAYOUTS = {"full": 0, "upper": 1}

# ps_status -> exception class (include/phasesync.h)
PS_OK = 0
STATUS_EXC = {
    1: errors.ShapeError,
    2: errors.AllSamplesMaskedError,
    3: errors.EmptyEffectiveWindowError,
    4: ValueError,
    5: errors.UnsupportedError,
    6: errors.CudaError,
    7: errors.CudaError,
    8: MemoryError,
    9: RuntimeError,
    10: errors.SignalTooShortError,
    11: errors.WindowTooLongError,
    12: errors.EmptyBandError,
}

DTYPES = {"f32": 0, "f64": 1, "c64": 2, "c128": 3}
INPUT_KINDS = {"real": 0, "analytic": 1, "phasor": 2}
PRECISIONS = {"split": 0, "f16x3": 0, "fp64": 1}
TRIAL_REDUCE = {"mean": 0, "none": 1, "pool": 2, "sum": 3}
METRIC_BITS = {"plv": 1, "iplv": 2, "ciplv": 4, "cre": 8, "cim": 16}
METRIC_ORDER = ("plv", "iplv", "ciplv", "cre", "cim")


class Fir(ctypes.Structure):
    """Mirror of ps_fir (band-pass front end; taps is a HOST pointer)."""

    _fields_ = [
        ("taps", ctypes.POINTER(ctypes.c_double)),
        ("n_taps", ctypes.c_int64),
        ("pad_samples", ctypes.c_int64),
    ]


class PlvArgs(ctypes.Structure):
    """Mirror of ps_plv_args (include/phasesync.h)."""

    _fields_ = [
        ("input", ctypes.c_void_p),
        ("dtype", ctypes.c_int32),
        ("input_kind", ctypes.c_int32),
        ("n_bands", ctypes.c_int64),
        ("n_signals", ctypes.c_int64),
        ("n_samples", ctypes.c_int64),
        ("n_trials", ctypes.c_int64),
        ("stride_band", ctypes.c_int64),
        ("stride_signal", ctypes.c_int64),
        ("stride_sample", ctypes.c_int64),
        ("stride_trial", ctypes.c_int64),
        ("amp_floor", ctypes.c_double),
        ("metrics", ctypes.c_uint32),
        ("precision", ctypes.c_int32),
        ("trial_reduce", ctypes.c_int32),
        ("out_plv", ctypes.c_void_p),
        ("out_iplv", ctypes.c_void_p),
        ("out_ciplv", ctypes.c_void_p),
        ("out_cre", ctypes.c_void_p),
        ("out_cim", ctypes.c_void_p),
        ("shard_index", ctypes.c_int32),
        ("shard_count", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("mode", ctypes.c_int32),
        ("out_layout", ctypes.c_int32),
        ("fir", ctypes.POINTER(Fir)),
    ]


class Welch(ctypes.Structure):
    """Mirror of ps_welch (Welch coherence configuration + band)."""

    _fields_ = [
        ("window_len", ctypes.c_int64),
        ("overlap", ctypes.c_int64),
        ("band_low", ctypes.c_double),
        ("band_high", ctypes.c_double),
        ("reduce", ctypes.c_int32),
        ("reserved0", ctypes.c_int32),
    ]


class PlvResult(ctypes.Structure):
    """Mirror of ps_plv_result."""

    _fields_ = [
        ("n_observations", ctypes.c_int64),
        ("n_masked_samples", ctypes.c_int64),
        ("n_refined_pairs", ctypes.c_int64),
        ("input_copied", ctypes.c_int32),
        ("n_kernel_launches", ctypes.c_int32),
        ("ms_hilbert", ctypes.c_float),
        ("ms_normalize", ctypes.c_float),
        ("ms_gram", ctypes.c_float),
        ("ms_finish", ctypes.c_float),
        ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64),
        ("gram_variant", ctypes.c_int32),
        ("n_indeterminate_ciplv", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


# exported symbols and their signatures (kept in sync with include/phasesync.h)
_SIGNATURES = {
    "ps_abi_version": ([], ctypes.c_int),
    "ps_last_error": ([], ctypes.c_char_p),
    "ps_ctx_create": ([ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "ps_ctx_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "ps_ctx_set_timing": ([ctypes.c_void_p, ctypes.c_int], ctypes.c_int),
    "ps_plv_family": ([ctypes.c_void_p, ctypes.POINTER(PlvArgs), ctypes.POINTER(PlvResult)], ctypes.c_int),
    "ps_plv_family_host": ([ctypes.c_void_p, ctypes.POINTER(PlvArgs), ctypes.POINTER(PlvResult)], ctypes.c_int),
    "ps_plv_family_to_host": ([ctypes.c_void_p, ctypes.POINTER(PlvArgs), ctypes.POINTER(PlvResult)], ctypes.c_int),
    "ps_plv_family_staged": ([ctypes.c_void_p, ctypes.POINTER(PlvArgs), ctypes.POINTER(PlvResult), ctypes.c_int32,
                              ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "ps_analytic_signal": ([ctypes.c_void_p, ctypes.POINTER(PlvArgs), ctypes.c_void_p], ctypes.c_int),
    "ps_filter_two_pass": ([ctypes.c_void_p, ctypes.POINTER(PlvArgs), ctypes.c_void_p], ctypes.c_int),
    "ps_coherence": ([ctypes.c_void_p, ctypes.POINTER(PlvArgs), ctypes.POINTER(Welch), ctypes.POINTER(PlvResult)],
                     ctypes.c_int),
    "ps_welch_bins": ([ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.POINTER(ctypes.c_int64)],
                      ctypes.c_int64),
    "ps_normalize_phasors": ([ctypes.c_void_p, ctypes.POINTER(PlvArgs), ctypes.c_void_p, ctypes.c_void_p],
                             ctypes.c_int),
    "ps_pair_shard": ([ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64],
                      ctypes.c_int32),
    "ps_tile_count": ([ctypes.c_int64, ctypes.c_int32], ctypes.c_int64),
    "ps_reduce_partials": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                            ctypes.c_double, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "ps_shard_tiles": ([ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                        ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)], ctypes.c_int64),
    "ps_shard_pack": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "ps_shard_unpack": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p], ctypes.c_int),
}

_lib = None
_lib_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """Load (once) and return the native library; raises NativeLibraryError."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise errors.NativeLibraryError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1710_08037_b200._build` "
                "(there is no CPU fallback)")
        try:
            handle = ctypes.CDLL(str(LIB_PATH))
        except OSError as exc:  # pragma: no cover - environment dependent
            raise errors.NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (argtypes, restype) in _SIGNATURES.items():
            try:
                fn = getattr(handle, name)
            except AttributeError as exc:
                raise errors.NativeLibraryError(f"{LIB_PATH} does not export {name}") from exc
            fn.argtypes = argtypes
            fn.restype = restype
        ver = handle.ps_abi_version()
        if ver != ABI_VERSION:
            raise errors.NativeLibraryError(f"ABI version mismatch: library {ver}, binding {ABI_VERSION}")
        _lib = handle
        return _lib


def check(status: int) -> None:
    """Raise the exception class mapped from a ps_status."""
    if status == PS_OK:
        return
    msg = lib().ps_last_error()
    msg = msg.decode(errors="replace") if msg else ""
    exc = STATUS_EXC.get(status, RuntimeError)
    raise exc(msg or f"phasesync native status {status}")


class Context:
    """Owns one ps_ctx (cuFFT plans + workspace) on one CUDA device."""

    def __init__(self, device: int = 0):
        self.device = int(device)
        h = ctypes.c_void_p()
        check(lib().ps_ctx_create(self.device, ctypes.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def set_timing(self, enable: bool) -> None:
        check(lib().ps_ctx_set_timing(self._h, 1 if enable else 0))

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().ps_ctx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass


_contexts: dict = {}
_ctx_lock = threading.Lock()


def context(device: int = 0) -> Context:
    """Per-(thread, device) context: the C ABI asks for one ctx per thread."""
    key = (threading.get_ident(), int(device))
    with _ctx_lock:
        ctx = _contexts.get(key)
        if ctx is None:
            ctx = Context(device)
            _contexts[key] = ctx
        return ctx


def pair_shard(n_signals: int, precision: str, shard_count: int, i: int, j: int) -> int:
    """Which output-tile shard owns pair (i, j) (host logic, CPU-callable)."""
    return int(lib().ps_pair_shard(n_signals, PRECISIONS[precision], shard_count, i, j))


def tile_count(n_signals: int, precision: str) -> int:
    return int(lib().ps_tile_count(n_signals, PRECISIONS[precision]))


def shard_tiles(n_signals: int, precision: str, shard_count: int, shard_index: int) -> tuple:
    """(number of tiles shard `shard_index` owns, tile rows, tile cols) -- the
    packed-buffer geometry of ps_shard_pack (host logic, CPU-callable)."""
    r, c = ctypes.c_int32(), ctypes.c_int32()
    n = lib().ps_shard_tiles(n_signals, PRECISIONS[precision], shard_count, shard_index, ctypes.byref(r),
                             ctypes.byref(c))
    return int(n), int(r.value), int(c.value)
