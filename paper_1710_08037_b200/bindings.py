"""bindings -- the reference's host-ecosystem entry points.

  py_analytic_signal(real array) -> complex array
  py_plv / py_iplv / py_ciplv(arrays, config) -> matrix SPEC.md:538-544

No numerical logic lives here: every call delegates to the same
core functions (connectivity / signalprep), so binding and core agree
bit-exactly.  Errors are the core's exceptions.
The GIL is released inside the native call (ctypes.CDLL).
"""
from __future__ import annotations

from . import connectivity, signalprep

_DEFAULTS = {"input_kind": None, "amp_floor": 1e-6, "trial_reduce": "mean", "precision": "split"}


def _config(config):
    cfg = dict(_DEFAULTS)
    if config:
        unknown = set(config) - set(_DEFAULTS)
        if unknown:
            raise ValueError(f"unknown config keys {sorted(unknown)}; allowed {sorted(_DEFAULTS)}")
        cfg.update(config)
    return cfg


def py_analytic_signal(real_array):
    """delegates to signalprep.analytic_signal."""
    return signalprep.analytic_signal(real_array).data


def _py_metric(metric, arrays, config):
    cfg = _config(config)
    res = connectivity.plv_family(arrays, metrics=(metric,), input_kind=cfg["input_kind"],
                                  amp_floor=cfg["amp_floor"], trial_reduce=cfg["trial_reduce"],
                                  precision=cfg["precision"])
    return res[metric].values


def py_plv(arrays, config=None):
    """SPEC.md:538-544 (Eq 7)."""
    return _py_metric("plv", arrays, config)


def py_iplv(arrays, config=None):
    """SPEC.md:538-544 (Eq 13)."""
    return _py_metric("iplv", arrays, config)


def py_ciplv(arrays, config=None):
    """SPEC.md:538-544 (Eq 14)."""
    return _py_metric("ciplv", arrays, config)


def py_plv_family(arrays, config=None, metrics=("plv", "iplv", "ciplv")):
    """All three from one Gram (the B200 build's fused entry point)."""
    cfg = _config(config)
    res = connectivity.plv_family(arrays, metrics=metrics, input_kind=cfg["input_kind"],
                                  amp_floor=cfg["amp_floor"], trial_reduce=cfg["trial_reduce"],
                                  precision=cfg["precision"])
    return {m: r.values for m, r in res.items()}
