"""phasesync.bindings -- reference import name (pkg/pyproject.toml:6) for paper_1710_08037_b200.bindings."""
from paper_1710_08037_b200.bindings import *  # noqa: F401,F403
from paper_1710_08037_b200 import bindings as _impl

__all__ = [n for n in dir(_impl) if not n.startswith("_")]
globals().update({n: getattr(_impl, n) for n in __all__})
