"""phasesync.connectivity -- reference import name (pkg/pyproject.toml:6) for paper_1710_08037_b200.connectivity."""
from paper_1710_08037_b200.connectivity import *  # noqa: F401,F403
from paper_1710_08037_b200 import connectivity as _impl

__all__ = [n for n in dir(_impl) if not n.startswith("_")]
globals().update({n: getattr(_impl, n) for n in __all__})
