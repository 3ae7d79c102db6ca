"""CPU oracle (test infrastructure only; see plv_oracle.py header)."""
from . import plv_oracle  # noqa: F401
