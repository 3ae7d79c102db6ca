"""phasesync -- drop-in import name of the reference package (pkg/pyproject.toml:6).

`import phasesync.connectivity` etc. resolve to the B200 implementation in
paper_1710_08037_b200.
"""
from paper_1710_08037_b200 import __version__  # noqa: F401
from . import errors  # noqa: F401
