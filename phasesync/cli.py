"""phasesync.cli -- reference import name (pkg/pyproject.toml:19) for paper_1710_08037_b200.cli."""
from paper_1710_08037_b200.cli import *  # noqa: F401,F403
from paper_1710_08037_b200.cli import cmd_connectivity, entrypoint, read_bundle, write_bundle  # noqa: F401
