"""paper_1710_08037_b200 -- B200-native PLV / iPLV / ciPLV (arXiv 1710.08037).

The reference's `phasesync` API (pkg/pyproject.toml:6; SPEC.md modules
`signalprep`, `connectivity`, `bindings`, `errors`) backed by
libphasesync_cuda.so (sm_100a: cuFFT Hilbert, split-plane normalisation,
tcgen05 upper-triangle Gram with a fused PLV-family epilogue, FP64 DMMA
accuracy mode).  The top-level `phasesync` package re-exports these modules
under the reference's import names.
"""
from . import errors  # noqa: F401

__version__ = "0.1.0"

__all__ = ["errors", "signalprep", "connectivity", "bindings", "workloads"]


def __getattr__(name):  # lazy: importing the package must not require a GPU
    if name in ("signalprep", "connectivity", "bindings", "workloads", "_native"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
