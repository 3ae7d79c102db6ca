"""phasesync.bench -- reference import name.  make_surrogate
 is provided; the Matlab-style three-implementation sweep
(run_benchmark / emit_report) is outside this build's scope -- its protocol
(warm-up, repetitions, equality gate) is what the repository's bench.py
measures the B200 path with."""
import numpy as np

from paper_1710_08037_b200.signalprep import PhasorEpochs

_SCOPE = ("phasesync.bench.{} (SPEC.md:379-433) is outside this build's scope; the repository's bench.py "
          "times the B200 path (DESIGN.md section 7)")


def make_surrogate(n_signals: int, n_samples: int, n_trials: int, seed: int) -> PhasorEpochs:
    """seeded uniform random phases mapped to unit phasors,
    shape [n_signals, n_samples, n_trials] (complex128), no masked samples."""
    if min(n_signals, n_samples, n_trials) <= 0:
        raise ValueError("dimensions must be positive")
    ph = np.random.default_rng(seed).uniform(0.0, 2.0 * np.pi, (n_signals, n_samples, n_trials))
    z = np.exp(1j * ph)
    return PhasorEpochs(data=z, mask=np.zeros(z.shape, dtype=bool))


def run_benchmark(*args, **kwargs):
    raise NotImplementedError(_SCOPE.format("run_benchmark"))


def emit_report(*args, **kwargs):
    raise NotImplementedError(_SCOPE.format("emit_report"))
