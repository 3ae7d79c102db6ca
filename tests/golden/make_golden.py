"""Generates the committed golden fixtures under tests/golden/.

The reference ships no executable implementation or golden vectors
(SURVEY 8(c)); these fixtures freeze (a) the SPEC's closed-form known-answer
cases with their exact expected values and (b) oracle outputs on small seeded
versions of the five BASELINE configs, so the GPU parity tests compare
against committed bytes and any drift of the oracle itself is caught.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import plv_oracle as O  # noqa: E402
from paper_1710_08037_b200 import workloads as W  # noqa: E402


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)


def kat_offsets():
    # SPEC.md:202-203,210-211 and acceptance #3: constant phase offsets
    rng = np.random.default_rng(100)
    T = 1000
    phis = np.array([0.0, np.pi / 6, np.pi / 4, np.pi / 2, 3 * np.pi / 4])
    z0 = np.exp(1j * rng.uniform(-np.pi, np.pi, T))
    z = np.stack([z0] + [z0 * np.exp(-1j * p) for p in phis[1:]])[:, :, None]
    n = len(phis)
    plv = np.ones((n, n))
    d = phis[:, None] - phis[None, :]
    iplv = np.abs(np.sin(d))
    ciplv = np.where(np.abs(np.cos(d)) >= 1 - 1e-12, 0.0, 1.0)
    np.fill_diagonal(iplv, 0)
    np.fill_diagonal(ciplv, 0)
    save("kat_offsets", z=z.astype(np.complex128), phis=phis, plv=plv, iplv=iplv, ciplv=ciplv)


def kat_cancel():
    # T = 4, dphi = {0, pi/2, pi, 3pi/2} -> PLV = 0
    z = np.array([[1, 1, 1, 1], [1, np.exp(-0.5j * np.pi), np.exp(-1j * np.pi), np.exp(-1.5j * np.pi)]])
    save("kat_cancel", z=z[:, :, None].astype(np.complex128), plv01=np.array(0.0))


def config_case(name, x, input_kind, trial_reduce="mean", bands=False):
    xs = x if not bands else x
    outs = {}
    if bands:
        per = [O.plv_family(x[b], input_kind=input_kind, trial_reduce=trial_reduce) for b in range(x.shape[0])]
        for m in ("plv", "iplv", "ciplv"):
            outs[m] = np.stack([p[m] for p in per])
    else:
        r = O.plv_family(xs, input_kind=input_kind, trial_reduce=trial_reduce)
        for m in ("plv", "iplv", "ciplv"):
            outs[m] = r[m]
    save(name, x=np.ascontiguousarray(x), input_kind=np.array(input_kind), trial_reduce=np.array(trial_reduce),
         **outs)


def main():
    kat_offsets()
    kat_cancel()
    config_case("c1_full", W.c1(), "real")                                     # configs[0] verbatim
    config_case("c2_small", W.c2(n_signals=64, n_samples=1000, n_trials=4, n_coupled=10), "real")
    config_case("c3_small", W.c3(n_signals=48, n_samples=4096), "real")
    config_case("c4_small", W.c4(n_signals=32, n_samples=512, n_trials=3, n_latent=4), "real", bands=True)
    config_case("c5_small", W.c5(n_signals=64, n_samples=1024, n_latent=4), "analytic")


if __name__ == "__main__":
    main()
