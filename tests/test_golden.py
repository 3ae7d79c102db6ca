"""The oracle reproduces the committed golden fixtures (tests/golden/*.npz,
made by tests/golden/make_golden.py) and the SPEC closed-form KAT values."""
import os

import numpy as np
import pytest

from oracle import plv_oracle as O

G = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(G, name + ".npz"), allow_pickle=False)


def test_kat_offsets_exact():
    d = load("kat_offsets")
    r = O.plv_family(d["z"], input_kind="phasor")
    for m in ("plv", "iplv", "ciplv"):
        assert np.max(np.abs(r[m] - d[m])) < 1e-9, m


def test_kat_cancel():
    d = load("kat_cancel")
    assert O.plv_family(d["z"], input_kind="phasor")["plv"][0, 1] < 1e-12


@pytest.mark.parametrize("name", ["c1_full", "c2_small", "c3_small", "c5_small"])
def test_config_fixtures(name):
    d = load(name)
    r = O.plv_family(d["x"], input_kind=str(d["input_kind"]), trial_reduce=str(d["trial_reduce"]))
    for m in ("plv", "iplv", "ciplv"):
        assert np.max(np.abs(r[m] - d[m])) < 1e-12, m


def test_c4_fixture_bands():
    d = load("c4_small")
    x = d["x"]
    for b in range(x.shape[0]):
        r = O.plv_family(x[b], input_kind="real")
        for m in ("plv", "iplv", "ciplv"):
            assert np.max(np.abs(r[m] - d[m][b])) < 1e-12
