"""MatrixBundle format and CLI plumbing.  CPU only."""
import json

import numpy as np
import pytest

from paper_1710_08037_b200 import cli, errors


def test_bundle_round_trip(tmp_path):
    a = np.random.default_rng(0).standard_normal((3, 5, 2))
    cli.write_bundle(tmp_path / "x", a, axes=["signal", "sample", "trial"], meta={"fs": 1000})
    b, hdr = cli.read_bundle(tmp_path / "x.json")
    assert np.array_equal(a, b) and hdr["dims"] == [3, 5, 2] and hdr["dtype"] == "f64"
    assert hdr["meta"]["fs"] == 1000
    c = a + 1j * a
    cli.write_bundle(tmp_path / "c.bin", c)
    d, hdr = cli.read_bundle(tmp_path / "c")
    assert np.array_equal(c, d) and hdr["dtype"] == "c128"
    assert (tmp_path / "c.json").exists() and (tmp_path / "c.bin").stat().st_size == c.size * 16


def test_bundle_format_errors(tmp_path):
    a = np.zeros((2, 3))
    cli.write_bundle(tmp_path / "x", a)
    with open(tmp_path / "x.bin", "ab") as f:
        f.write(b"\0")
    with pytest.raises(errors.FormatError):
        cli.read_bundle(tmp_path / "x")
    (tmp_path / "y.json").write_text("{not json")
    with pytest.raises(errors.FormatError):
        cli.read_bundle(tmp_path / "y")
    (tmp_path / "z.json").write_text(json.dumps({"dims": [2], "dtype": "i8", "order": "row-major"}))
    with pytest.raises(errors.FormatError):
        cli.read_bundle(tmp_path / "z")
    with pytest.raises(errors.FormatError):
        cli.read_bundle(tmp_path / "missing")


def test_cli_usage_exit_codes(tmp_path):
    assert cli.entrypoint([]) == 2
    assert cli.entrypoint(["simulate"]) == 2
    cli.write_bundle(tmp_path / "x", np.zeros((2, 8, 1)))
    out = tmp_path / "o"
    assert cli.entrypoint(["connectivity", str(tmp_path / "x"), "--metric", "coh_max", "-o", str(out)]) == 2
    # reversed band edges: InvalidBandError -> usage/format exit 2
    assert cli.entrypoint(["connectivity", str(tmp_path / "x"), "--band", "0.2", "0.1", "-o", str(out)]) == 2
    assert cli.entrypoint(["connectivity", str(tmp_path / "nope"), "-o", str(out)]) == 2


def test_csv_full_precision(tmp_path):
    m = np.array([[1.0, 0.1234567890123456789], [0.1234567890123456789, 1.0]])
    cli.write_csv(tmp_path / "m.csv", m, "PLV")
    lines = (tmp_path / "m.csv").read_text().splitlines()
    assert lines[0] == "metric,i,j,value" and len(lines) == 5
    assert float(lines[2].split(",")[3]) == m[0, 1]
