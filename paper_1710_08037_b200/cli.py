"""cli -- MatrixBundle I/O and `phasesync connectivity`.

Mirrors the reference's on-disk format and the connectivity command
(SPEC.md:445-517):
  MatrixBundle  JSON header {dims, dtype f64|c128, order row-major, axes, meta}
                + raw little-endian payload sharing the basename
  RunManifest   command line, config snapshot, seeds, version, timestamp
                
  cmd_connectivity  bundle in -> ConnectivityMatrix bundle + CSV (17 significant
                digits) + manifest; exit 0 ok / 1 acceptance / 2
                usage-or-format
Only the PLV-family metrics run here (on the GPU path); coherence metrics and
the FIR band-pass are outside this build and exit with
status 2.
"""
from __future__ import annotations

import argparse
import datetime as _dt
import json
import os
import sys
from pathlib import Path

import numpy as np

from . import __version__, errors

_DTYPES = {"f64": np.dtype("<f8"), "c128": np.dtype("<c16"), "f32": np.dtype("<f4"), "c64": np.dtype("<c8")}


def _paths(path) -> tuple[Path, Path]:
    p = Path(path)
    base = p.with_suffix("") if p.suffix in (".json", ".bin") else p
    return base.with_suffix(".json"), base.with_suffix(".bin")


def write_bundle(path, array, axes=None, meta=None) -> tuple[Path, Path]:
    """Write a MatrixBundle."""
    a = np.ascontiguousarray(array)
    code = {np.dtype("float64"): "f64", np.dtype("complex128"): "c128", np.dtype("float32"): "f32",
            np.dtype("complex64"): "c64"}.get(a.dtype)
    if code is None:
        a = a.astype(np.float64)
        code = "f64"
    hdr, bin_ = _paths(path)
    header = {"dims": list(a.shape), "dtype": code, "order": "row-major",
              "axes": list(axes) if axes is not None else [f"axis{k}" for k in range(a.ndim)],
              "meta": meta or {}}
    hdr.write_text(json.dumps(header, indent=1))
    a.astype(_DTYPES[code], copy=False).tofile(bin_)
    return hdr, bin_


def read_bundle(path) -> tuple[np.ndarray, dict]:
    """Read a MatrixBundle; FormatError on any header/payload mismatch."""
    hdr, bin_ = _paths(path)
    try:
        header = json.loads(hdr.read_text())
    except FileNotFoundError as exc:
        raise errors.FormatError(f"{hdr}: header not found") from exc
    except json.JSONDecodeError as exc:
        raise errors.FormatError(f"{hdr}: invalid JSON header ({exc})") from exc
    for key in ("dims", "dtype", "order"):
        if key not in header:
            raise errors.FormatError(f"{hdr}: header lacks '{key}'")
    if header["order"] != "row-major":
        raise errors.FormatError(f"{hdr}: order must be 'row-major'")
    if header["dtype"] not in _DTYPES:
        raise errors.FormatError(f"{hdr}: unsupported dtype {header['dtype']!r}")
    dims = [int(d) for d in header["dims"]]
    dt = _DTYPES[header["dtype"]]
    expected = int(np.prod(dims)) * dt.itemsize
    if not bin_.exists():
        raise errors.FormatError(f"{bin_}: payload not found")
    size = bin_.stat().st_size
    if size != expected:
        raise errors.FormatError(f"{bin_}: payload is {size} bytes, header implies {expected} "
                                 f"(dims {dims} x {dt.itemsize} B)")
    data = np.fromfile(bin_, dtype=dt).reshape(dims)
    return data, header


def write_csv(path, matrix, metric: str) -> None:
    """Long-format CSV, 17 significant digits."""
    m = np.asarray(matrix, dtype=np.float64)
    with open(path, "w") as f:
        f.write("metric,i,j,value\n")
        n = m.shape[0]
        for i in range(n):
            row = m[i]
            f.write("".join(f"{metric},{i},{j},{row[j]:.17g}\n" for j in range(n)))


def write_manifest(path, argv, config: dict) -> None:
    """RunManifest."""
    Path(path).write_text(json.dumps({
        "command_line": list(argv),
        "config": config,
        "seeds": config.get("seeds", []),
        "library_version": __version__,
        "timestamp": _dt.datetime.now(_dt.timezone.utc).isoformat(),
    }, indent=1))


def cmd_connectivity(argv=None) -> int:
    """SPEC.md:462-470."""
    ap = argparse.ArgumentParser(prog="phasesync connectivity")
    ap.add_argument("input", help="MatrixBundle [n_signals x n_samples x n_trials] (real) or phasors (complex)")
    ap.add_argument("--metric", default="plv", choices=["plv", "iplv", "ciplv", "coh_max", "coh_mean"])
    ap.add_argument("--phasors", action="store_true", help="input holds unit phasors (masked samples = 0)")
    ap.add_argument("--analytic", action="store_true", help="input holds analytic signals")
    ap.add_argument("--band", nargs=2, type=float, default=None, metavar=("LOW", "HIGH"),
                    help="radians per sample: FIR band-pass edges for plv/iplv/ciplv (real input; SPEC.md:58), "
                         "the aggregated band for coh_max/coh_mean (SPEC.md:229)")
    ap.add_argument("--window", type=int, default=400, help="Welch window length (coherence; Fig 2: 400)")
    ap.add_argument("--overlap", type=int, default=200, help="Welch overlap (coherence; Fig 2: 200)")
    ap.add_argument("--order", type=int, default=2000, help="FIR order (even; paper: 2000)")
    ap.add_argument("--pad", type=int, default=None,
                    help="reflection padding per side in samples (default: order, capped at n_samples - 1)")
    ap.add_argument("--trial-reduce", default="mean", choices=["mean", "none", "pool"])
    ap.add_argument("--precision", default="split", choices=["split", "fp64"])
    ap.add_argument("--output", "-o", required=True)
    try:
        args = ap.parse_args(argv)
    except SystemExit as exc:
        return 2 if exc.code else 0
    coh = args.metric.startswith("coh")
    if coh and args.band is None:
        print("phasesync: coh_max / coh_mean need --band LOW HIGH (SPEC.md:229)", file=sys.stderr)
        return 2
    try:
        x, header = read_bundle(args.input)
    except errors.FormatError as exc:
        print(f"phasesync: {exc}", file=sys.stderr)
        return 2
    if x.ndim == 2:
        x = x[:, :, None]
    if x.ndim != 3:
        print(f"phasesync: expected axes [n_signals x n_samples x n_trials], got dims {list(x.shape)}",
              file=sys.stderr)
        return 2
    from . import connectivity

    kind = "phasor" if args.phasors else ("analytic" if (args.analytic or np.iscomplexobj(x)) else "real")
    fir, pad = None, 0
    try:
        if coh:  # band_coherence(coherence_welch) for all pairs
            if kind != "real":
                raise ValueError("coherence metrics take real epochs")
            mode = args.metric.split("_")[1]
            res = connectivity.coherence_matrix(x, connectivity.WelchConfig(args.window, args.overlap),
                                                tuple(args.band), mode=mode, precision=args.precision)["coh"]
        elif args.band is not None:  # band-pass -> analytic (padded) -> trim
            if kind != "real":
                raise ValueError("--band applies to real input only")
            from .signalprep import design_bandpass_fir

            fir = design_bandpass_fir(tuple(args.band), args.order)
            pad = args.pad if args.pad is not None else min(args.order, x.shape[1] - 1)
        if not coh:
            res = connectivity.plv_family(x, input_kind=kind, metrics=(args.metric,), precision=args.precision,
                                          trial_reduce=args.trial_reduce, fir=fir, pad_samples=pad)[args.metric]
    except (ValueError, RuntimeError) as exc:
        print(f"phasesync: {type(exc).__name__}: {exc}", file=sys.stderr)
        return 2
    values = np.asarray(res.values)
    out = Path(args.output)
    out.parent.mkdir(parents=True, exist_ok=True)
    axes = ["signal", "signal"] + (["trial"] if values.ndim == 3 else [])
    write_bundle(out, values.astype(np.float64), axes=axes,
                 meta={"metric": res.metric, "n_observations": res.n_observations, "input": str(args.input),
                       "input_kind": kind, "precision": args.precision, "trial_reduce": args.trial_reduce})
    if values.ndim == 2:
        write_csv(out.with_suffix(".csv"), values, res.metric)
    write_manifest(out.with_suffix(".manifest.json"), ["phasesync", "connectivity"] + list(argv or sys.argv[2:]),
                   {"metric": args.metric, "input_kind": kind, "precision": args.precision,
                    "trial_reduce": args.trial_reduce, "input_header": header, "seeds": [],
                    "band": args.band, "order": args.order if fir is not None else None,
                    "pad_samples": pad if fir is not None else None,
                    "welch": {"window_len": args.window, "overlap": args.overlap} if coh else None})
    return 0


def entrypoint(argv=None) -> int:
    """`phasesync <command> ...` (pkg/pyproject.toml:19)."""
    argv = list(sys.argv[1:] if argv is None else argv)
    if not argv or argv[0] in ("-h", "--help"):
        print("usage: phasesync connectivity INPUT --metric {plv,iplv,ciplv} -o OUTPUT [options]")
        return 0 if argv else 2
    cmd, rest = argv[0], argv[1:]
    if cmd == "connectivity":
        return cmd_connectivity(rest)
    print(f"phasesync: command {cmd!r} is not part of this build (simulate / reproduce / bench: "
          "DESIGN.md section 7)", file=sys.stderr)
    return 2


if __name__ == "__main__":
    sys.exit(entrypoint())
