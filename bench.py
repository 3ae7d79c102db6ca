#!/usr/bin/env python
"""Benchmark of the PLV / iPLV / ciPLV hot path (BASELINE.json metric:
pair.samples/s for PLV+iPLV+ciPLV at 1/2/4/8 GPUs, % of tensor / HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl reference]

A step = one pass of the hot path over one batch of the synthetic workload
(SURVEY 8(d)): analytic/real input resident in HBM -> normalise (+Hilbert for
real configs) -> upper-triangle Gram + fused PLV/iPLV/ciPLV epilogue, all
three metrics written to HBM.  Default workload = config C5 (20k signals,
BASELINE.json configs[4]): the config the metric's 1->8 GPU scaling target is
quoted on; it fits one B200.  Multi-GPU (one rank per GPU over NCCL; with
--gpus N and no torchrun environment the script re-launches itself under
torch.distributed.run): single-trial configs keep the input on rank 0 and
broadcast it over NVLink inside the timed region, output tiles sharded across
ranks (no gather); multi-trial configs (C2, C4) pre-place each rank's
contiguous chunk of (band, trial) units and combine the per-rank trial sums
with a fixed-order reduce-scatter (all-to-all + ordered sum) inside the timed
region.

Rank 0 prints ONE JSON line.  `--impl reference` times the reference's CPU
algorithm (the NumPy restatement in oracle/, all host cores) on a bounded
sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1710_08037_b200 import workloads as W  # noqa: E402

METRIC = "pair·samples/s for PLV+iPLV+ciPLV at 1/2/4/8 GPU; % tensor/HBM roofline"
UNIT = "pair·samples/s"
FLOPS_PER_PAIR_SAMPLE = 8  # complex MAC
FP64_DGEMM_TFLOPS_FALLBACK = 35.5  # only if the live DGEMM probe fails (tools/fp64_peak.py, K6)


def fp64_peak_tflops(dev):
    """FP64 roofline measured live on this GPU (MEASURED_PEAKS.json has no
    FP64 entry): best of 5 cuBLAS DGEMMs 8192^3 (2 N^3 flop), CUDA events."""
    import torch

    try:
        n = 8192
        a = torch.randn(n, n, dtype=torch.float64, device=dev)
        b = torch.randn(n, n, dtype=torch.float64, device=dev)
        torch.matmul(a, b)
        torch.cuda.synchronize(dev)
        best = None
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        del a, b
        return 2.0 * n ** 3 / (best / 1e3) / 1e12, "measured live: cuBLAS DGEMM 8192^3, best of 5 (this run)"
    except Exception as exc:  # pragma: no cover - device dependent
        return FP64_DGEMM_TFLOPS_FALLBACK, f"fallback {FP64_DGEMM_TFLOPS_FALLBACK} (probe failed: {exc})"


def relaunch_under_torchrun(n: int) -> None:
    """`bench.py --gpus N` without a torchrun environment: re-exec under
    torch.distributed.run with N local ranks (one per GPU), 127.0.0.1
    rendezvous and NCCL's communicator-init lines enabled.  Fails loudly when
    fewer than N GPUs are visible (never silently runs fewer ranks)."""
    import socket

    if "--launch-selftest" not in sys.argv:
        import torch

        have = torch.cuda.device_count()
        if have < n:
            print(json.dumps({"error": f"--gpus {n} requested but only {have} CUDA device(s) are visible"}),
                  flush=True)
            sys.exit(3)
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    argv = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execvpe(sys.executable, argv, env)


def launch_selftest(args):
    """CPU check of the launcher (gloo): every rank reports the world size it
    sees; rank 0 prints the line a GPU run would carry n_gpus in."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.ones(1)
    if world > 1:
        dist.all_reduce(t)
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps({"launch_selftest": True, "n_gpus": world, "gpus_requested": args.gpus,
                          "ranks_seen": int(t.item()), "nccl_debug": os.environ.get("NCCL_DEBUG")}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def finite(obj):
    """JSON-safe copy: non-finite floats become null (strict JSON parsers)."""
    if isinstance(obj, dict):
        return {k: finite(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [finite(v) for v in obj]
    if isinstance(obj, float) and not math.isfinite(obj):
        return None
    return obj


def peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        p.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
        p["source"] = "measured (MEASURED_PEAKS.json)"
    return p


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join("/tmp", f"ps_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [s.strip() for s in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------- CPU legs
def cpu_sample_run(x, kind, n_sig, trial_reduce="mean", reps=1):
    """Time the oracle (NumPy/OpenBLAS restatement of Appendix impl 3) on the
    first n_sig signals of the workload; returns (pair.samples/s, seconds)."""
    from oracle import plv_oracle as O

    xs = np.ascontiguousarray(x[:n_sig])
    N, T, R = xs.shape
    O.plv_family(xs[: min(n_sig, 64)], input_kind=kind, trial_reduce=trial_reduce)  # warm-up
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        O.plv_family(xs, input_kind=kind, trial_reduce=trial_reduce)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return W.pair_samples(N, T, R) / best, best


def cpu_baseline(x, kind, target_s=10.0, max_sig=None):
    """Grow the signal sample until one oracle pass takes >= target_s / 4."""
    N = x.shape[0]
    n = min(N, 256)
    while True:
        rate, dt = cpu_sample_run(x, kind, n)
        if dt >= target_s / 4 or n >= N or (max_sig and n >= max_sig):
            break
        n = min(N, int(n * max(1.5, min(4.0, (target_s / 4 / max(dt, 1e-3)) ** 0.5))))
    return rate, dt, n


def cores():
    return os.cpu_count() or 1


# ----------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(W.CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--precision", default="split", choices=["split", "fp64"])
    ap.add_argument("--layout", default=None, choices=["full", "upper"],
                    help="output layout (default: 'upper' for c5, whose BASELINE config asks for the upper "
                         "triangle of each metric; 'full' otherwise)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-stage-bcast", dest="stage_bcast", action="store_false",
                    help="N>1: broadcast the whole input before computing instead of overlapping row chunks")
    ap.add_argument("--launch-selftest", action="store_true", help="CPU/gloo check of the --gpus N launcher")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args.gpus)  # does not return
    if args.launch_selftest:
        launch_selftest(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    N, T, R, B, dt, kind = W.CONFIGS[args.config]
    layout = args.layout or ("upper" if args.config == "c5" else "full")
    work = W.pair_samples(N, T, R, B)
    cfg = {"workload": f"{args.config}: {W.DESCRIPTIONS[args.config]}", "n_signals": N, "n_samples": T,
           "n_trials": R, "n_bands": B, "input": dt, "input_kind": kind, "trial_reduce": "mean",
           "precision": args.precision, "pair_samples_per_step": work,
           "output_layout": layout + (" (i <= j of each [N][N] matrix, BASELINE configs[4])" if layout == "upper"
                                      else " (both triangles)"),
           "l2": "inputs larger than L2 (126 MB) every step",
           "parallelism": (f"output-tile shards x{world} + chunked NCCL broadcast of the input from rank 0, "
                           "overlapped with compute" if R == 1 and B == 1 else
                           f"(band, trial) unit shards x{world}: each rank holds and normalises only its "
                           "contiguous chunk of units (pre-placed), per-rank trial sums, fixed-order "
                           "reduce-scatter (NCCL all-to-all + ordered sum) of the trial mean, output rows "
                           "sharded") if world > 1 else "single GPU"}

    if args.impl == "reference":
        if rank != 0:
            return
        cfg["precision"] = "fp64 (the reference's CPU arithmetic: complex128 zgemm, SPEC.md:265)"
        os.environ.setdefault("OPENBLAS_NUM_THREADS", str(cores()))
        x = W.generate(args.config)
        if x.ndim == 4:
            x = x[0]
        for _ in range(max(0, args.warmup)):
            cpu_sample_run(x, kind, min(N, 128))
        n_s = None
        rates = []
        for _ in range(args.steps):
            if n_s is None:
                rate, dt_s, n_s = cpu_baseline(x, kind, target_s=8.0)
            else:
                rate, dt_s = cpu_sample_run(x, kind, n_s)
            rates.append(rate)
        val = float(np.median(rates))
        sample = f"first {n_s} of {N} signals x {T} samples x {R} trials (band 0), full pipeline per step"
        line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": work / val * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded, SURVEY 8(d))", "config": cfg,
                "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores(), "kind": "port", "sample": sample},
                "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    from paper_1710_08037_b200 import _native
    from paper_1710_08037_b200 import connectivity as C
    from paper_1710_08037_b200 import sharding

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    # ---- workload: generated on the host (seeded), resident in HBM --------
    x_host = W.generate(args.config)
    if x_host.ndim == 3:
        x_store = np.ascontiguousarray(np.transpose(x_host, (2, 0, 1)))[None]  # [1, R, N, T]
    else:
        x_store = np.ascontiguousarray(np.transpose(x_host, (0, 3, 1, 2)))     # [B, R, N, T]
    bands = x_host.ndim == 4
    fp64 = args.precision == "fp64"
    odt = torch.float64 if fp64 else torch.float32
    metrics = ("plv", "iplv", "ciplv")
    single = R == 1 and B == 1
    units = world > 1 and not single  # (band, trial) unit sharding (C2, C4)
    shard = (rank, world) if not units else (0, 1)

    if units:
        # each rank holds only its contiguous chunk of (band, trial) units,
        # pre-placed on its GPU outside the timed region
        frags_ix = sharding.unit_ranges(B, R, world, rank)
        frags_dev = [(b, torch.from_numpy(np.ascontiguousarray(x_store[b, t0:t1])).to(dev).permute(1, 2, 0))
                     for b, t0, t1 in frags_ix]
        my_units = sum(t1 - t0 for _, t0, t1 in frags_ix)
        parts = {m: torch.zeros((B, N, N), dtype=odt, device=dev) for m in metrics}
        xd = None
    else:
        xd = torch.from_numpy(x_store).to(dev)                                  # [B, R, N, T]
        if world > 1 and rank != 0:
            xd.zero_()  # single-trial configs: only rank 0 holds the input (broadcast in the timed region)
        xv = xd[0].permute(1, 2, 0) if not bands else xd.permute(0, 2, 3, 1)
        outs = {m: torch.zeros((B, N, N), dtype=odt, device=dev) for m in metrics}
        bcast_t = torch.view_as_real(xd) if xd.is_complex() else xd

    # N > 1, single-trial configs: the input lives on rank 0 and is broadcast
    # over NVLink in row chunks; each rank starts a chunk's normalisation and
    # the Gram tiles it unlocks as soon as it arrives (ps_plv_family_staged).
    staged = world > 1 and single and args.stage_bcast
    cols = sharding.stage_cols(N, n_stages=8) if staged else None
    comm = torch.cuda.Stream() if staged else None
    rows_view = bcast_t[0, 0] if staged else None  # [N, T] (real) or [N, T, 2] (complex as float pairs)

    def step(timing=False):
        """One pass of the hot path; returns (metas of the library calls)."""
        if units:
            _, metas = sharding.unit_partial_sums(frags_dev, B, N, input_kind=kind, precision=args.precision,
                                                  metrics=metrics, layout=layout, out=parts, timing=timing)
            sharding.reduce_trial_partials(parts, R)  # the exchange step: trial mean of this rank's row slice
            return metas
        if staged:
            events = sharding.broadcast_input_staged(rows_view, cols, src=0, stream=comm)
            r = C.plv_family(xv, input_kind=kind, precision=args.precision, bands=bands, shard=shard,
                             out=outs, timing=timing, stages=(cols, events), layout=layout)
            return [r["plv"].meta]
        if world > 1:
            sharding.broadcast_input(bcast_t, src=0)
        r = C.plv_family(xv, input_kind=kind, precision=args.precision, bands=bands, shard=shard,
                         out=outs, timing=timing, layout=layout)
        return [r["plv"].meta]

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # ---- timed region ------------------------------------------------------
    clk = ClockSampler(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ else local)
    clk.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    gram_ms, launches = [], 0
    e0.record(stream)
    for _ in range(args.steps):
        metas = step(timing=True)
        gram_ms.append(sum(float(mt["ms_gram"]) for mt in metas))
        launches += sum(int(mt["n_kernel_launches"]) for mt in metas)
        if units:
            launches += len(metrics)  # ps_reduce_partials: one ordered-sum kernel per metric
    info = metas[0]
    variant = int(info.get("gram_variant", 0))
    e1.record(stream)
    torch.cuda.synchronize()
    ms_total = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        dist.barrier()
    clocks = clk.stop()
    ms_step = ms_total / args.steps
    value = work / (ms_step / 1e3)

    # ---- roofline of the dominant kernel (Gram + fused epilogue) ----------
    pk = peaks()
    if units:
        my_frac = my_units / (B * R)
    else:
        my_tiles = sum(1 for t in range(_native.tile_count(N, args.precision)) if t % world == rank)
        my_frac = my_tiles / max(1, _native.tile_count(N, args.precision))
    gram_avg = float(np.mean(gram_ms)) if gram_ms else 0.0
    algo_flops = FLOPS_PER_PAIR_SAMPLE * work * my_frac
    # (the library reports the Gram's CUDA-event time; without it, fall back
    # to the whole step so the JSON never carries inf / nan)
    if not gram_avg > 0.0:
        gram_avg = ms_step
    achieved = algo_flops / (gram_avg / 1e3) / 1e12
    # SURVEY 8(d) denominator: bf16 burst peak / 3 split passes, i.e. 8
    # algorithmic flop per pair-sample against 24 fp16 tensor flop (the
    # 4-product split).  The Gauss form runs 18 tensor flop per pair-sample;
    # its own (stricter) ceiling is reported as frac_of_variant_ceiling.
    hw_flops = 18.0 if variant == 1 else 24.0
    if fp64:
        peak, fp64_basis = fp64_peak_tflops(dev)
        variant_peak = peak
    else:
        peak = pk["bf16_tflops"] * FLOPS_PER_PAIR_SAMPLE / 24.0
        variant_peak = pk["bf16_tflops"] * FLOPS_PER_PAIR_SAMPLE / hw_flops
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "gram_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            if tj.get("config") == args.config and tj.get("precision") == args.precision:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "gram_split_kernel (tcgen05 fp16x3 upper-triangle Gram + fused PLV/iPLV/ciPLV)"
                if not fp64 else "gram_f64_kernel (DMMA)",
                "algorithmic_flops_per_launch": algo_flops, "gram_ms_per_launch": gram_avg,
                "gram_share_of_step": gram_avg / ms_step,
                "gram_variant": {0: "split fp16x3, 4 real products (12 UMMA / K step)",
                                 1: "split fp16x3, Gauss 3-product form (9 UMMA / K step)",
                                 2: "fp64 DMMA"}.get(variant, str(variant)),
                "fp16_tensor_tflops_executed": achieved * hw_flops / FLOPS_PER_PAIR_SAMPLE if not fp64 else None,
                "peak_basis": (f"SURVEY 8(d): bf16_tflops {pk['bf16_tflops']} ({pk['source']}, burst) / 3 split "
                               "passes (8 algorithmic / 24 fp16 tensor flop per pair-sample)") if not fp64 else
                fp64_basis,
                "variant_ceiling": variant_peak, "frac_of_variant_ceiling": achieved / variant_peak,
                "frac_of_bf16_peak": achieved / pk["bf16_tflops"] if not fp64 else None}

    # ---- normalisation stage against the HBM roofline ----------------------
    # algorithmic bytes per sample: the input sample in, the
    # operand planes out (4 fp16 split planes, or re / im in f64); the Gauss
    # form's S / D planes (8 more bytes) are listed apart
    in_b = {"f32": 4, "f64": 8, "c64": 8, "c128": 16}.get(dt, 8)
    out_b = 16 if fp64 else 8
    n_samples = float(B) * R * N * T * (my_units / (B * R) if units else 1.0)
    ms_norm = float(info["ms_normalize"])
    norm_gbs = n_samples * (in_b + out_b) / (ms_norm / 1e3) / 1e9 if ms_norm > 0 else None
    normalize_roofline = {"bound": "hbm", "achieved": norm_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                          "frac": norm_gbs / pk["hbm_gbs"] if norm_gbs else None,
                          "bytes_per_sample": in_b + out_b,
                          "gauss_plane_bytes_per_sample": 8 if variant == 1 else 0,
                          "achieved_incl_gauss_planes": (norm_gbs * (in_b + out_b + (8 if variant == 1 else 0)) /
                                                         (in_b + out_b)) if norm_gbs else None,
                          "ms": ms_norm,
                          "stage": ("Hilbert (cuFFT chain or fused radix-16 kernel) + normalise -> operand planes"
                                    if kind == "real" else "normalise -> operand planes")}

    # ---- end to end through the public host API ----------------------------
    e2e = None
    if not args.no_e2e:
        hout = {m: torch.zeros((B, N, N), dtype=odt, pin_memory=True).numpy() for m in metrics}
        if units:
            # each rank copies only its units from pinned host memory over its
            # own link, computes its trial sums, joins the fixed-order
            # reduce-scatter and copies its rows of the trial mean back
            frag_host = [(b, torch.from_numpy(np.ascontiguousarray(x_store[b, t0:t1])).pin_memory())
                         for b, t0, t1 in frags_ix]
            in_bytes = sum(h.numel() * h.element_size() for _, h in frag_host)
            F = B * N
            r0, r1 = sharding.row_slice(F, rank, world)
            row_host = {m: torch.zeros((r1 - r0, N), dtype=odt, pin_memory=True) for m in metrics}
            out_bytes = sum(v.numel() * v.element_size() for v in row_host.values())
        elif world > 1:
            # single trial: each rank copies in only its own row slice (its own
            # host link) and one NCCL all-gather over NVLink assembles the
            # input; each rank then computes and copies out its row bands
            # (ps_plv_family_to_host, streamed)
            r0, r1 = sharding.row_slice(N, rank, world)
            loc = torch.from_numpy(np.ascontiguousarray(x_store[0, 0, r0:r1])).pin_memory()
            loc_rows = torch.view_as_real(loc) if loc.is_complex() else loc
            in_bytes = loc.numel() * loc.element_size()
        else:
            xin = torch.empty(x_store.shape, dtype=torch.from_numpy(x_store[:1, :1, :1, :1]).dtype, pin_memory=True)
            xin.numpy()[...] = x_store
            xin_np = xin.numpy()
            xin_view = np.transpose(xin_np[0], (1, 2, 0)) if not bands else np.transpose(xin_np, (0, 2, 3, 1))

        def e2e_step():
            if units:
                fr = [(b, h.to(dev, non_blocking=True).permute(1, 2, 0)) for b, h in frag_host]
                _, metas_e = sharding.unit_partial_sums(fr, B, N, input_kind=kind, precision=args.precision,
                                                        metrics=metrics, layout=layout, out=parts)
                red = sharding.reduce_trial_partials(parts, R)
                for m in metrics:
                    row_host[m].copy_(red[m][0], non_blocking=True)
                torch.cuda.synchronize()
                return dict(metas_e[0], h2d_bytes=in_bytes, d2h_bytes=out_bytes)
            if world > 1:
                xg = sharding.all_gather_rows(loc_rows, N)
                xg = torch.view_as_complex(xg) if loc.is_complex() else xg
                r = C.plv_family(xg, input_kind=kind, precision=args.precision, shard=shard, out=hout,
                                 layout=layout)
                return dict(next(iter(r.values())).meta, h2d_bytes=in_bytes)
            r = C.plv_family(xin_view, input_kind=kind, precision=args.precision, bands=bands, shard=shard,
                             out=hout, layout=layout)
            return dict(next(iter(r.values())).meta)

        e2e_step()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            meta_e = e2e_step()
        dt_e = (time.perf_counter() - t0) / args.steps
        if world > 1:
            t = torch.tensor([dt_e], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt_e = float(t.item())
            # whole-job link bytes: the sum over ranks
            nb = torch.tensor([float(meta_e.get("h2d_bytes") or 0), float(meta_e.get("d2h_bytes") or 0)],
                              device=dev, dtype=torch.float64)
            dist.all_reduce(nb, op=dist.ReduceOp.SUM)
            meta_e["h2d_bytes"], meta_e["d2h_bytes"] = int(nb[0].item()), int(nb[1].item())
        # bytes the library actually moved over the host link
        e2e = {"value": work / dt_e, "unit": UNIT,
               "h2d_bytes_per_step": int(meta_e.get("h2d_bytes") or x_store.nbytes),
               "d2h_bytes_per_step": int(meta_e.get("d2h_bytes") or sum(v.nbytes for v in hout.values())),
               "output_bytes_per_step": int(sum(v.nbytes for v in hout.values())),
               "ms_per_step": dt_e * 1e3,
               "api": ("per-rank (band, trial) units (pinned) -> H2D -> sharding.unit_partial_sums "
                       "(connectivity.plv_family trial_reduce='sum' -> ps_plv_family) -> "
                       "sharding.reduce_trial_partials (NCCL all-to-all + ps_reduce_partials) -> D2H of the "
                       "rank's rows of the trial mean") if units else
                      ("per-rank row slice (pinned) -> NCCL all-gather -> connectivity.plv_family(cuda input, "
                       "numpy pinned outputs) -> ps_plv_family_to_host (C ABI), each rank its row bands")
                      if world > 1 else
                      "paper_1710_08037_b200.connectivity.plv_family(numpy pinned) -> ps_plv_family_host (C ABI)"}

    # ---- CPU baseline (rank 0, N=1 only) -----------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        os.environ.setdefault("OPENBLAS_NUM_THREADS", str(cores()))
        xs = x_host if x_host.ndim == 3 else x_host[0]
        rate, dt_s, n_s = cpu_baseline(xs, kind, target_s=12.0)
        cpu = {"value": rate, "unit": UNIT, "cores": cores(), "kind": "port",
               "sample": f"oracle/plv_oracle.py (NumPy + OpenBLAS, {cores()} threads) on the first {n_s} of "
                         f"{N} signals x {T} samples x {R} trials{' (band 0)' if B > 1 else ''}: "
                         f"{dt_s:.2f} s per pass"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None,
                "dtype": "f16x3 split (fp32 accumulate, fp32 out)" if not fp64 else "f64",
                "data": "synthetic (seeded numpy generator, SURVEY 8(d)); stands in for the paper's MEG data",
                "config": cfg, "roofline": roofline, "normalize_roofline": normalize_roofline, "cpu_baseline": cpu,
                "e2e": e2e,
                "gpu_launches": launches, "clocks": clocks,
                "stages_ms": {"normalize": float(info["ms_normalize"]), "gram": gram_avg,
                              "finish": float(info["ms_finish"])}}
        print(json.dumps(finite(line)), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
