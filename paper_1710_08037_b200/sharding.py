"""Multi-GPU output-tile sharding for the PLV family.

One process per GPU (torchrun / torch.distributed over NCCL).  Each rank
computes the upper-triangle output tiles t with t % world_size == rank
(``ps_plv_args.shard_index/shard_count``) into zero-initialised outputs; every
pair (i, j) and its mirror is written by exactly one tile, so the full matrix
is the element-wise SUM of the shards -- a single NCCL reduce / all-reduce
gathers it exactly (x + 0 == x), and only when the caller asks for it.

When the input lives on one rank only ("input on GPU 0"),
``broadcast_input`` ships it over NVLink before the compute; with per-rank
pre-placed inputs (independent bands / trials) nothing crosses the link.
"""
from __future__ import annotations

import numpy as np

from . import _native

SPLIT_TILE = (256, 128)
FP64_TILE = (64, 64)


def tiles(n_signals: int, precision: str = "split"):
    """Upper-triangle tile list in the library's enumeration order
    (capi.cu build_tiles): J-major, tiles holding at least one pair i <= j."""
    bm, bn = SPLIT_TILE if _native.PRECISIONS[precision] == 0 else FP64_TILE
    out = []
    nj = -(-n_signals // bn)
    ni = -(-n_signals // bm)
    for J in range(nj):
        jmax = min(J * bn + bn, n_signals) - 1
        for I in range(ni):
            if I * bm <= jmax:
                out.append((I, J))
    return out


def owner_matrix(n_signals: int, precision: str, shard_count: int) -> np.ndarray:
    """owner[i, j] = shard that writes (i, j) (symmetric)."""
    bm, bn = SPLIT_TILE if _native.PRECISIONS[precision] == 0 else FP64_TILE
    own = np.full((n_signals, n_signals), -1, dtype=np.int32)
    for t, (I, J) in enumerate(tiles(n_signals, precision)):
        i0, i1 = I * bm, min(I * bm + bm, n_signals)
        j0, j1 = J * bn, min(J * bn + bn, n_signals)
        blk = own[i0:i1, j0:j1]
        ii, jj = np.meshgrid(np.arange(i0, i1), np.arange(j0, j1), indexing="ij")
        sel = ii <= jj
        blk[sel] = t % shard_count
    iu = np.triu_indices(n_signals)
    own.T[iu] = own[iu]
    return own


def broadcast_input(x, src: int = 0, group=None):
    """Ship a device input from rank `src` to every rank (NCCL broadcast)."""
    import torch.distributed as dist

    dist.broadcast(x, src=src, group=group)
    return x


def stage_cols(n_signals: int, n_stages: int = 8, min_width: int = 1024) -> list:
    """Stage boundaries for the staged ("growing square") schedule: interior
    boundaries are multiples of 256 (the split tile height)."""
    per_stage = -(-n_signals // n_stages)                 # ceil(N / n_stages)
    width = max(min_width, -(-per_stage // 256) * 256)    # rounded up to 256
    cols = list(range(0, n_signals, width)) + [n_signals]
    return cols


def broadcast_input_staged(rows_view, cols, src: int = 0, group=None, stream=None):
    """Chunked NCCL broadcast of a device input whose signal rows lie along
    dim 0 (`rows_view[c0:c1]` must be contiguous, e.g. a single-trial
    [N, T] / [N, T, 2] tensor).  Returns one torch.cuda.Event per chunk,
    recorded on `stream` after that chunk's broadcast; feed them with `cols`
    to connectivity.plv_family(stages=(cols, events)) so each rank starts
    normalising / computing a chunk as soon as it has arrived."""
    import torch
    import torch.distributed as dist

    stream = stream or torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())  # earlier work on the buffer is ordered first
    events = []
    with torch.cuda.stream(stream):
        for c0, c1 in zip(cols[:-1], cols[1:]):
            dist.broadcast(rows_view[c0:c1], src=src, group=group)
            ev = torch.cuda.Event()
            ev.record(stream)
            events.append(ev)
    return events


def row_slice(n_signals: int, rank: int, world: int) -> tuple:
    """Rows [r0, r1) of the input a rank holds / copies in for
    ``all_gather_rows`` (equal ceil(N / world) slices, the last one short)."""
    per = -(-n_signals // world)
    return min(rank * per, n_signals), min((rank + 1) * per, n_signals)


def all_gather_rows(local_rows, n_signals: int, group=None, device=None):
    """Assemble a single-trial input on every rank from per-rank row slices:
    `local_rows` is this rank's rows ``row_slice(N, rank, world)`` -- a host
    (pinned) or device tensor [rows, ...] -- copied in by this rank alone, then
    one NCCL all-gather over NVLink gives every rank all N rows.  Returns the
    device tensor [N, ...] (a view of the gathered buffer)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    per = -(-n_signals // world)
    dev = device or (torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available()
                     else torch.device("cpu"))
    mine = torch.zeros((per,) + tuple(local_rows.shape[1:]), dtype=local_rows.dtype, device=dev)
    if local_rows.shape[0]:
        mine[: local_rows.shape[0]].copy_(local_rows, non_blocking=True)
    full = torch.empty((per * world,) + tuple(local_rows.shape[1:]), dtype=local_rows.dtype, device=dev)
    if dev.type == "cuda":
        dist.all_gather_into_tensor(full, mine, group=group)
    else:  # gloo (CPU tests)
        dist.all_gather(list(full.chunk(world)), mine, group=group)
    return full[:n_signals]


def gather_dense(outputs: dict, dst: int | None = 0, group=None) -> dict:
    """Assemble sharded outputs by a dense SUM reduce (dst given) / all-reduce
    (dst None) of the zero-filled shards -- exact (each entry has one writer)
    but every rank pushes whole N x N matrices; ``gather`` moves only the tiles
    each rank owns.  Kept for callers whose outputs are not tile-sharded."""
    import torch.distributed as dist

    for v in outputs.values():
        t = v.values if hasattr(v, "values") and not hasattr(v, "dtype") else v
        if dst is None:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        else:
            dist.reduce(t, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return outputs


def _native_pack(mat, n_signals, precision, world, rank, packed):
    import torch

    from . import _native

    ctx = _native.context(mat.device.index)
    with torch.cuda.device(mat.device):
        st = torch.cuda.current_stream(mat.device).cuda_stream
        _native.check(_native.lib().ps_shard_pack(ctx.handle, n_signals, _native.PRECISIONS[precision], world, rank,
                                                  mat.data_ptr(), packed.data_ptr(), st))


def _native_unpack(packed, n_signals, precision, world, shard, mat, mirror):
    import torch

    from . import _native

    ctx = _native.context(mat.device.index)
    with torch.cuda.device(mat.device):
        st = torch.cuda.current_stream(mat.device).cuda_stream
        _native.check(_native.lib().ps_shard_unpack(ctx.handle, n_signals, _native.PRECISIONS[precision], world,
                                                    shard, packed.data_ptr(), mat.data_ptr(), int(mirror), st))


def gather(outputs: dict, n_signals: int, precision: str = "split", layout: str = "full", group=None,
           packer=None, unpacker=None, tile_counts=None) -> dict:
    """All-gather of owned output tiles ("gathering the output
    only if the caller asks for it").  Each rank packs the upper-triangle
    tiles it owns (ps_shard_pack, the ps_pair_shard rule) of every [N][N]
    slot of every metric into one dense buffer, one NCCL all-gather moves
    1/P of the output per rank, and every rank unpacks the other ranks'
    tiles (ps_shard_unpack: owned entries i <= j, plus the mirror for the full
    layout -- negated for the antisymmetric 'cim').  ``outputs``: {metric:
    CUDA tensor [..., N, N] or ConnectivityMatrix}, filled in place.
    packer / unpacker / tile_counts: injectable for the CPU (gloo) tests of
    the exchange; the product path uses the library's kernels."""
    import torch
    import torch.distributed as dist

    from . import _native

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        return outputs
    packer = packer or _native_pack
    unpacker = unpacker or _native_unpack
    if tile_counts is None:
        geo = [_native.shard_tiles(n_signals, precision, world, s) for s in range(world)]
        counts = [g[0] for g in geo]
        te = geo[0][1] * geo[0][2]
    else:
        counts, te = tile_counts
    per = max(counts) * te
    for name, v in outputs.items():
        t = v.values if hasattr(v, "values") and not hasattr(v, "dtype") else v
        mats = t.reshape(-1, n_signals, n_signals)
        mirror = 0 if layout == "upper" else (-1 if name == "cim" else 1)
        for slot in range(mats.shape[0]):
            mat = mats[slot]
            mine = torch.zeros(per, dtype=mat.dtype, device=mat.device)
            packer(mat, n_signals, precision, world, rank, mine)
            allp = torch.empty(world * per, dtype=mat.dtype, device=mat.device)
            if mat.is_cuda:
                dist.all_gather_into_tensor(allp, mine, group=group)
            else:  # gloo (CPU tests)
                dist.all_gather(list(allp.chunk(world)), mine, group=group)
            for s in range(world):
                if s != rank:
                    unpacker(allp[s * per:(s + 1) * per], n_signals, precision, world, s, mat, mirror)
    return outputs


# ---------------------------------------------------------------------------
# (band, trial) unit sharding for multi-trial configs (C2, C4)
# ---------------------------------------------------------------------------
def unit_ranges(n_bands: int, n_trials: int, world: int, rank: int) -> list:
    """This rank's contiguous chunk of the flattened (band, trial) unit list
    (units u = b * R + t; chunk sizes differ by at most one) as
    [(band, t0, t1), ...] -- at most one fragment per band.  SPEC.md:128:
    per-trial work is independent."""
    U = n_bands * n_trials
    u0, u1 = U * rank // world, U * (rank + 1) // world
    out = []
    u = u0
    while u < u1:
        b, t0 = divmod(u, n_trials)
        t1 = min(n_trials, t0 + (u1 - u))
        out.append((b, t0, t1))
        u += t1 - t0
    return out


def unit_partial_sums(fragments, n_bands: int, n_signals: int, *, input_kind: str = "real",
                      precision: str = "split", metrics=("plv", "iplv", "ciplv"), layout: str = "full",
                      out: dict | None = None, timing: bool = False) -> tuple:
    """Per-band sums over this rank's trials of the per-trial metrics
    (trial_reduce='sum'): ``fragments`` = [(band, x)] with x this rank's
    trials of that band as a CUDA [N, T, r] array (e.g. a view of its
    pre-placed [r, N, T] units).  Returns ({metric: [B, N, N] tensor, zero for
    bands this rank holds no trial of}, [meta of each call])."""
    import torch

    from . import connectivity as C

    fp64 = precision == "fp64"
    dev = None
    for _, xf in fragments:
        dev = xf.device
        break
    if dev is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    tdt = torch.float64 if fp64 else torch.float32
    parts = out if out is not None else {
        m: torch.zeros((n_bands, n_signals, n_signals), dtype=tdt, device=dev) for m in metrics}
    if out is not None:
        for m in metrics:
            parts[m].zero_()
    metas = []
    for b, xf in fragments:
        res = C.plv_family(xf, input_kind=input_kind, metrics=metrics, precision=precision, trial_reduce="sum",
                           out={m: parts[m][b:b + 1] for m in metrics}, layout=layout, timing=timing)
        metas.append(next(iter(res.values())).meta)
    return parts, metas


def _native_reduce(parts, n_parts, stride, n, divisor, out):
    import torch

    from . import _native

    ctx = _native.context(out.device.index)
    with torch.cuda.device(out.device):
        st = torch.cuda.current_stream(out.device).cuda_stream
        dt = _native.DTYPES["f64"] if out.dtype == torch.float64 else _native.DTYPES["f32"]
        _native.check(_native.lib().ps_reduce_partials(ctx.handle, parts.data_ptr(), n_parts, stride, n,
                                                       float(divisor), dt, out.data_ptr(), st))


def reduce_trial_partials(parts: dict, n_trials: int, group=None, gather_all: bool = False, reducer=None) -> dict:
    """Combine the ranks' per-band trial sums into the trial mean, in a fixed
    rank order.  The [B, N, N] slots are read as B*N flat rows
    split into ``row_slice`` chunks; one all-to-all hands rank s the P
    partials of its row chunk, and ps_reduce_partials sums them left to right
    (rank 0 first) and divides by the global trial count: a deterministic
    reduce-scatter.  Returns {metric: (rows [r0, r1) of the flat [B*N, N]
    result, (r0, r1))}; with gather_all=True the full [B, N, N] mean on every
    rank instead (one more all-gather).  ``reducer`` is injectable for the
    CPU (gloo) tests; the product path uses the library's kernel."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    reducer = reducer or _native_reduce
    out = {}
    for m, t in parts.items():
        B, N = t.shape[0], t.shape[-1]
        F = B * N
        flat = t.reshape(F, N)
        sl = [row_slice(F, s, world) for s in range(world)]
        r0, r1 = sl[rank]
        mine = r1 - r0
        if world == 1:
            recv = flat.contiguous().reshape(-1)
        else:
            recv = torch.empty(world * mine * N, dtype=t.dtype, device=t.device)
            dist.all_to_all_single(recv, flat.contiguous().reshape(-1), output_split_sizes=[mine * N] * world,
                                   input_split_sizes=[(b - a) * N for a, b in sl], group=group)
        res = torch.empty(mine * N, dtype=t.dtype, device=t.device)
        if mine:
            reducer(recv, world, mine * N, mine * N, float(n_trials), res)
        rows = res.reshape(mine, N)
        if gather_all:
            full = all_gather_rows(rows, F, group=group, device=t.device)
            out[m] = full.reshape(B, N, N)
        else:
            out[m] = (rows, (r0, r1))
    return out
