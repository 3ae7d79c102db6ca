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


def gather(outputs: dict, dst: int | None = 0, group=None) -> dict:
    """Assemble sharded outputs: reduce (dst given) or all-reduce (dst None)."""
    import torch.distributed as dist

    for v in outputs.values():
        t = v.values if hasattr(v, "values") and not hasattr(v, "dtype") else v
        if dst is None:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        else:
            dist.reduce(t, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return outputs
