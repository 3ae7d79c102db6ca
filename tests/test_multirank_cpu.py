"""N>1 host logic on CPU: world_size-2 gloo processes each own the tiles the
library assigns them (ps_pair_shard), fill only those entries (standing in
for their GPU outputs) and `sharding.gather_dense` / `sharding.gather` (the
all-gather of owned tiles) reassemble the oracle matrix bit-exactly; the
input broadcast, the (band, trial) unit split and the fixed-order
reduce-scatter of trial partial sums are exercised too."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import plv_oracle as O
from paper_1710_08037_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, prec, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = torch.zeros(N, 256, dtype=torch.complex128)
        if rank == 0:
            x.copy_(torch.from_numpy(O.make_surrogate(N, 256, 1, seed=77)[:, :, 0]))
        xr = torch.view_as_real(x)
        sharding.broadcast_input(xr, src=0)
        z = x.numpy()[:, :, None]
        full = O.plv_family(z, input_kind="phasor")
        own = sharding.owner_matrix(N, prec, world)
        outs = {}
        for m in ("plv", "iplv", "ciplv"):
            shard = np.where(own == rank, full[m], 0.0)
            outs[m] = torch.from_numpy(np.ascontiguousarray(shard))
        sharding.gather_dense(outs, dst=None)
        ok = all(np.array_equal(outs[m].numpy(), full[m]) for m in outs)
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("prec", ["split", "fp64"])
def test_two_rank_shard_and_gather(prec):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    N = 300
    procs = [ctx.Process(target=_worker, args=(r, 2, port, N, prec, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)]


def _gather_worker(rank, world, port, N, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = np.random.default_rng(78).standard_normal((N, 64, 2)).astype(np.float32)
        r0, r1 = sharding.row_slice(N, rank, world)
        got = sharding.all_gather_rows(torch.from_numpy(full[r0:r1]), N, device=torch.device("cpu"))
        q.put((rank, tuple(got.shape) == full.shape and np.array_equal(got.numpy(), full)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N", [(2, 301), (3, 300), (3, 2)])
def test_all_gather_rows_from_per_rank_slices(world, N):
    # multi-GPU host input: each rank copies in only its row slice, one
    # all-gather assembles the whole input on every rank (uneven and empty
    # slices included)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, N, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, True) for r in range(world)]


# ---- all-gather of owned tiles (sharding.gather) ---------------------------
def _tile_geo(N, prec):
    bm, bn = sharding.SPLIT_TILE if prec == "split" else sharding.FP64_TILE
    return sharding.tiles(N, prec), bm, bn


def _np_pack(mat, N, prec, world, rank, packed):
    # CPU stand-in for ps_shard_pack (the product path runs the library kernel)
    tl, bm, bn = _tile_geo(N, prec)
    mine = [t for k, t in enumerate(tl) if k % world == rank]
    buf = packed.view(-1)
    for q, (I, J) in enumerate(mine):
        blk = torch.zeros(bm, bn, dtype=mat.dtype)
        sub = mat[I * bm:min(N, I * bm + bm), J * bn:min(N, J * bn + bn)]
        blk[:sub.shape[0], :sub.shape[1]] = sub
        buf[q * bm * bn:(q + 1) * bm * bn] = blk.reshape(-1)


def _np_unpack(packed, N, prec, world, shard, mat, mirror):
    tl, bm, bn = _tile_geo(N, prec)
    mine = [t for k, t in enumerate(tl) if k % world == shard]
    for q, (I, J) in enumerate(mine):
        blk = packed[q * bm * bn:(q + 1) * bm * bn].reshape(bm, bn)
        for r in range(bm):
            i = I * bm + r
            if i >= N:
                break
            for c in range(bn):
                j = J * bn + c
                if j >= N or i > j:
                    continue
                mat[i, j] = blk[r, c]
                if mirror and i != j:
                    mat[j, i] = -blk[r, c] if mirror < 0 else blk[r, c]


def _tile_gather_worker(rank, world, port, N, prec, layout, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        z = O.make_surrogate(N, 128, 1, seed=79)
        full = O.plv_family(z, input_kind="phasor")
        for m in ("plv", "ciplv"):  # the library's outputs are exactly symmetric (upper mirrored)
            full[m] = np.triu(full[m]) + np.triu(full[m], 1).T
        full["cim"] = np.triu(np.random.default_rng(3).standard_normal((N, N)), 1)
        full["cim"] = full["cim"] - full["cim"].T
        own = sharding.owner_matrix(N, prec, world)
        upper = np.triu(np.ones((N, N), dtype=bool))
        outs = {}
        for m in ("plv", "ciplv", "cim"):
            keep = (own == rank) & (upper if layout == "upper" else True)
            outs[m] = torch.from_numpy(np.ascontiguousarray(np.where(keep, full[m], 0.0)))
        tl, bm, bn = _tile_geo(N, prec)
        counts = [sum(1 for k in range(len(tl)) if k % world == s) for s in range(world)]
        sharding.gather(outs, N, prec, layout, packer=_np_pack, unpacker=_np_unpack, tile_counts=(counts, bm * bn))
        ok = True
        for m, t in outs.items():
            want = full[m] if layout == "full" else np.where(upper, full[m], 0.0)
            ok = ok and np.array_equal(t.numpy(), want)
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("prec,layout,N", [("split", "full", 300), ("fp64", "upper", 150)])
def test_two_rank_gather_owned_tiles(prec, layout, N):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tile_gather_worker, args=(r, 2, port, N, prec, layout, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)]


# ---- (band, trial) units and the fixed-order reduce of trial partials ------
@pytest.mark.parametrize("B,R,world", [(5, 60, 8), (1, 20, 8), (1, 20, 3), (2, 3, 4), (1, 1, 2)])
def test_unit_ranges_partition(B, R, world):
    seen = []
    sizes = []
    for r in range(world):
        fr = sharding.unit_ranges(B, R, world, r)
        assert len({b for b, _, _ in fr}) == len(fr)  # at most one fragment per band
        n = 0
        for b, t0, t1 in fr:
            assert 0 <= t0 < t1 <= R and 0 <= b < B
            seen += [b * R + t for t in range(t0, t1)]
            n += t1 - t0
        sizes.append(n)
    assert seen == list(range(B * R))  # contiguous, in order, each unit once
    assert max(sizes) - min(sizes) <= 1


def _np_reduce(parts, n_parts, stride, n, divisor, out):
    # CPU stand-in for ps_reduce_partials: left-to-right sum, then / divisor
    acc = parts[:n].clone()
    for p in range(1, n_parts):
        acc += parts[p * stride:p * stride + n]
    out.copy_(acc / divisor)


def _reduce_worker(rank, world, port, B, N, R, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(80)
        per_trial = rng.uniform(0, 1, size=(B, R, N, N)).astype(np.float32)
        part = np.zeros((B, N, N), dtype=np.float32)
        for b, t0, t1 in sharding.unit_ranges(B, R, world, rank):
            for t in range(t0, t1):
                part[b] += per_trial[b, t]
        # every rank's partial sums, for the expected fixed-order result
        allp = np.zeros((world, B, N, N), dtype=np.float32)
        for s in range(world):
            for b, t0, t1 in sharding.unit_ranges(B, R, world, s):
                for t in range(t0, t1):
                    allp[s, b] += per_trial[b, t]
        want = allp[0].copy()
        for s in range(1, world):
            want += allp[s]
        want /= np.float32(R)
        got = sharding.reduce_trial_partials({"plv": torch.from_numpy(part)}, R, reducer=_np_reduce)
        rows, (r0, r1) = got["plv"]
        ok = np.array_equal(rows.numpy(), want.reshape(B * N, N)[r0:r1])
        full = sharding.reduce_trial_partials({"plv": torch.from_numpy(part)}, R, reducer=_np_reduce,
                                              gather_all=True)["plv"]
        ok = ok and np.array_equal(full.numpy(), want)
        ok = ok and np.allclose(want, per_trial.mean(axis=1), atol=1e-6)
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,B,N,R", [(2, 3, 17, 5), (3, 1, 10, 20)])
def test_reduce_trial_partials_fixed_order(world, B, N, R):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_reduce_worker, args=(r, world, port, B, N, R, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, True) for r in range(world)]
