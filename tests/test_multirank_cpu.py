"""N>1 host logic on CPU: world_size-2 gloo processes each own the tiles the
library assigns them (ps_pair_shard), fill only those entries (standing in
for their GPU outputs) and `sharding.gather` reassembles the oracle matrix
bit-exactly; the input broadcast path is exercised too."""
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
        sharding.gather(outs, dst=None)
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
