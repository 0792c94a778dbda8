"""The multi-rank exchange (row all-gather + gradient all-reduce) of the
full-graph trainer, driven with the gloo backend on CPU at world_size 2 and 3."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, offsets, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_06837_b200.train import RowExchange
    ex = RowExchange(np.asarray(offsets), rank, world, dist.group.WORLD)
    n = offsets[-1]
    full = torch.zeros(n, 5)
    lo, hi = offsets[rank], offsets[rank + 1]
    full[lo:hi] = torch.arange(lo, hi, dtype=torch.float32)[:, None] * 10 + torch.arange(5)
    ex.allgather_rows(full)
    g = torch.full((3, 4), float(rank + 1))
    ex.allreduce(g)
    q.put((rank, full.numpy().copy(), g.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("offsets", [[0, 4, 8], [0, 5, 9], [0, 3, 6, 7]])
def test_row_exchange_gloo(offsets):
    world = len(offsets) - 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, offsets, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=90) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = offsets[-1]
    want = np.arange(n, dtype=np.float32)[:, None] * 10 + np.arange(5)
    for rank, full, g in res:
        assert np.array_equal(full, want)
        assert np.all(g == sum(range(1, world + 1)))


def test_trainer_block_layout():
    """Ceil-sized blocks: every gather block has the same size, the last may be short."""
    n, world = 232965, 8
    B = -(-n // world)
    offs = np.minimum(np.arange(world + 1) * B, n)
    assert offs[-1] == n and np.all(np.diff(offs)[:-1] == B) and 0 < offs[-1] - offs[-2] <= B
