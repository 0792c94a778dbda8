"""The multi-rank exchange (row all-gather + gradient all-reduce) of the
full-graph trainer, driven with the gloo backend on CPU at world sizes 2, 3, 4
and 8 (one box of 8 B200s: 7 peers per rank)."""
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


def _ceil_blocks(n, world):
    B = -(-n // world)
    return [int(x) for x in np.minimum(np.arange(world + 1) * B, n)]


@pytest.mark.parametrize("offsets", [[0, 4, 8], [0, 5, 9], [0, 3, 6, 7], _ceil_blocks(30, 4),
                                     _ceil_blocks(61, 8), list(range(0, 9 * 5, 5))])
def test_row_exchange_gloo(offsets):
    world = len(offsets) - 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, offsets, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = offsets[-1]
    want = np.arange(n, dtype=np.float32)[:, None] * 10 + np.arange(5)
    for rank, full, g in res:
        assert np.array_equal(full, want)
        assert np.all(g == sum(range(1, world + 1)))


@pytest.mark.parametrize("world", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("n", [232965, 2449029, 111059956, 9])
def test_trainer_block_layout(n, world):
    """Ceil-sized blocks (FullGraphTrainer and csrc/trainer.cu): every gather block has the
    same size B, rank r's rows sit at [r B, r B + nloc) in every GPU's gathered buffer, the
    last block may be short, and the blocks tile [0, n) exactly."""
    B = -(-n // world)
    offs = np.minimum(np.arange(world + 1) * B, n)
    assert offs[0] == 0 and offs[-1] == n
    nloc = np.diff(offs)
    assert np.array_equal(nloc, np.clip(n - np.arange(world) * B, 0, B)) and nloc.sum() == n
    if n >= world * (world - 1):       # the BASELINE shapes: only the last block is short
        assert np.all(nloc[:-1] == B) and 0 < nloc[-1] <= B
    # the gathered buffer (world * B rows) holds every rank's block at the same offset
    assert world * B >= n and world * B - n < world


def _needs_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_06837_b200.cobatch import exchange_row_needs
    B = 50
    rng = np.random.default_rng(rank)
    cols = torch.from_numpy(rng.integers(0, world * B, 400).astype(np.int32))
    recv, off = exchange_row_needs(cols, B, rank, world, dist.group.WORLD)
    allcols = [None] * world
    dist.all_gather_object(allcols, cols.numpy())
    # what each peer reads from my block, computed here from its columns
    exp = []
    for p in range(world):
        if p == rank:
            continue
        c = allcols[p]
        exp.append(np.unique(c[(c >= rank * B) & (c < (rank + 1) * B)]) - rank * B)
    got = [recv[off[i]:off[i + 1]].numpy() for i in range(world - 1)]
    q.put((rank, all(np.array_equal(a, b) for a, b in zip(got, exp)), off))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_sparse_push_row_lists_gloo(world):
    """The cooperative-batch sparse push's row lists (all_to_all of per-source needs)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_needs_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in ps:
        p.join(timeout=120)
    assert all(ok for _, ok, _ in res), res


def test_kernel_selection_helpers():
    from paper_2311_06837_b200.train import AGG_ROWS, AGG_ROWS2, _splitk_eff, agg_variant
    assert agg_variant(64, 114_624_474, 232_965) == 0          # Reddit 64-wide: warp per row
    assert agg_variant(48, 114_624_474, 232_965) == AGG_ROWS   # 48-wide rows
    assert agg_variant(64, 15_600_000, 6_000_000) == AGG_ROWS   # cobatch: 2.6 edges per row (predicated tail)
    assert agg_variant(64, 42_000_000, 6_000_000) == AGG_ROWS2  # degree 7
    assert agg_variant(64, 72_000_000, 6_000_000) == AGG_ROWS2  # degree 12
    for sk, k in [(96, 232965), (296, 100), (7, 64), (5, 0), (300, 6_000_000)]:
        e = _splitk_eff(sk, k)
        kb = -(-k // 64)
        assert 1 <= e <= max(1, min(sk, kb))
        if kb > 1:
            per = -(-kb // e)
            assert (e - 1) * per < kb           # no empty split
