"""Multi-process host logic (gloo, world_size 2, CPU): receiver sharding,
max-over-ranks timing, the RSSI-table all-gather and the gradient
all-reduce used by the NCCL path on the GPUs."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_24290_b200.dist import (allreduce_grads, coverage_grid, coverage_shard, gather_rows, gather_table,
                                        max_over_ranks, shard_range)


def test_shard_range_partitions():
    for n in (0, 1, 7, 1024, 1023):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1


def test_coverage_grid_tiles_the_table():
    """Every (tx, rx) cell of the table belongs to exactly one rank."""
    for world in (1, 2, 3, 4, 6, 8):
        for n_tx, n_rx in ((64, 1024), (5, 7), (1, 16), (64, 3)):
            gt, gr = coverage_grid(n_tx, n_rx, world)
            assert gt * gr == world
            seen = [[0] * n_rx for _ in range(n_tx)]
            for r in range(world):
                tb, te, rb, re_ = coverage_shard(n_tx, n_rx, r, world)
                for t in range(tb, te):
                    for j in range(rb, re_):
                        seen[t][j] += 1
            assert all(v == 1 for row in seen for v in row)


def test_coverage_grid_shards_transmitters_for_config3():
    """Config 3 (64 Tx x 1024 Rx, K=500k): the per-Tx state builds dominate,
    so 2 and 4 ranks split the transmitters, 8 ranks a 4 x 2 grid."""
    assert coverage_grid(64, 1024, 1) == (1, 1)
    assert coverage_grid(64, 1024, 2) == (2, 1)
    assert coverage_grid(64, 1024, 4) == (4, 1)
    assert coverage_grid(64, 1024, 8) == (4, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_rx, n_tx = 10, 3
        b, e = shard_range(n_rx, rank, world)
        # each rank "renders" its receiver shard: rssi[tx, rx] = 100 tx + rx
        local = torch.tensor([[100.0 * t + j for t in range(n_tx)] for j in range(b, e)])
        table = gather_rows(local, n_rx)
        mx = max_over_ranks(1.5 + rank)
        g = torch.full((5,), float(rank + 1))
        allreduce_grads(g)
        # coverage table over a 2 x 1 rank grid (transmitter blocks), 5 Tx x 4 Rx
        tb, te, rb, re_ = coverage_shard(5, 4, rank, world, (2, 1))
        blk = torch.tensor([[10.0 * t + j for j in range(rb, re_)] for t in range(tb, te)])
        cov = gather_table(blk, 5, 4, (2, 1))
        out[rank] = (table.tolist(), mx, g.tolist(), cov.tolist())
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_world2_shard_gather_reduce():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    expect = [[100.0 * t + j for t in range(3)] for j in range(10)]
    for r in range(world):
        table, mx, g, cov = res[r]
        assert cov == [[10.0 * t + j for j in range(4)] for t in range(5)]
        assert table == expect
        assert mx == 2.5
        assert g == [3.0] * 5
