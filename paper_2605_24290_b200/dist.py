"""Multi-GPU plumbing: one process per GPU, torch.distributed.

Inference shards the query set across ranks with the Gaussians replicated:
there is no data-path collective.  Configs 2 and 5 split the receivers; the
config-3 coverage table (n_tx x n_rx) is split over a gt x gr grid of
ranks (transmitter blocks x receiver blocks), chosen by a cost model so
neither the receiver-side conditioning cache nor the per-transmitter state
builds are replicated more than they must be.  The only exchanges are the
timing max-reduce and an optional all-gather of the (tiny) RSSI table.
Training (config 4) all-reduces one flat gradient buffer.  The same code
runs over NCCL (GPU tensors) and gloo (CPU tensors, used by the tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [begin, end) of n_total items for `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, rem = divmod(n_total, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


# Per-item costs (ms, one B200, K=500k, 90x360) of the coverage-table phases
# (bench config3 phase_ms, round 1): the receiver-side conditioning cache
# (Tx-independent), the per-transmitter state (projection, sort, walk) and
# the per-(tx, rx) signal + compositing.  Only their ratios matter.
COVERAGE_COSTS = (27.3 / 1024, 71.1 / 64, 87.4 / 65536)


def coverage_grid(n_tx: int, n_rx: int, world: int, costs=COVERAGE_COSTS) -> tuple[int, int]:
    """(gt, gr) with gt * gr == world: transmitter blocks x receiver blocks
    of the coverage table, minimising the slowest rank's modelled time
    c_rx * rx_block + c_tx * tx_block + c_q * tx_block * rx_block."""
    c_rx, c_tx, c_q = costs
    best = None
    for gt in range(1, world + 1):
        if world % gt:
            continue
        gr = world // gt
        bt, br = -(-n_tx // gt), -(-n_rx // gr)
        cost = c_rx * br + c_tx * bt + c_q * bt * br
        if best is None or cost < best[0] - 1e-12:
            best = (cost, gt, gr)
    return best[1], best[2]


def coverage_shard(n_tx: int, n_rx: int, rank: int, world: int, grid=None) -> tuple[int, int, int, int]:
    """This rank's block [tx_begin, tx_end) x [rx_begin, rx_end) of the table;
    rank = it * gr + ir over the (gt, gr) grid."""
    gt, gr = grid if grid is not None else coverage_grid(n_tx, n_rx, world)
    if gt * gr != world:
        raise ValueError("grid does not cover the world")
    it, ir = divmod(rank, gr)
    tb, te = shard_range(n_tx, it, gt)
    rb, re_ = shard_range(n_rx, ir, gr)
    return tb, te, rb, re_


def gather_table(local: torch.Tensor, n_tx: int, n_rx: int, grid=None) -> torch.Tensor:
    """All-gather the per-rank blocks of coverage_shard into the n_tx x n_rx table."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    grid = grid if grid is not None else coverage_grid(n_tx, n_rx, world)
    blocks = [coverage_shard(n_tx, n_rx, r, world, grid) for r in range(world)]
    ht = max(te - tb for tb, te, _, _ in blocks)
    wr = max(re_ - rb for _, _, rb, re_ in blocks)
    pad = torch.zeros((ht, wr), dtype=local.dtype, device=local.device)
    pad[: local.shape[0], : local.shape[1]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    out = torch.empty((n_tx, n_rx), dtype=local.dtype, device=local.device)
    for p, (tb, te, rb, re_) in zip(parts, blocks):
        out[tb:te, rb:re_] = p[: te - tb, : re_ - rb]
    return out


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device time) over all ranks."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local: torch.Tensor, n_total: int) -> torch.Tensor:
    """All-gather per-rank row blocks produced by shard_range into one table
    (e.g. the config-3 RSSI coverage table, n_tx x n_rx)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world = dist.get_world_size()
    sizes = [shard_range(n_total, r, world) for r in range(world)]
    width = max(e - b for b, e in sizes)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([p[: e - b] for p, (b, e) in zip(parts, sizes)], dim=0)


def allreduce_grads(flat: torch.Tensor) -> torch.Tensor:
    """Sum the flat gradient buffer over ranks in place (the training step's
    only collective; NCCL over NVLink on the GPUs)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM)
    return flat


def nccl_comm_ptr(group=None) -> int:
    """The ncclComm_t behind torch's NCCL process group (for
    Trainer.allreduce, which issues ncclAllReduce on the library's stream).
    The communicator must exist: run one collective on the group first."""
    pg = group if group is not None else dist.distributed_c10d._get_default_group()
    return int(pg._get_backend(torch.device("cuda"))._comm_ptr())
