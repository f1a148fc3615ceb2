"""Multi-GPU plumbing: one process per GPU, torch.distributed.

Inference shards the receiver (query) set across ranks with the Gaussians
replicated: there is no data-path collective.  The only exchanges are the
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
