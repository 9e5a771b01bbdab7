"""Multi-GPU plumbing for the PBSA path.

Every (batch, head) unit is independent for K1-K4 (per-head persistent memory, SPEC.md:241;
per-head routing), so units are partitioned across ranks with no data-path
collective.  torch.distributed (NCCL on the GPU box, gloo in the CPU tests) is used only for the
barrier, the max-over-ranks timing reduction and -- when a head-sharded consumer needs every head
-- the output gather.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def partition_units(total_units: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced split of `total_units` (batch x heads) over `world` ranks:
    returns (first_unit, n_units) of `rank`; sizes differ by at most one."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("partition_units: bad world/rank")
    base, extra = divmod(total_units, world)
    n = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return first, n


def is_dist() -> bool:
    return dist.is_available() and dist.is_initialized()


def barrier() -> None:
    if is_dist() and dist.get_world_size() > 1:
        dist.barrier()


def max_over_ranks(x: float, device: torch.device | str = "cpu") -> float:
    """Max of a per-rank scalar (device-timed milliseconds) over all ranks."""
    if not is_dist() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_units(o_local: torch.Tensor, total_units: int) -> torch.Tensor:
    """All-gather head/batch-sharded outputs [n_local_units, ...] into [total_units, ...] in unit
    order (uneven shards are padded to the largest shard for the collective)."""
    if not is_dist() or dist.get_world_size() == 1:
        return o_local
    world = dist.get_world_size()
    sizes = [partition_units(total_units, world, r)[1] for r in range(world)]
    mx = max(sizes)
    pad = torch.zeros((mx,) + tuple(o_local.shape[1:]), dtype=o_local.dtype, device=o_local.device)
    pad[: o_local.shape[0]] = o_local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return torch.cat([b[:n] for b, n in zip(bufs, sizes)], 0)
