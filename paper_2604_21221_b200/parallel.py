"""Multi-GPU plumbing for the PBSA path.

Every (batch, head) unit is independent for K1-K4 (per-head persistent memory, SPEC.md:241;
per-head routing), so units are partitioned across ranks with no data-path
collective.  torch.distributed (NCCL on the GPU box, gloo in the CPU tests) is used only for the
barrier, the max-over-ranks timing reduction and the output gather: with the head-partitioned
layout (`HeadLayout`) the attention outputs of a batch element's heads are spread over ranks and
one all-to-all per call brings every head of batch element e to rank e, where the head-mixing
consumer (the output projection) runs.
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


class _Done:
    """Completed work handle (single-rank exchange)."""

    def wait(self):
        return True


class HeadLayout:
    """Head-partitioned layout of `batch` x `heads` units over `world` ranks.

    Global unit u = e * heads + h (batch element e, head h) is computed on rank u % world (round
    robin: every rank gets batch*heads/world units even when heads % world != 0, e.g. 12 heads on
    8 GPUs).  Batch element e is consumed on rank e % world.  Local units are ordered by
    (destination rank, u), so a rank's output tensor [n_local, n_q, d] is already in all-to-all
    send order (no gather before the collective).  After each PBSA call, `exchange` moves every
    unit's output from its compute rank to its batch element's rank with ONE all-to-all (NCCL over
    NVLink on the GPU box)."""

    def __init__(self, batch: int, heads: int, world: int, rank: int):
        if world < 1 or not (0 <= rank < world):
            raise ValueError("HeadLayout: bad world/rank")
        self.batch, self.heads, self.world, self.rank = batch, heads, world, rank
        total = batch * heads
        mine = list(range(rank, total, world))
        # global ids computed here, in send order: by destination rank, then by global unit id
        self.local_units = sorted(mine, key=lambda u: ((u // heads) % world, u))
        self.my_batch = [e for e in range(batch) if e % world == rank]  # batch elements consumed here
        dest = [(u // heads) % world for u in self.local_units]
        self.send_splits = [sum(1 for x in dest if x == r) for r in range(world)]
        # receive order: by source rank, then by global unit id; each received unit -> (batch slot, head)
        recv = []
        for src in range(world):
            for u in range(src, total, world):
                if (u // heads) % world == rank:
                    recv.append(u)
        self.recv_splits = [sum(1 for u in recv if u % world == r) for r in range(world)]
        self.recv_units = recv
        slot = {e: i for i, e in enumerate(self.my_batch)}
        self.recv_index = [slot[u // heads] * heads + (u % heads) for u in recv]

    @property
    def n_local(self) -> int:
        return len(self.local_units)

    def _index(self, device) -> torch.Tensor:
        key = str(device)
        cache = self.__dict__.setdefault("_idx_cache", {})
        if key not in cache:
            cache[key] = torch.tensor(self.recv_index, device=device, dtype=torch.long)
        return cache[key]

    def exchange(self, o_local: torch.Tensor, out: torch.Tensor | None = None, async_op: bool = False):
        """o_local [n_local, ...] (this rank's units, local order) -> [len(my_batch) * heads, ...]
        (every head of the batch elements consumed here, (element, head) order).  With
        async_op=True returns (work, finish) -- call finish() after work.wait() to scatter the
        received units into head order."""
        send = o_local.contiguous()
        recv = torch.empty((len(self.recv_units),) + tuple(o_local.shape[1:]), dtype=o_local.dtype,
                           device=o_local.device)
        if out is None:
            out = torch.empty((len(self.my_batch) * self.heads,) + tuple(o_local.shape[1:]),
                              dtype=o_local.dtype, device=o_local.device)
        idx = self._index(o_local.device)

        def finish():
            out.index_copy_(0, idx, recv)
            return out

        if not is_dist() or self.world == 1:
            recv.copy_(send)
            return finish() if not async_op else (_Done(), finish)
        work = dist.all_to_all_single(recv, send, self.recv_splits, self.send_splits, async_op=async_op)
        if async_op:
            return work, finish
        return finish()
