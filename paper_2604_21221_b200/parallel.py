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

import os

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


class QuerySplitLayout:
    """Batch-1 layout for any world size (config 2/3: 12 heads of one batch element on 1/2/4/8
    GPUs).

    The heads are cut into G = gcd(world, heads) groups of heads/G contiguous heads; every group is
    replicated on R = world / G ranks and replica r attends the contiguous range r of the chunk's
    query blocks (balanced split).  A replica holds the group's whole KV memory (the KV write is
    replicated) and its own query blocks, so the only exchanges are
      * at the k=0 pass, an all-gather of the query-block representatives Q^c inside the group
        (s_t averages the coarse attention over ALL query blocks; 40 KB per head at
        d = 128): every replica then scores all rows, so K2's s_t and K4's update are computed
        redundantly and deterministically -- no reduction whose order could break bit-exactness;
      * after every call, the output gather of O (the consumer needs all heads of every token).
    12 heads: N = 2 -> 2 groups of 6 heads, R = 1; N = 4 -> 4 x 3, R = 1; N = 8 -> 4 x 3, R = 2
    (24 half-head units, 3 per GPU)."""

    def __init__(self, heads: int, bpc: int, world: int, rank: int):
        if world < 1 or not (0 <= rank < world):
            raise ValueError("QuerySplitLayout: bad world/rank")
        import math
        self.heads, self.bpc, self.world, self.rank = heads, bpc, world, rank
        self.groups = math.gcd(world, heads)
        self.replicas = world // self.groups
        if bpc < self.replicas:
            raise ValueError(f"QuerySplitLayout: {bpc} query blocks cannot be split {self.replicas} ways")
        self.group, self.replica = divmod(rank, self.replicas)
        self.heads_per_group = heads // self.groups
        self.head0 = self.group * self.heads_per_group
        self.q_ranges = [partition_units(bpc, self.replicas, r) for r in range(self.replicas)]
        self.q_begin, self.q_count = self.q_ranges[self.replica]
        self.max_q = max(c for _, c in self.q_ranges)
        self._group_pg = None

    @property
    def n_local(self) -> int:
        return self.heads_per_group

    def group_ranks(self, group: int | None = None) -> list[int]:
        g = self.group if group is None else group
        return [g * self.replicas + r for r in range(self.replicas)]

    def setup(self) -> None:
        """Create the per-group process groups (collective: every rank calls it, same order)."""
        if not is_dist() or self.world == 1 or self.replicas == 1:
            return
        for g in range(self.groups):
            pg = dist.new_group(self.group_ranks(g))
            if g == self.group:
                self._group_pg = pg

    def gather_qc(self, qc_full: torch.Tensor) -> torch.Tensor:
        """qc_full [heads_per_group, bpc, d]: this replica's rows are filled; after the call every
        row is (all replicas of the group end with identical tensors)."""
        if self.replicas == 1:
            return qc_full
        units, _, d = qc_full.shape
        send = torch.zeros(units, self.max_q, d, dtype=qc_full.dtype, device=qc_full.device)
        send[:, : self.q_count] = qc_full[:, self.q_begin: self.q_begin + self.q_count]
        recv = torch.empty((self.replicas * units,) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
        if is_dist():
            dist.all_gather_into_tensor(recv, send, group=self._group_pg)
            recv = recv.view((self.replicas,) + tuple(send.shape))
        else:  # single-process simulation of one rank (tools/strong_rank_sim.py): own rows everywhere
            recv = recv.view((self.replicas,) + tuple(send.shape))
            recv[:] = send
        for r, (b, c) in enumerate(self.q_ranges):
            qc_full[:, b: b + c] = recv[r, :, :c]
        return qc_full

    def _gather_output_p2p(self, o_part, block_rows, out, async_op):
        """R > 1: every (source, head) shard is one contiguous token range of one head in `out`, so
        the shards are received straight into place by point-to-point transfers (one per source and
        head) -- no rank-major staging buffer and no permuting copy after an all-gather."""
        units = o_part.shape[0]
        ops = []
        for src in range(self.world):
            g, r = divmod(src, self.replicas)
            b, c = self.q_ranges[r]
            h0 = g * self.heads_per_group
            if src == self.rank:
                out[h0: h0 + units, b * block_rows: (b + c) * block_rows].copy_(o_part[:, : c * block_rows])
                continue
            for h in range(units):
                ops.append(dist.P2POp(dist.irecv, out[h0 + h, b * block_rows: (b + c) * block_rows], src))
        for dst in range(self.world):
            if dst == self.rank:
                continue
            for h in range(units):
                ops.append(dist.P2POp(dist.isend, o_part[h].contiguous(), dst))
        works = dist.batch_isend_irecv(ops) if ops else []

        class _All:
            def wait(self):
                for w in works:
                    w.wait()
                return True

        if async_op:
            return _All(), (lambda: out)
        _All().wait()
        return out

    def gather_output(self, o_part: torch.Tensor, block_rows: int, out: torch.Tensor | None = None,
                      async_op: bool = False):
        """o_part [heads_per_group, q_count * block_rows, d] -> [heads, bpc * block_rows, d] on every
        rank (all-gather of the padded shards).  async_op=True returns (work, finish).

        Rank order is (group, replica), so with R = 1 the gathered shards already ARE the output
        in head order and NCCL writes straight into `out` (no copy); with R > 1 (distributed) the
        shards are received in place point to point (`_gather_output_p2p`); the single-process
        simulation with R > 1 and equal query ranges uses one permuting copy ([G][R][units][rows]
        -> [G][units][R * rows]), unequal ranges per-source slice copies."""
        units, _, d = o_part.shape
        if out is None:
            out = torch.empty(self.heads, self.bpc * block_rows, d, dtype=o_part.dtype, device=o_part.device)
        # point-to-point in place: NCCL, or host tensors (gloo's send / recv take CPU tensors only;
        # the one-GPU gloo diagnostic of tools/multi_rank_check.sh keeps the all-gather below)
        if (self.replicas > 1 and is_dist() and self.world > 1 and out.is_contiguous()
                and (dist.get_backend() == "nccl" or not o_part.is_cuda)
                and os.environ.get("PBSA_GATHER_P2P", "1") != "0"):  # 0: all-gather + permute
            return self._gather_output_p2p(o_part, block_rows, out, async_op)
        mrows = self.max_q * block_rows
        send = o_part
        if o_part.shape[1] != mrows:
            send = torch.zeros(units, mrows, d, dtype=o_part.dtype, device=o_part.device)
            send[:, : o_part.shape[1]] = o_part
        equal = all(c == self.max_q for _, c in self.q_ranges)
        direct = self.replicas == 1 and equal and out.is_contiguous()
        if direct:
            flat = out.view(self.world * units, mrows, d)
        else:
            flat = torch.empty((self.world * units, mrows, d), dtype=o_part.dtype, device=o_part.device)
        recv = flat.view(self.world, units, mrows, d)

        def finish():
            if direct:
                return out
            if equal and out.is_contiguous():
                G, R = self.groups, self.replicas
                out.view(G, units, R, mrows, d).copy_(recv.view(G, R, units, mrows, d).transpose(1, 2))
                return out
            for src in range(self.world):
                g, r = divmod(src, self.replicas)
                b, c = self.q_ranges[r]
                h0 = g * self.heads_per_group
                out[h0: h0 + units, b * block_rows: (b + c) * block_rows] = recv[src, :, : c * block_rows]
            return out

        if not is_dist() or self.world == 1:
            # single process: only this rank's shard is real (tools/strong_rank_sim.py simulates one
            # rank); a real world-1 layout has one group and one replica, i.e. recv[0] is everything
            recv[self.rank if self.world > 1 else 0] = send
            return finish() if not async_op else (_Done(), finish)
        work = dist.all_gather_into_tensor(flat, send.contiguous(), async_op=async_op)
        if async_op:
            return work, finish
        return finish()
