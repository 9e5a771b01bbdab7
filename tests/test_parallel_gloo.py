"""The N>1 host logic on CPU with the gloo backend, world_size 2 (no GPU needed)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_21221_b200.parallel import HeadLayout, gather_units, max_over_ranks, partition_units


def test_partition_covers_every_unit_once():
    for total in [1, 12, 13, 320]:
        for world in [1, 2, 3, 4, 8]:
            seen = []
            for r in range(world):
                first, n = partition_units(total, world, r)
                seen += list(range(first, first + n))
            assert seen == list(range(total))
            sizes = [partition_units(total, world, r)[1] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        partition_units(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        total = 13
        first, n = partition_units(total, world, rank)
        local = torch.arange(first, first + n, dtype=torch.float32).reshape(n, 1).repeat(1, 3)
        full = gather_units(local, total)
        mx = max_over_ranks(10.0 + rank)
        q.put((rank, full[:, 0].tolist(), mx))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_and_max():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, full, mx in out:
        assert full == list(range(13))  # every unit once, in unit order
        assert mx == 11.0               # max over ranks


def test_head_layout_plan_single_process():
    """Every unit computed exactly once, balanced, and each batch element's heads land on one rank."""
    for batch, heads in [(1, 12), (2, 12), (4, 12), (8, 12), (8, 40), (3, 5)]:
        for world in [1, 2, 3, 4, 8]:
            lays = [HeadLayout(batch, heads, world, r) for r in range(world)]
            computed = sorted(u for l in lays for u in l.local_units)
            assert computed == list(range(batch * heads))
            sizes = [l.n_local for l in lays]
            assert max(sizes) - min(sizes) <= 1
            consumed = sorted(e for l in lays for e in l.my_batch)
            assert consumed == list(range(batch))
            for l in lays:  # what a rank receives is exactly its batch elements' heads
                assert sorted(l.recv_index) == list(range(len(l.my_batch) * heads))
                assert sum(l.recv_splits) == len(l.recv_units)
            for r, l in enumerate(lays):  # send and receive split sizes agree pairwise
                for q, m in enumerate(lays):
                    assert l.send_splits[q] == m.recv_splits[r]


def _exchange_worker(rank, world, port, q, batch, heads):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lay = HeadLayout(batch, heads, world, rank)
        # unit u's "attention output": 2 tokens x 3 channels filled with u
        o = torch.tensor(lay.local_units, dtype=torch.float32).reshape(-1, 1, 1).repeat(1, 2, 3)
        full = lay.exchange(o)
        work, finish = lay.exchange(o, async_op=True)
        work.wait()
        full2 = finish()
        q.put((rank, lay.my_batch, full[:, 0, 0].tolist(), full2[:, 0, 0].tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,batch,heads", [(2, 2, 12), (3, 3, 12), (2, 4, 5)])
def test_gloo_head_exchange(world, batch, heads):
    """Head-partitioned outputs -> every head of batch element e on rank e % world, via one
    all-to-all (the collective the GPU path runs over NCCL)."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q, batch, heads)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, my_batch, full, full2 in out:
        want = [float(e * heads + h) for e in my_batch for h in range(heads)]
        assert full == want and full2 == want
