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


# ------------------------------------------------------------------ batch-1 query-split layout
def test_query_split_layout_partition():
    from paper_2604_21221_b200.parallel import QuerySplitLayout
    for world, groups, replicas in [(1, 1, 1), (2, 2, 1), (4, 4, 1), (8, 4, 2), (3, 3, 1), (5, 1, 5), (16, 4, 4)]:
        lays = [QuerySplitLayout(12, 78, world, r) for r in range(world)]
        assert (lays[0].groups, lays[0].replicas) == (groups, replicas)
        # every (head, query block) pair is attended exactly once
        seen = {}
        for lay in lays:
            for h in range(lay.head0, lay.head0 + lay.n_local):
                for qb in range(lay.q_begin, lay.q_begin + lay.q_count):
                    seen[(h, qb)] = seen.get((h, qb), 0) + 1
        assert len(seen) == 12 * 78 and set(seen.values()) == {1}
        # replicas of a group hold the same heads
        for lay in lays:
            assert all(lays[r].head0 == lay.head0 for r in lay.group_ranks())
    with pytest.raises(ValueError):
        QuerySplitLayout(12, 1, 8, 0)  # 1 query block cannot be split over 2 replicas


def _qs_worker(rank, world, port, q, heads=12, bpc=7, use_async=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_21221_b200.parallel import QuerySplitLayout
        b, d = 2, 4
        lay = QuerySplitLayout(heads, bpc, world, rank)
        lay.setup()
        # Q^c: this replica fills only its rows; after the gather every replica of the group holds
        # the group's full, identical Q^c (value = 1000 * head + block)
        qc = torch.full((lay.n_local, bpc, d), -1.0)
        for i in range(lay.n_local):
            for qb in range(lay.q_begin, lay.q_begin + lay.q_count):
                qc[i, qb] = 1000.0 * (lay.head0 + i) + qb
        lay.gather_qc(qc)
        want_qc = torch.tensor([[1000.0 * (lay.head0 + i) + qb for qb in range(bpc)] for i in range(lay.n_local)])
        ok_qc = torch.equal(qc[:, :, 0], want_qc) and bool((qc == qc[:, :, :1]).all())
        # O: every rank ends with all heads x all query rows
        o_part = torch.zeros(lay.n_local, lay.q_count * b, d)
        for i in range(lay.n_local):
            for r in range(lay.q_count * b):
                o_part[i, r] = 1000.0 * (lay.head0 + i) + lay.q_begin * b + r
        if use_async:
            work, finish = lay.gather_output(o_part, b, async_op=True)
            work.wait()
            full = finish()
        else:
            full = lay.gather_output(o_part, b)
        want = torch.tensor([[1000.0 * h + r for r in range(bpc * b)] for h in range(heads)])
        q.put((rank, ok_qc, torch.equal(full[:, :, 0], want)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,heads,bpc,use_async", [(2, 12, 7, False), (4, 12, 7, True), (4, 2, 8, True),
                                                      (4, 2, 7, False)])
def test_gloo_query_split_gathers(world, heads, bpc, use_async):
    """world 2 / 4 over 12 heads (R = 1: NCCL-style direct gather into the output), and 2 heads on
    4 ranks (2 groups x 2 replicas, the N = 8 shape of config 2 in miniature): equal query ranges
    (8 blocks: one permuting copy) and unequal ones (7 blocks: 4 + 3, per-source slices)."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_qs_worker, args=(r, world, port, q, heads, bpc, use_async)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok_qc and ok_o for _, ok_qc, ok_o in res), res


def _qs_replica_worker(rank, world, port, q):
    """heads = 1: one group replicated on every rank (R = world), query blocks split 7 -> 4 + 3."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_21221_b200.parallel import QuerySplitLayout
        lay = QuerySplitLayout(1, 7, world, rank)
        lay.setup()
        qc = torch.full((1, 7, 3), -1.0)
        qc[:, lay.q_begin:lay.q_begin + lay.q_count] = torch.arange(lay.q_begin, lay.q_begin + lay.q_count,
                                                                   dtype=torch.float32).view(1, -1, 1)
        lay.gather_qc(qc)
        q.put((rank, lay.replicas, qc[0, :, 0].tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_query_split_replicas_gather_identical_qc():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_qs_replica_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert [r[1] for r in res] == [2, 2]
    assert res[0][2] == res[1][2] == [float(i) for i in range(7)]
