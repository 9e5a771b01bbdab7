"""The N>1 host logic on CPU with the gloo backend, world_size 2 (no GPU needed)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_21221_b200.parallel import gather_units, max_over_ranks, partition_units


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
