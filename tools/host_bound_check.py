#!/usr/bin/env python
"""Is the per-rank chunk step host-bound?  (perf experiment)  Times rank 0's share of the
strong-scaling config-2 step (N = 1/2/4/8, no collectives) two ways: (a) back to back as the bench
runs it, (b) with the whole step sequence enqueued behind a long GPU sleep, so the device never
waits for the host -- (b) is the pure device time; (a) - (b) is host launch overhead."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21221_b200 as pb  # noqa: E402
from paper_2604_21221_b200.parallel import QuerySplitLayout  # noqa: E402
import bench  # noqa: E402

g = bench.GEOM
U, d, b, bpc, C, W, T, k_top = g["heads"], g["d"], g["b"], g["bpc"], g["C"], g["W"], g["T"], g["k_top"]
dev = torch.device("cuda", 0)
steps = int(os.environ.get("STEPS", "12"))
for n in [int(x) for x in os.environ.get("NS", "1,2,4,8").split(",")]:
    qs = QuerySplitLayout(U, bpc, n, 0)
    Ul, qb0, qn = qs.n_local, qs.q_begin, qs.q_count
    split = qs.replicas > 1
    mem = pb.Memory(Ul, C, W, bpc, b, d)
    gen = torch.Generator(device=dev).manual_seed(7)
    sets = [[torch.randn(Ul, (qn if i == 0 else bpc) * b, d, device=dev, generator=gen).bfloat16() for i in range(3)]
            for _ in range(2 * (T + 1))]
    out = torch.empty(Ul, qn * b, d, device=dev, dtype=torch.bfloat16)
    qc_full = torch.zeros(Ul, bpc, d, device=dev, dtype=torch.float32)

    exch = os.environ.get("EXCHANGE") == "1"  # also run the bench's gathers (single-process form)
    gathered = [torch.empty(U, bpc * b, d, device=dev, dtype=torch.bfloat16) for _ in range(2)]
    outs = [torch.empty_like(out) for _ in range(2)]
    ncall = [0]

    def call(q, kk, vv, mode):
        o = outs[ncall[0] & 1] if exch else out
        if not split:
            mem.attend_qkv(q, kk, vv, k_top, mode, out=o)
        else:
            mem.attend_part_ingest(q, qb0, kk, vv, qc_full)
            if exch and mode == pb.MODE_CACHE_UPDATE:
                qs.gather_qc(qc_full)
            mem.attend_part(q, qb0, qc_full, k_top, mode, out=o)
        if exch:
            work, finish = qs.gather_output(o, b, out=gathered[ncall[0] & 1], async_op=True)
            work.wait()
            finish()
        ncall[0] += 1

    i = 0
    while True:
        inf = mem.info()
        if inf.n_p == C and inf.n_l == W * bpc and inf.chunks_committed > W + 2:
            break
        call(*sets[i % len(sets)], pb.MODE_CACHE_UPDATE)
        i += 1

    def run():
        for s in range(steps):
            for j in range(T + 1):
                q, kk, vv = sets[(s * (T + 1) + j) % len(sets)]
                call(q, kk, vv, pb.MODE_CACHE_UPDATE if j == T else pb.MODE_DENOISE)

    run()
    torch.cuda.synchronize()
    res = {}
    for label in ("back_to_back", "queued_behind_sleep"):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize()
        if label == "queued_behind_sleep":
            torch.cuda._sleep(int(2e9 * steps * 5e-3))  # ~5 ms per step of head start at ~2 GHz
        t0 = time.perf_counter()
        e0.record()
        run()
        e1.record()
        t_host = time.perf_counter() - t0
        torch.cuda.synchronize()
        res[label] = (e0.elapsed_time(e1) / steps, t_host * 1e3 / steps)
    print(f"N={n}: device ms/chunk back-to-back {res['back_to_back'][0]:.3f}, queued {res['queued_behind_sleep'][0]:.3f}; "
          f"host enqueue ms/chunk {res['back_to_back'][1]:.3f}", flush=True)
    del mem
