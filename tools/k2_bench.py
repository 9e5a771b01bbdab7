#!/usr/bin/env python
"""K2 microbenchmark at the config-5 geometry (320 units, 78 query blocks, 6006-block local window,
k = 1502) and the config-2 geometry (12 units, 312-block window, k = 78; plus the k=0 pass over 546
keys with s_t).  Prints ms per launch (CUDA events, median of reps)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21221_b200 as pb  # noqa: E402


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


g = torch.Generator(device="cuda").manual_seed(0)
for name, U, nqb, nl, extra, k in (("config5", 320, 78, 6006, 234, 1502), ("config2", 12, 78, 312, 234, 78)):
    S = nl + extra
    qc = torch.randn(U, nqb, 128, device="cuda", generator=g)
    krep = torch.randn(U, S, 128, device="cuda", generator=g)
    keys = torch.stack([torch.randperm(S, device="cuda", generator=g) for _ in range(U)]).int()
    local = keys[:, :nl].contiguous()
    sels = {}
    for mode in ("0", "1"):  # exact fp64 path vs certified fp32 ranking (PBSA_K2_CERT)
        os.environ["PBSA_K2_CERT"] = mode
        ms = timeit(lambda: pb.score_select(qc, krep, local, 0, nl, k))
        sels[mode] = pb.score_select(qc, krep, local, 0, nl, k)
        print(f"{name} denoise PBSA_K2_CERT={mode}: ms={ms:.3f}")
    os.environ.pop("PBSA_K2_CERT")
    print(f"{name} selections identical: {bool(torch.equal(sels['0'], sels['1']))}")
    if len(sys.argv) > 1 and sys.argv[1] == "--full":
        ms = timeit(lambda: pb.score_select(qc, krep, keys, extra, nl, k, want_scores=True))
        print(f"{name} k=0 pass (all {S} keys + s_t): ms={ms:.3f}")
