#!/usr/bin/env python
"""PBSA backward at the config-2 geometry (12 heads, 78 query blocks of 60, 234 dense + top-78 of
312 local blocks): ms per backward call and TFLOP/s on the algorithmic backward FLOPs (5 GEMMs of
2*b*b*d per visible (query block, key block) pair: S, dP, dQ, dK, dV); the forward beside it."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21221_b200 as pb  # noqa: E402

U, nqb, b, d, S, nd, nl, k = 12, 78, 60, 128, 546, 234, 312, 78
g = torch.Generator(device="cuda").manual_seed(0)
kp = torch.zeros(U, S, 64, d, device="cuda", dtype=torch.bfloat16)
vp = torch.zeros_like(kp)
kp[:, :, :b] = torch.randn(U, S, b, d, device="cuda", generator=g).bfloat16()
vp[:, :, :b] = torch.randn(U, S, b, d, device="cuda", generator=g).bfloat16()
q = torch.randn(U, nqb * b, d, device="cuda", generator=g).bfloat16()
do = torch.randn(U, nqb * b, d, device="cuda", generator=g).bfloat16()
perm = torch.stack([torch.randperm(S, device="cuda", generator=g) for _ in range(U)]).int()
dense, local = perm[:, :nd].contiguous(), perm[:, nd:nd + nl].contiguous()
sel = torch.stack([torch.stack([torch.randperm(nl, device="cuda", generator=g)[:k].sort().values
                                for _ in range(nqb)]) for _ in range(U)]).int().contiguous()
args = (q, kp, vp, dense, local, sel, b)


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


o, lse = pb.attention_sparse(*args, want_lse=True, validate=False)
ms_f = timeit(lambda: pb.attention_sparse(*args, want_lse=True, validate=False))
ms_b = timeit(lambda: pb.attention_sparse_backward(*args, o, lse, do))
pairs = nqb * U * (nd + k)  # visible (query block, key block) pairs
fwd = 2 * 2.0 * b * b * d * pairs
bwd = 5 * 2.0 * b * b * d * pairs
print(f"config2 forward ms={ms_f:.3f} ({fwd / ms_f / 1e9:.0f} TFLOP/s)  backward ms={ms_b:.3f} "
      f"({bwd / ms_b / 1e9:.0f} TFLOP/s alg, bwd/fwd time {ms_b / ms_f:.2f}x)")
