#!/usr/bin/env python
"""A/B of the config-2 chunk step without per-stage profiling events (perf experiments):
   PBSA_PDL=0|1 python tools/step_ab.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21221_b200 as pb  # noqa: E402

U, d, b, bpc, C, W, T, k = 12, 128, 60, 78, 156, 4, 4, 78
mem = pb.Memory(U, C, W, bpc, b, d)
g = torch.Generator(device="cuda").manual_seed(0)
sets = [[torch.randn(U, bpc * b, d, device="cuda", generator=g).bfloat16() for _ in range(3)] for _ in range(10)]
out = torch.empty(U, bpc * b, d, device="cuda", dtype=torch.bfloat16)
for i in range(12):
    q, kk, vv = sets[i % 10]
    mem.attend_qkv(q, kk, vv, k, pb.MODE_CACHE_UPDATE, out=out)


def step(i):
    for j in range(T + 1):
        q, kk, vv = sets[(i * 5 + j) % 10]
        mem.attend_qkv(q, kk, vv, k, pb.MODE_CACHE_UPDATE if j == T else pb.MODE_DENOISE, out=out)


for i in range(5):
    step(i)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
n = 50
e0.record()
for i in range(n):
    step(i)
e1.record()
torch.cuda.synchronize()
print(f"PBSA_PDL={os.environ.get('PBSA_PDL', '1')} ms/step={e0.elapsed_time(e1) / n:.4f}")
