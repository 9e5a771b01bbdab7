#!/usr/bin/env python
"""BASELINE.json config 5 as a per-chunk decode step on one B200: batch 8 x 40 heads = 320 units,
d = 128, 60-token blocks, 3-frame chunks (78 blocks), 240-frame cache = P 6 + L 231 + current 3
frames, Top-K 25 % of the window.  One step = 4 denoise + 1 cache-update PBSA call through
Memory.attend_qkv at steady state (memory filled: P = 156, L = 6006 blocks per unit).

The 2/4/8-GPU partitions of config 5 split the 320 units (batch x heads) with no data-path
exchange, so --units 160 / 80 / 40 measures the per-GPU step of N = 2 / 4 / 8 on this one GPU.
  python tools/config5_step.py [--units 320] [--steps 3]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21221_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--units", type=int, default=320)
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
U, d, b, bpc, C, W, T = a.units, 128, 60, 78, 156, 77, 4
k = pb.topk_count(W * bpc, 0.25)
mem = pb.Memory(U, C, W, bpc, b, d)
g = torch.Generator(device="cuda").manual_seed(5)
sets = [[torch.randn(U, bpc * b, d, device="cuda", generator=g).bfloat16() for _ in range(3)] for _ in range(3)]
out = torch.empty(U, bpc * b, d, device="cuda", dtype=torch.bfloat16)
i = 0
while True:  # fill: cheap k = 1 cache updates until P and L are full
    inf = mem.info()
    if inf.n_p == C and inf.n_l == W * bpc and inf.chunks_committed > W + 2:
        break
    # fresh K/V for every filled chunk: a window built from a few repeated chunks would hold
    # identical key blocks, whose exactly tied scores pull every Top-K towards the oldest copies
    q, kk, vv = (torch.randn(U, bpc * b, d, device="cuda", generator=g).bfloat16() for _ in range(3))
    mem.attend_qkv(q, kk, vv, 1, pb.MODE_CACHE_UPDATE, out=out)
    i += 1
torch.cuda.synchronize()


def step(s):
    for j in range(T + 1):
        q, kk, vv = sets[(s + j) % 3]
        mem.attend_qkv(q, kk, vv, k, pb.MODE_CACHE_UPDATE if j == T else pb.MODE_DENOISE, out=out)


step(0)
torch.cuda.synchronize()
mem.profile(True, 4096)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for s in range(a.steps):
    step(s)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
prof = mem.profile_read()
inf = mem.info()
alg_call = 4.0 * b * d * (inf.n_p + bpc + k) * b * bpc * U
print(json.dumps({"workload": "config5 step (4 denoise + 1 k=0 PBSA calls)", "units": U, "fill_chunks": i,
                  "window_blocks": inf.n_l, "persistent_blocks": inf.n_p, "top_k": k,
                  "chunk_latency_ms": ms, "alg_tflops": 5 * alg_call / ms / 1e9,
                  "stage_ms_per_step": {kk_: v / a.steps for kk_, v in prof["ms"].items()}}))
