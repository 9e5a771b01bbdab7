#!/usr/bin/env python
"""One steady-state PBSA chunk step inside a cudaProfilerStart/Stop range, for ncu captures of every
kernel of the step (`ncu --profile-from-start off ...`):

  python tools/prof_step.py --config 2          # Wan-1.3B layer (bench.py's workload): 4 denoise + 1 k=0 call
  python tools/prof_step.py --config 5 --calls 2  # 14B-shape batch 8 x 40 heads, 240-frame cache: the last
                                                 # denoise call + the k=0 call

The memory is filled to steady state first (untimed, outside the profiled range)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21221_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, choices=[2, 5], default=2)
ap.add_argument("--calls", type=int, default=5, help="last N calls of the chunk step are profiled")
ap.add_argument("--units", type=int, default=None)
a = ap.parse_args()
if a.config == 2:
    U, d, b, bpc, C, W, k = 12, 128, 60, 78, 156, 4, 78
else:
    U, d, b, bpc, C, W = 320, 128, 60, 78, 156, 77
    k = pb.topk_count(W * bpc, 0.25)
U = a.units or U
T = 4
mem = pb.Memory(U, C, W, bpc, b, d)
g = torch.Generator(device="cuda").manual_seed(5)
sets = [[torch.randn(U, bpc * b, d, device="cuda", generator=g).bfloat16() for _ in range(3)] for _ in range(3)]
out = torch.empty(U, bpc * b, d, device="cuda", dtype=torch.bfloat16)
i = 0
while True:  # fill (cheap k = 1 cache updates) until P and L are full
    inf = mem.info()
    if inf.n_p == C and inf.n_l == W * bpc and inf.chunks_committed > W + 2:
        break
    # fresh K/V for every filled chunk: a window built from a few repeated chunks would hold
    # identical key blocks, whose exactly tied scores pull every Top-K towards the oldest copies
    q, kk, vv = (torch.randn(U, bpc * b, d, device="cuda", generator=g).bfloat16() for _ in range(3))
    mem.attend_qkv(q, kk, vv, 1, pb.MODE_CACHE_UPDATE, out=out)
    i += 1
for j in range(T + 1):  # one warm chunk step
    q, kk, vv = sets[j % 3]
    mem.attend_qkv(q, kk, vv, k, pb.MODE_CACHE_UPDATE if j == T else pb.MODE_DENOISE, out=out)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for j in range(T + 1 - a.calls, T + 1):
    q, kk, vv = sets[j % 3]
    mem.attend_qkv(q, kk, vv, k, pb.MODE_CACHE_UPDATE if j == T else pb.MODE_DENOISE, out=out)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"profiled config {a.config}: {a.calls} calls, units {U}, k {k}, plan {pb.bsa_fwd_last_plan().schedule}")
