#!/usr/bin/env python
"""Energy per config-2 chunk step (NVML total-energy counter) next to its time, for A/B variants
that can be toggled inside one process (env read per call): the K3 tile pairing on / off.  Perf
experiment only -- the question is whether the power-capped step follows energy or time."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21221_b200 as pb  # noqa: E402
import bench  # noqa: E402

import pynvml  # noqa: E402

g = bench.GEOM
U, d, b, bpc, C, W, T, k = g["heads"], g["d"], g["b"], g["bpc"], g["C"], g["W"], g["T"], g["k_top"]
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
mem = pb.Memory(U, C, W, bpc, b, d)
gen = torch.Generator(device="cuda").manual_seed(3)
sets = [[torch.randn(U, bpc * b, d, device="cuda", generator=gen).bfloat16() for _ in range(3)] for _ in range(10)]
out = torch.empty(U, bpc * b, d, device="cuda", dtype=torch.bfloat16)
while True:
    inf = mem.info()
    if inf.n_p == C and inf.n_l == W * bpc and inf.chunks_committed > W + 2:
        break
    q, kk, vv = sets[inf.chunks_committed % 10]
    mem.attend_qkv(q, kk, vv, k, pb.MODE_CACHE_UPDATE, out=out)


def steps(n):
    for s in range(n):
        for j in range(T + 1):
            q, kk, vv = sets[(s * (T + 1) + j) % 10]
            mem.attend_qkv(q, kk, vv, k, pb.MODE_CACHE_UPDATE if j == T else pb.MODE_DENOISE, out=out)


steps(5)
torch.cuda.synchronize()
n = int(os.environ.get("STEPS", "300"))
for rep in range(2):
    for name, env in (("pairing off", "0"), ("pairing on", "1")):
        os.environ["PBSA_TILE_PAIRING"] = env
        steps(3)
        torch.cuda.synchronize()
        time.sleep(0.5)
        e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        a, z = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        steps(n)
        z.record()
        torch.cuda.synchronize()
        e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        ms = a.elapsed_time(z) / n
        print(f"{name}: {ms:.3f} ms/chunk, {(e1 - e0) / n:.1f} mJ/chunk, {(e1 - e0) / (a.elapsed_time(z)):.0f} W")
