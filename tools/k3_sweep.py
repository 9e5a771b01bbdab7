#!/usr/bin/env python
"""K3 microbenchmark at the config-2 geometry (12 heads, 78 query blocks of 60, 546-slot pools,
234 dense + top-78 of 312 local blocks).  Prints ms / launch and TFLOP/s (algorithmic and executed).
PBSA_ABLATE=1 makes the softmax warps skip their math (pipeline / tensor-core upper bound)."""
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21221_b200 as pb  # noqa: E402

U, nqb, b, d, S, nd, nl, k = 12, 78, 60, 128, 546, 234, 312, 78
U, nqb = int(os.environ.get("U", U)), int(os.environ.get("NQB", nqb))  # e.g. U=3 NQB=39: one rank of N=8
g = torch.Generator(device="cuda").manual_seed(0)
kp = torch.zeros(U, S, 64, d, device="cuda", dtype=torch.bfloat16)
vp = torch.zeros_like(kp)
kp[:, :, :b] = torch.randn(U, S, b, d, device="cuda", generator=g).bfloat16()
vp[:, :, :b] = torch.randn(U, S, b, d, device="cuda", generator=g).bfloat16()
q = torch.randn(U, nqb * b, d, device="cuda", generator=g).bfloat16()
perm = torch.stack([torch.randperm(S, device="cuda", generator=g) for _ in range(U)]).int()
if os.environ.get("SEQ_SLOTS"):  # dense = slots [0, nd), local = [nd, nd + nl) in order (a Memory's layout)
    perm = torch.arange(S, device="cuda", dtype=torch.int32).repeat(U, 1)
dense = perm[:, :nd].contiguous()
local = perm[:, nd:nd + nl].contiguous()
sel = torch.stack([torch.stack([torch.randperm(nl, device="cuda", generator=g)[:k].sort().values
                                for _ in range(nqb)]) for _ in range(U)]).int().contiguous()
alg = 4.0 * b * d * (nd + k) * b * nqb * U
un = 0
sc = sel.cpu()
for u in range(U):
    for t in range(0, nqb, 2):
        un += nd + len(set(sc[u, t].tolist()) | (set(sc[u, t + 1].tolist()) if t + 1 < nqb else set()))
exe = 4.0 * 128 * 64 * d * un
for sk in ((True,) if os.environ.get("PBSA_SWEEP_SK_ONLY") else (True, False)):
    for _ in range(3):
        pb.attention_sparse(q, kp, vp, dense, local, sel, b, stream_k=sk, validate=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    reps = int(os.environ.get("REPS", 20))
    clk, pw = [], []
    stop = threading.Event()

    def sample():  # SM clock under load (power capping shows here, not in the max clock)
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        while not stop.is_set():
            clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
            time.sleep(0.002)

    th = threading.Thread(target=sample)
    th.start()
    gap = int(os.environ.get("GAP_CYCLES", 0))  # idle gap between launches (power / clock study)
    if gap:
        ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(reps)]
        for a, z in ev:
            torch.cuda._sleep(gap)
            a.record()
            pb.attention_sparse(q, kp, vp, dense, local, sel, b, stream_k=sk, validate=False)
            z.record()
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(z) for a, z in ev)[reps // 2]
    else:
        e0.record()
        for _ in range(reps):
            pb.attention_sparse(q, kp, vp, dense, local, sel, b, stream_k=sk, validate=False)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
    stop.set()
    th.join()
    print(f"ablate={os.environ.get('PBSA_ABLATE', '0')} stream_k={sk} ms={ms:.4f} alg_TFLOPs={alg / ms / 1e9:.1f} "
          f"exec_TFLOPs={exe / ms / 1e9:.1f} exec/alg={exe / alg:.3f} "
          f"sm_mhz_median={sorted(clk)[len(clk) // 2] if clk else 0} "
          f"power_w_median={sorted(pw)[len(pw) // 2] if pw else 0:.0f}")
