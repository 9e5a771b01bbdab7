#!/usr/bin/env python
"""Handshake timeline of the paired-block K3 variant (CTA 0, per key-block PAIR): clock64 stamps of
the MMA issuer and of one warp of each softmax group.  Perf experiment only.

  make trace-lib && PBSA_K3_PAIR=1 PBSA_LIB_PATH=build/trace/libpbsa_b200.so python tools/k3_pair_timeline.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21221_b200 as pb  # noqa: E402
from paper_2604_21221_b200 import _capi  # noqa: E402

U, nqb, b, d, S, nd, nl, k = 12, 78, 60, 128, 546, 234, 312, 78
g = torch.Generator(device="cuda").manual_seed(0)
kp = torch.zeros(U, S, 64, d, device="cuda", dtype=torch.bfloat16)
vp = torch.zeros_like(kp)
kp[:, :, :b] = torch.randn(U, S, b, d, device="cuda", generator=g).bfloat16()
vp[:, :, :b] = torch.randn(U, S, b, d, device="cuda", generator=g).bfloat16()
q = torch.randn(U, nqb * b, d, device="cuda", generator=g).bfloat16()
perm = torch.stack([torch.randperm(S, device="cuda", generator=g) for _ in range(U)]).int()
dense, local = perm[:, :nd].contiguous(), perm[:, nd:nd + nl].contiguous()
sel = torch.stack([torch.stack([torch.randperm(nl, device="cuda", generator=g)[:k].sort().values
                                for _ in range(nqb)]) for _ in range(U)]).int().contiguous()
buf = torch.zeros(15 * 256 + 16 * 1024, dtype=torch.int64, device="cuda")
fn = _capi.LIB.pbsa_debug_trace_buffer
fn.argtypes = [ctypes.c_void_p]
for _ in range(2):
    pb.attention_sparse(q, kp, vp, dense, local, sel, b, validate=False)
fn(buf.data_ptr())
pb.attention_sparse(q, kp, vp, dense, local, sel, b, validate=False)
torch.cuda.synchronize()
fn(None)
t = buf[:15 * 256].view(15, 256).cpu().numpy().astype("int64")
lo, hi = 10, 150
med = lambda x: int(np.median(x))  # noqa: E731
print("median period per pair (group A P arrivals):", med(np.diff(t[6, lo:hi])))
print("median period per pair (group B P arrivals):", med(np.diff(t[9, lo:hi])))
print("A: wait for S:", med(t[5, lo:hi] - t[4, lo:hi]), " softmax (S seen -> P arrive):", med(t[6, lo:hi] - t[5, lo:hi]))
print("B: wait for S:", med(t[8, lo:hi] - t[7, lo:hi]), " softmax (S seen -> P arrive):", med(t[9, lo:hi] - t[8, lo:hi]))
print("B P arrive - A P arrive:", med(t[9, lo:hi] - t[6, lo:hi]))
print("MMA: issue of S_{pg+1} (pre -> issued):", med(t[1, lo:hi] - t[0, lo:hi]))
print("MMA: P_a seen - A arrival:", med(t[2, lo:hi] - t[6, lo:hi]), " P_b seen - B arrival:", med(t[11, lo:hi] - t[9, lo:hi]))
print("MMA: PV_a issue:", med(t[3, lo:hi] - t[2, lo:hi]), " PV_b issue:", med(t[12, lo:hi] - t[11, lo:hi]))
print("S_{pg+1} issued -> A sees it:", med(t[5, lo + 1:hi + 1] - t[1, lo:hi]))
print("MMA: (S_{pg+1} issued) - (A P_pg arrival):", med(t[1, lo:hi] - t[6, lo:hi]))
