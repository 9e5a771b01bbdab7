#!/usr/bin/env python
"""Handshake timeline of the dK/dV backward kernel (CTA 0, first 256 entries): clock64 stamps of the
MMA issuer and of elementwise warp 2.  Perf experiment only (pbsa_debug_bwd_trace_buffer).

  make trace-lib && PBSA_LIB_PATH=build/trace/libpbsa_b200.so python tools/bwd_timeline.py"""
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
do = torch.randn(U, nqb * b, d, device="cuda", generator=g).bfloat16()
perm = torch.stack([torch.randperm(S, device="cuda", generator=g) for _ in range(U)]).int()
dense, local = perm[:, :nd].contiguous(), perm[:, nd:nd + nl].contiguous()
sel = torch.stack([torch.stack([torch.randperm(nl, device="cuda", generator=g)[:k].sort().values
                                for _ in range(nqb)]) for _ in range(U)]).int().contiguous()
args = (q, kp, vp, dense, local, sel, b)
o, lse = pb.attention_sparse(*args, want_lse=True, validate=False)
buf = torch.zeros(10 * 256, dtype=torch.int64, device="cuda")
fn = _capi.LIB.pbsa_debug_bwd_trace_buffer
fn.argtypes = [ctypes.c_void_p]
for _ in range(2):
    pb.attention_sparse_backward(*args, o, lse, do)
fn(buf.data_ptr())
pb.attention_sparse_backward(*args, o, lse, do)
torch.cuda.synchronize()
fn(None)
t = buf.view(10, 256).cpu().numpy().astype("int64")
n = int((t[6] > 0).sum())
r = slice(4, min(n, 250))
r1 = slice(5, min(n, 251))
med = lambda x: int(np.median(x))  # noqa: E731
print("entries traced:", n)
print("median period (P arrivals):", med(np.diff(t[6, 4:min(n, 250)])))
print("median S_j issue (pre -> issued):", med(t[1, r] - t[0, r]))
print("median S_j issued -> S_j seen by elementwise:", med(t[5, r] - t[1, r]))
print("median elementwise compute (S seen -> P arrive):", med(t[6, r] - t[5, r]))
print("median elementwise wait for S:", med(t[5, r] - t[4, r]))
print("median P_j arrive -> MMA sees P_j:", med(t[2, r] - t[6, r]))
print("median dV/dK issue (P seen -> issued):", med(t[3, r] - t[2, r]))
print("median MMA: dV/dK_{j-1} issued -> Q_{j+1} present (next S):", med(t[0, r1] - t[3, r]))
f = int((t[9] > 0).sum())
if f:
    print("fragments traced:", f, " median acc wait:", med(t[8, :f] - t[7, :f]),
          " median epilogue:", med(t[9, :f] - t[8, :f]))
