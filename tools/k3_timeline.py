#!/usr/bin/env python
"""Handshake timeline of K3 (CTA 0, first 256 blocks): clock64 stamps of the MMA issuer and of
softmax warp 2, printed as per-block deltas.  Perf experiment only (pbsa_debug_trace_buffer).

  make trace-lib && PBSA_LIB_PATH=build/trace/libpbsa_b200.so python tools/k3_timeline.py"""
import ctypes
import os
import sys

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
buf = torch.zeros(15 * 256, dtype=torch.int64, device="cuda")
fn = _capi.LIB.pbsa_debug_trace_buffer
fn.argtypes = [ctypes.c_void_p]
for _ in range(2):
    pb.attention_sparse(q, kp, vp, dense, local, sel, b, validate=False)
fn(buf.data_ptr())
pb.attention_sparse(q, kp, vp, dense, local, sel, b, validate=False)
torch.cuda.synchronize()
fn(None)
t = buf.view(15, 256).cpu().numpy().astype("int64")
names = ["mma_pre_S", "mma_S_issued", "mma_P_seen", "mma_PV_issued", "sm_wait_S", "sm_S_seen", "sm_P_arrive",
         "sm_S_regs", "sm_exps", "sm_P_ready", "sm_P_stored", "w2_arr", "w3_arr", "w4_arr", "w5_arr"]
t0 = t[4, 0]
print("j  " + " ".join(f"{n:>13s}" for n in names) + "  period")
for j in range(0, 0):
    row = t[:, j] - t0
    per = t[6, j] - t[6, j - 1] if j else 0
    print(f"{j:3d} " + " ".join(f"{v:13d}" for v in row) + f"  {per:6d}")
import numpy as np
per = np.diff(t[6, 10:200])
print("median period (cycles per block, CTA 0):", int(np.median(per)))
print("median S-issue -> S-seen:", int(np.median(t[5, 11:200] - t[1, 10:199])))
print("median P-arrive -> MMA sees P:", int(np.median(t[2, 10:200] - t[6, 10:200])))
print("median softmax compute (S seen -> P arrive):", int(np.median(t[6, 10:200] - t[5, 10:200])))
print("median softmax wait for S:", int(np.median(t[5, 10:200] - t[4, 10:200])))
for a, b, what in ((5, 7, "S seen -> S in regs (LDTM)"), (7, 8, "exps + packs + sums"),
                   (8, 9, "overflow check"), (9, 10, "STTM + wait"), (10, 6, "fence + arrive"),
                   (11, 12, "warp3 - warp2 arrival"), (11, 13, "warp4 - warp2 arrival"),
                   (11, 14, "warp5 - warp2 arrival"), (11, 2, "warp2 arrival -> MMA sees P")):
    print(f"median {what}:", int(np.median(t[b, 10:200] - t[a, 10:200])))
print("median (S_{j+1} issued) - (P_j arrival):", int(np.median(t[1, 10:200] - t[6, 10:200])))
print("median (MMA sees P_j) - (S_{j+1} issued):", int(np.median(t[2, 10:200] - t[1, 10:200])))
print("median (S_{j+1} issue start) - (P_j arrival):", int(np.median(t[0, 10:200] - t[6, 10:200])))
print("median PV_j issued - MMA sees P_j:", int(np.median(t[3, 10:200] - t[2, 10:200])))
print("median S_{j+1} issue duration (pre_S -> S_issued):", int(np.median(t[1, 10:200] - t[0, 10:200])))
