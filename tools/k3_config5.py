#!/usr/bin/env python
"""K3 alone at the config-5 geometry (B=8 x H=40 units, 6006-block window, k = 25 %) for ncu
captures (perf experiments):  ncu -k regex:bsa_fwd ... python tools/k3_config5.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21221_b200 as pb  # noqa: E402
from tools.config_sweeps import synth_tables  # noqa: E402

U, d, b, bpc, C, Lw = int(os.environ.get("UNITS", "320")), 128, 60, 78, 156, 77
nl, nd = Lw * bpc, C + bpc
k = pb.topk_count(nl, 0.25)
S = C + nl + bpc
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(U, bpc * b, d, device="cuda", generator=g).bfloat16()
dense, local, sel = synth_tables(U, S, nd, nl, bpc, k, g)
if os.environ.get("SAMESEL"):  # experiment: both query blocks of a tile share one selection (no union)
    sel[:, 1::2] = sel[:, 0::2]
kp = torch.empty(U, S, 64, d, device="cuda", dtype=torch.bfloat16)
kp.normal_(generator=g)
kp[:, :, b:] = 0
vp = torch.empty_like(kp)
vp.normal_(generator=g)
vp[:, :, b:] = 0
reps = int(os.environ.get("REPS", "2"))
for _ in range(reps):
    pb.attention_sparse(q, kp, vp, dense, local, sel, b, validate=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
pb.attention_sparse(q, kp, vp, dense, local, sel, b, validate=False)
e1.record()
torch.cuda.synchronize()
print(f"k3 config5 ms={e0.elapsed_time(e1):.2f}")
