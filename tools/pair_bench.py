#!/usr/bin/env python
"""Time pbsa_pair_tiles (the K3 tile pairing) at the config-2 and config-5 call shapes on K2-like
selections (block means of N(0,1) tokens, Top-K of q . k).  Perf experiment only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21221_b200 as pb  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
for name, U, nq, nl, k in (("config2", 12, 78, 312, 78), ("config5", 320, 78, 6006, 1502)):
    q = torch.randn(U, nq, 128, device="cuda", generator=g)
    kk = torch.randn(U, nl, 128, device="cuda", generator=g)
    sel = torch.topk(torch.bmm(q, kk.transpose(1, 2)), k, dim=2).indices.sort(dim=2).values.int().contiguous()
    for _ in range(3):
        pb.pair_tiles(sel, nl)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20):
        pb.pair_tiles(sel, nl)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: pair_tiles {e0.elapsed_time(e1) / 20 * 1000:.1f} us per call")
