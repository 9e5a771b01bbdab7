import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2604_21221_b200 as pb
g = torch.Generator(device="cuda").manual_seed(0)
for d, nl, k, mode in ((128, 1030, 257, "3"), (64, 2100, 500, "1"), (128, 1200, 100, "2"), (128, 300, 78, "0")):
    os.environ["PBSA_K2_CERT"] = mode if mode != "3" else "1"
    if mode == "3":
        os.environ.pop("PBSA_K2_CERT")
    U, nqb = 2, 5
    S = nl + 8
    qc = torch.randn(U, nqb, d, device="cuda", generator=g)
    krep = torch.randn(U, S, d, device="cuda", generator=g)
    keys = torch.stack([torch.randperm(S, device="cuda", generator=g) for _ in range(U)]).int()
    sel = pb.score_select(qc, krep, keys, 4, nl, k)
    torch.cuda.synchronize()
    print(d, nl, k, mode, "ok", sel.shape)
