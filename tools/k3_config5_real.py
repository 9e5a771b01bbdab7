#!/usr/bin/env python
"""K3 at config 5 on the tables a real steady-state memory produces (slot pools, dense / local
lists and the K2 selections of a denoise call) next to the synthetic tables of k3_config5.py:
time, executed blocks (union sizes) and per-unit selection overlap.  Perf experiment only.
  python tools/k3_config5_real.py [--units 320]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21221_b200 as pb  # noqa: E402
from tools.config_sweeps import synth_tables, timeit  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--units", type=int, default=320)
a = ap.parse_args()
U, d, b, bpc, C, W = a.units, 128, 60, 78, 156, 77
k = pb.topk_count(W * bpc, 0.25)
mem = pb.Memory(U, C, W, bpc, b, d)
g = torch.Generator(device="cuda").manual_seed(5)
sets = [[torch.randn(U, bpc * b, d, device="cuda", generator=g).bfloat16() for _ in range(3)] for _ in range(3)]
i = 0
while True:
    inf = mem.info()
    if inf.n_p == C and inf.n_l == W * bpc and inf.chunks_committed > W + 2:
        break
    # fresh K/V for every filled chunk: a window built from a few repeated chunks would hold
    # identical key blocks, whose exactly tied scores pull every Top-K towards the oldest copies
    q, kk, vv = (torch.randn(U, bpc * b, d, device="cuda", generator=g).bfloat16() for _ in range(3))
    mem.attend_qkv(q, kk, vv, 1, pb.MODE_CACHE_UPDATE)
    i += 1
q, kk, vv = sets[0]
mem.attend_qkv(q, kk, vv, k, pb.MODE_DENOISE)
sel, _ = mem.last_selection()
dense, local, keys, stage = mem.slot_tables()
inf = mem.info()
nd = inf.n_p + bpc
kp, vp, _ = mem.pools()
# the denoise call's own query / current chunk: K3 sees P ++ stage dense, L local
dense = dense[:, :nd].contiguous()
local = local[:, :inf.n_l].contiguous()


def union_stats(s):
    s = s.cpu()
    sizes, inter = [], 0
    for u in range(min(U, 16)):
        for t in range(0, bpc, 2):
            x, y = set(s[u, t].tolist()), set(s[u, t + 1].tolist())
            sizes.append(len(x | y))
            inter += len(x & y)
    sz = torch.tensor(sizes, dtype=torch.float32)
    # per unit: the longest tile list (a gang round waits for it)
    per_unit_max = sz.view(-1, (bpc + 1) // 2).max(1).values.mean().item()
    return round(sz.mean().item(), 1), round(inter / len(sizes), 1), round(sz.std().item(), 1), per_unit_max


ms_real = timeit(lambda: pb.attention_sparse(q, kp, vp, dense, local, sel, b, validate=False), reps=3, warm=1)
print("real tables: ms", ms_real, "plan", pb.bsa_fwd_last_plan().schedule, "union mean / intersection / union std / mean per-unit max union", union_stats(sel))
S = kp.shape[1]
sd, sl, ss = synth_tables(U, S, nd, inf.n_l, bpc, k, g)
ms_syn = timeit(lambda: pb.attention_sparse(q, kp, vp, sd, sl, ss, b, validate=False), reps=3, warm=1)
print("synthetic tables (same pools): ms", ms_syn, "union/intersection per tile", union_stats(ss))
ms_mix = timeit(lambda: pb.attention_sparse(q, kp, vp, dense, local, ss, b, validate=False), reps=3, warm=1)
print("real slot lists + synthetic selections: ms", ms_mix)
os.environ["PBSA_K3_GANG"] = "0"
print("no gangs: real %.1f ms, synthetic %.1f ms" % (
    timeit(lambda: pb.attention_sparse(q, kp, vp, dense, local, sel, b, validate=False), reps=2, warm=1),
    timeit(lambda: pb.attention_sparse(q, kp, vp, dense, local, ss, b, validate=False), reps=2, warm=1)))
del os.environ["PBSA_K3_GANG"]
# how often each local block is selected across a unit's query blocks
s0 = sel[0].flatten().cpu()
cnt = torch.bincount(s0, minlength=inf.n_l).float()
print("selection count per local block (unit 0): mean %.2f std %.2f max %d zeros %d" % (
    cnt.mean(), cnt.std(), int(cnt.max()), int((cnt == 0).sum())))


# Pairing study: union sizes when each unit's query blocks are paired greedily by largest selection
# overlap (instead of (2t, 2t + 1)): total executed list entries and the per-unit longest tile.
def greedy_pairs(s_u, n_l):
    nq = s_u.shape[0]
    bits = torch.zeros(nq, n_l, dtype=torch.float32, device=s_u.device)
    bits.scatter_(1, s_u.long(), 1.0)
    ov = bits @ bits.T  # pairwise overlaps
    ov.fill_diagonal_(-1)
    free = torch.ones(nq, dtype=torch.bool, device=s_u.device)
    pairs = []
    for _ in range(nq // 2):
        m = ov.clone()
        m[~free] = -2
        m[:, ~free] = -2
        idx = int(torch.argmax(m))
        i, j = divmod(idx, nq)
        pairs.append((i, j))
        free[i] = free[j] = False
    rest = [i for i in range(nq) if free[i]]
    return pairs, rest, ov


tot_nat, tot_greedy, mx_nat, mx_greedy = 0, 0, [], []
for u in range(16):
    s_u = sel[u]
    pairs, rest, ov = greedy_pairs(s_u, inf.n_l)
    kk = s_u.shape[1]
    nat = [2 * kk - int(ov[t, t + 1]) for t in range(0, bpc - 1, 2)]
    gr = [2 * kk - int(ov[i, j]) for i, j in pairs] + [kk for _ in rest]
    tot_nat += sum(nat)
    tot_greedy += sum(gr)
    mx_nat.append(max(nat))
    mx_greedy.append(max(gr))
print("pairing (16 units): union entries natural %d greedy %d (%.3f); mean per-unit max natural %.1f greedy %.1f" % (
    tot_nat, tot_greedy, tot_greedy / tot_nat, sum(mx_nat) / 16, sum(mx_greedy) / 16))
