#!/usr/bin/env python
"""Per-CTA milestones of ONE K3 launch at the strong-scaling rank shape (perf experiment only):
global-timer stamps (start, first list built, first S seen, last P arrived, partial written, merge
start/end, exit) of every CTA, summarised as distributions relative to the earliest start.

  make trace-lib && PBSA_LIB_PATH=build/trace/libpbsa_b200.so NS=8 python tools/k3_cta_timeline.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21221_b200 as pb  # noqa: E402
from paper_2604_21221_b200 import _capi  # noqa: E402
from paper_2604_21221_b200.parallel import QuerySplitLayout  # noqa: E402
import bench  # noqa: E402

g = bench.GEOM
U, d, b, bpc, C, W, T, k_top = g["heads"], g["d"], g["b"], g["bpc"], g["C"], g["W"], g["T"], g["k_top"]
dev = torch.device("cuda", 0)
n = int(os.environ.get("NS", "8"))
qs = QuerySplitLayout(U, bpc, n, 0)
Ul, qb0, qn = qs.n_local, qs.q_begin, qs.q_count
mem = pb.Memory(Ul, C, W, bpc, b, d)
gen = torch.Generator(device=dev).manual_seed(7)
sets = [[torch.randn(Ul, (qn if i == 0 else bpc) * b, d, device=dev, generator=gen).bfloat16() for i in range(3)]
        for _ in range(4)]
out = torch.empty(Ul, qn * b, d, device=dev, dtype=torch.bfloat16)
qc_full = torch.zeros(Ul, bpc, d, device=dev, dtype=torch.float32)


def call(q, kk, vv, mode):
    if qs.replicas == 1:
        mem.attend_qkv(q, kk, vv, k_top, mode, out=out)
    else:
        mem.attend_part_ingest(q, qb0, kk, vv, qc_full)
        mem.attend_part(q, qb0, qc_full, k_top, mode, out=out)


i = 0
while True:
    inf = mem.info()
    if inf.n_p == C and inf.n_l == W * bpc and inf.chunks_committed > W + 2:
        break
    call(*sets[i % 4], pb.MODE_CACHE_UPDATE)
    i += 1
for _ in range(3):
    call(*sets[0], pb.MODE_DENOISE)
buf = torch.zeros(15 * 256 + 10 * 1024, dtype=torch.int64, device=dev)
fn = _capi.LIB.pbsa_debug_trace_buffer
fn.argtypes = [ctypes.c_void_p]
torch.cuda.synchronize()
fn(buf.data_ptr())
call(*sets[1], pb.MODE_DENOISE)
torch.cuda.synchronize()
fn(None)
plan = pb.bsa_fwd_last_plan()
grid = plan.grid
t = buf[15 * 256: 15 * 256 + 8 * grid].view(grid, 8).cpu().numpy().astype(np.int64)
smid = buf[15 * 256 + 8 * 1024: 15 * 256 + 8 * 1024 + grid].cpu().numpy()
t0 = t[:, 0].min()
rel = np.where(t > 0, t - t0, -1) / 1e3  # microseconds
names = ["start", "list_built", "first_S", "last_P", "partial_written", "merge_start", "merge_end", "exit"]
print(f"N={n} units={Ul} q_blocks={qn} grid={grid} schedule={plan.schedule} n_tiles={plan.n_tiles}")
for e, nm in enumerate(names):
    v = rel[:, e][rel[:, e] >= 0]
    if len(v):
        print(f"{nm:16s} n={len(v):4d} min {v.min():8.1f} med {np.median(v):8.1f} max {v.max():8.1f} us")
per_sm = {}
for c in range(grid):
    per_sm.setdefault(int(smid[c]), []).append(c)
dbl = sum(1 for v in per_sm.values() if len(v) > 1)
print(f"SMs used {len(per_sm)}, with 2 CTAs {dbl}")
work = rel[:, 3] - rel[:, 2]
print(f"first S -> last P per CTA: min {work.min():.1f} med {np.median(work):.1f} max {work.max():.1f} us")
lead = rel[:, 2] - rel[:, 0]
print(f"start -> first S per CTA: min {lead.min():.1f} med {np.median(lead):.1f} max {lead.max():.1f} us")
merge = rel[:, 6] - rel[:, 5]
mv = merge[(rel[:, 5] >= 0)]
if len(mv):
    print(f"merge duration: min {mv.min():.1f} med {np.median(mv):.1f} max {mv.max():.1f} us")
ep = rel[:, 4] - rel[:, 3]
print(f"last P -> partial written: med {np.median(ep[rel[:, 4] >= 0]) if (rel[:, 4] >= 0).any() else -1:.1f} us")
ent = buf[15 * 256 + 9 * 1024: 15 * 256 + 9 * 1024 + grid].cpu().numpy()
print(f"entries per CTA: min {ent.min()} med {int(np.median(ent))} max {ent.max()}")
rate = work / np.maximum(ent, 1) * 1e3
print(f"ns per entry (first S -> last P): min {rate.min():.0f} med {np.median(rate):.0f} max {rate.max():.0f}")
# SMs hosting two CTAs: per-SM total entries and the later CTA's finish time
tot = {sm: sum(int(ent[c]) for c in cs) for sm, cs in per_sm.items()}
fin = {sm: max(rel[c, 3] for c in cs) for sm, cs in per_sm.items()}
v = np.array([tot[s] for s in per_sm]); f = np.array([fin[s] for s in per_sm])
print(f"per-SM entries: min {v.min()} med {int(np.median(v))} max {v.max()}; per-SM last P: min {f.min():.1f} med {np.median(f):.1f} max {f.max():.1f}")
print("corr(per-SM entries, per-SM finish):", float(np.corrcoef(v, f)[0, 1]))
