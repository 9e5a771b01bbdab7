#!/usr/bin/env python
"""Small end-to-end exercise of every entry point for compute-sanitizer (perf-irrelevant sizes):
  compute-sanitizer --tool memcheck python tools/sanitize_paths.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21221_b200 as pb  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
U, C, W, bpc, b, d = 2, 12, 2, 6, 60, 128
mem = pb.Memory(U, C, W, bpc, b, d)
for c in range(6):  # device path, both modes
    q, k, v = (torch.randn(U, bpc * b, d, device="cuda", generator=g).bfloat16() for _ in range(3))
    mem.attend_qkv(q, k, v, 3, pb.MODE_DENOISE)
    mem.attend_qkv(q, k, v, 3, pb.MODE_CACHE_UPDATE)
hq = [torch.randn(U, bpc * b, d, generator=torch.Generator().manual_seed(i)).bfloat16().pin_memory() for i in range(3)]
outs = [mem.attend_qkv_host(*hq, 3, pb.MODE_DENOISE) for _ in range(3)]  # host path
mem.host_sync()
# standalone attention forward + backward
S, nd, nl, kk, nqb = 40, 10, 24, 5, 6
kp = torch.zeros(U, S, 64, d, device="cuda", dtype=torch.bfloat16)
vp = torch.zeros_like(kp)
kp[:, :, :b] = torch.randn(U, S, b, d, device="cuda", generator=g).bfloat16()
vp[:, :, :b] = torch.randn(U, S, b, d, device="cuda", generator=g).bfloat16()
q = torch.randn(U, nqb * b, d, device="cuda", generator=g).bfloat16()
do = torch.randn_like(q)
perm = torch.stack([torch.randperm(S, device="cuda", generator=g) for _ in range(U)]).int()
dense, local = perm[:, :nd].contiguous(), perm[:, nd:nd + nl].contiguous()
sel = torch.stack([torch.stack([torch.randperm(nl, device="cuda", generator=g)[:kk].sort().values
                                for _ in range(nqb)]) for _ in range(U)]).int().contiguous()
o, lse = pb.attention_sparse(q, kp, vp, dense, local, sel, b, want_lse=True)
grads = pb.attention_sparse_backward(q, kp, vp, dense, local, sel, b, o, lse, do)
# unit-gang K3 schedule (forced) and a 16-bit-list launch
os.environ["PBSA_K3_GANG"] = "1"
pb.attention_sparse(q, kp, vp, dense, local, sel, b, validate=False)
# 40 units x 17 query blocks: 32 full gangs of 9 tiles + the extra gang (8 members, two tiles each)
U2, nqb2 = 40, 17
kp2 = torch.zeros(U2, S, 64, d, device="cuda", dtype=torch.bfloat16)
vp2 = torch.zeros_like(kp2)
kp2[:, :, :b] = torch.randn(U2, S, b, d, device="cuda", generator=g).bfloat16()
vp2[:, :, :b] = torch.randn(U2, S, b, d, device="cuda", generator=g).bfloat16()
q2 = torch.randn(U2, nqb2 * b, d, device="cuda", generator=g).bfloat16()
perm2 = torch.stack([torch.randperm(S, device="cuda", generator=g) for _ in range(U2)]).int()
sel2 = torch.stack([torch.stack([torch.randperm(nl, device="cuda", generator=g)[:kk].sort().values
                                 for _ in range(nqb2)]) for _ in range(U2)]).int().contiguous()
pb.attention_sparse(q2, kp2, vp2, perm2[:, :nd].contiguous(), perm2[:, nd:nd + nl].contiguous(), sel2, b,
                    validate=False)
del os.environ["PBSA_K3_GANG"]
# query-split calls (2 replicas of the same heads) and the drop-sink fault path of K4
parts = [pb.Memory(U, C, W, bpc, b, d) for _ in range(2)]
qc = [torch.zeros(U, bpc, d, device="cuda") for _ in range(2)]
for c in range(5):
    q6, k6, v6 = (torch.randn(U, bpc * b, d, device="cuda", generator=g).bfloat16() for _ in range(3))
    for mode in (pb.MODE_DENOISE, pb.MODE_CACHE_UPDATE):
        for r, (qb, qn) in enumerate(((0, 3), (3, 3))):
            qp = q6.view(U, bpc, b, d)[:, qb:qb + qn].reshape(U, qn * b, d).contiguous()
            parts[r].attend_part_ingest(qp, qb, k6, v6, qc[r])
        qc[0][:, 3:] = qc[1][:, 3:]
        qc[1][:, :3] = qc[0][:, :3]
        for r, (qb, qn) in enumerate(((0, 3), (3, 3))):
            qp = q6.view(U, bpc, b, d)[:, qb:qb + qn].reshape(U, qn * b, d).contiguous()
            parts[r].attend_part(qp, qb, qc[r], 3, mode)
pb.debug_set_fault("drop-sink")
for c in range(4):
    q6, k6, v6 = (torch.randn(U, bpc * b, d, device="cuda", generator=g).bfloat16() for _ in range(3))
    parts[0].attend_qkv(q6, k6, v6, 3, pb.MODE_CACHE_UPDATE)
pb.debug_set_fault(None)
# SPEC-op primitives
a = torch.randn(37, 129, device="cuda", generator=g)
bm = torch.randn(129, 41, device="cuda", generator=g)
pb.matmul(a, bm)
pb.matmul(a, bm.t().contiguous(), transpose_b=True)
sm = pb.masked_softmax_rows(a)
pb.aggregate_scores(sm)
pb.select_topk(sm, 17)
lat = torch.randn(3, 30, 52, 8, device="cuda", generator=g)
pb.unblockify(pb.blockify(lat, (1, 15, 4)), lat.shape, (1, 15, 4))
pb.topc_select(torch.arange(40, device="cuda"), torch.rand(40, device="cuda", generator=g), 13)
# K3 tile pairing: standalone, and inside attend (forced for these short windows)
selp = torch.stack([torch.stack([torch.randperm(40, device="cuda", generator=g)[:9].sort().values
                                 for _ in range(7)]) for _ in range(2)]).int().contiguous()
pb.pair_tiles(selp, 40)
os.environ["PBSA_TILE_PAIRING"] = "1"
for c in range(3):
    q6, k6, v6 = (torch.randn(U, bpc * b, d, device="cuda", generator=g).bfloat16() for _ in range(3))
    parts[1].attend_qkv(q6, k6, v6, 3, pb.MODE_DENOISE if c % 2 else pb.MODE_CACHE_UPDATE)
del os.environ["PBSA_TILE_PAIRING"]
torch.cuda.synchronize()
print("sanitize paths ok", mem.status(), [t.shape for t in grads])
for m in [mem] + parts:
    m.close()
