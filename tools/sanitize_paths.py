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
torch.cuda.synchronize()
print("sanitize paths ok", mem.status(), [t.shape for t in grads])
mem.close()
