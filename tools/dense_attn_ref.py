#!/usr/bin/env python
"""Context for K3's roofline fraction: dense bf16 attention from the libraries in this image
(torch SDPA: cuDNN / flash backends) at the config-2 shape K3 computes per call -- 12 heads x 4680
queries x 18720 visible keys (312 blocks x 60 tokens), d = 128 -- on the same box, CUDA events over
back-to-back launches.  FLOPs = 4 * n_q * n_k * d * heads (what K3's algorithmic count charges)."""
import os
import sys

import torch
import torch.nn.functional as F

H, NQ, NK, D = 12, 4680, 312 * 60, 128
flops = 4.0 * NQ * NK * D * H
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(1, H, NQ, D, device="cuda", dtype=torch.bfloat16, generator=g)
k = torch.randn(1, H, NK, D, device="cuda", dtype=torch.bfloat16, generator=g)
v = torch.randn(1, H, NK, D, device="cuda", dtype=torch.bfloat16, generator=g)
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402

for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                 ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
    try:
        with sdpa_kernel(be):
            for _ in range(3):
                F.scaled_dot_product_attention(q, k, v)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            reps = 50
            e0.record()
            for _ in range(reps):
                F.scaled_dot_product_attention(q, k, v)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            print(f"{name}: {ms:.3f} ms per call, {flops / ms / 1e9:.0f} TFLOP/s")
    except Exception as ex:  # backend unavailable for this shape / build
        print(f"{name}: unavailable ({str(ex).splitlines()[0][:100]})")
try:
    import flashinfer
    qf = q[0].transpose(0, 1).contiguous()  # [NQ, H, D]
    kf = k[0].transpose(0, 1).contiguous()
    vf = v[0].transpose(0, 1).contiguous()
    for _ in range(3):
        flashinfer.single_prefill_with_kv_cache(qf, kf, vf)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(50):
        flashinfer.single_prefill_with_kv_cache(qf, kf, vf)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    print(f"flashinfer single_prefill: {ms:.3f} ms per call, {flops / ms / 1e9:.0f} TFLOP/s")
except Exception as ex:
    print(f"flashinfer: unavailable ({str(ex).splitlines()[0][:120]})")
