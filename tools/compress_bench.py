"""K1 compress_blocks alone at the config-2 Q shape (perf experiment): 12 x 4680 x 128 bf16 -> 12 x 78 x 128."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_21221_b200 as pb
x = torch.randn(12, 78, 60, 128, device="cuda").bfloat16()
for _ in range(5):
    pb.compress_blocks(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
n = 200
e0.record()
for _ in range(n):
    pb.compress_blocks(x)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / n
print(f"compress_blocks 12x4680x128: {t * 1e3:.1f} us/launch, {x.numel() * 2 / t / 1e6:.0f} GB/s")
