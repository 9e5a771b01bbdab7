"""Per-call device time of config-2 denoise calls (no profiling events) and the per-stage split
(profiling events, which break the programmatic-launch overlap between stages) -- A/B harness for
launch-sequence changes (perf experiment): run it once per variant (env switch or build).  Round 2
used it to measure the chunk's K/V ingest on a second stream, concurrent with Q compression + K2:
0.586 vs 0.585 ms per call -- no gain (the programmatic-launch overlap into K3 is lost), dropped."""
import os, sys, torch
sys.path.insert(0, "/root/repo")
import paper_2604_21221_b200 as pb
import bench
g = bench.GEOM
U, d, b, bpc, C, W, T, k_top = g["heads"], g["d"], g["b"], g["bpc"], g["C"], g["W"], g["T"], g["k_top"]
dev = torch.device("cuda", 0)
mem = pb.Memory(U, C, W, bpc, b, d)
gen = torch.Generator(device=dev).manual_seed(7)
sets = [[torch.randn(U, bpc * b, d, device=dev, generator=gen).bfloat16() for i in range(3)] for _ in range(4)]
out = torch.empty(U, bpc * b, d, device=dev, dtype=torch.bfloat16)
i = 0
while True:
    inf = mem.info()
    if inf.n_p == C and inf.n_l == W * bpc and inf.chunks_committed > W + 2:
        break
    mem.attend_qkv(*sets[i % 4], k_top, pb.MODE_CACHE_UPDATE, out=out); i += 1
for _ in range(5):
    mem.attend_qkv(*sets[0], k_top, pb.MODE_DENOISE, out=out)
torch.cuda.synchronize()
n = 40
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for j in range(n):
    mem.attend_qkv(*sets[j % 4], k_top, pb.MODE_DENOISE, out=out)
e1.record()
torch.cuda.synchronize()
plain = e0.elapsed_time(e1) / n
mem.profile(True, max_calls=n + 2)
e0.record()
for j in range(n):
    mem.attend_qkv(*sets[j % 4], k_top, pb.MODE_DENOISE, out=out)
e1.record()
torch.cuda.synchronize()
pr = mem.profile_read()
print("per call ms %.4f (profiled %.4f)" % (plain, e0.elapsed_time(e1) / n), {k: round(v / n * 1e3, 1) for k, v in pr["ms"].items()}, "us/call")
