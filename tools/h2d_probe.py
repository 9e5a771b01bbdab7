import torch, time
n = 216 * 2**20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
o_h = torch.empty(72 * 2**20, dtype=torch.uint8).pin_memory()
o_d = torch.empty(72 * 2**20, dtype=torch.uint8, device="cuda")
def bw(nstreams, chunks, reps=10, d2h=False):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        step = n // chunks
        for c in range(chunks):
            with torch.cuda.stream(ss[c % nstreams]):
                d[c*step:(c+1)*step].copy_(h[c*step:(c+1)*step], non_blocking=True)
        if d2h:
            with torch.cuda.stream(ss[-1]):
                o_h.copy_(o_d, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    return n / dt / 1e9, dt * 1e3
for ns, ch in ((1, 1), (1, 8), (2, 2), (2, 8), (4, 8), (8, 16)):
    print(ns, ch, "H2D GB/s %.1f ms %.2f" % bw(ns, ch))
for ns, ch in ((1, 1), (2, 8), (4, 8)):
    print(ns, ch, "H2D+D2H GB/s %.1f ms %.2f" % bw(ns, ch, d2h=True))
