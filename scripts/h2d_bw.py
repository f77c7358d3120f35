import torch, time
n = 4_200_000_000
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); a = time.perf_counter(); fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - a)
    return best
one = t(lambda: d.copy_(h, non_blocking=True))
print(f"one copy: {n/one/1e9:.1f} GB/s ({one*1e3:.1f} ms)")
for chunk_mb in (32, 96, 256):
    c = chunk_mb << 20
    def chunks():
        for o in range(0, n, c):
            d[o:o+c].copy_(h[o:o+c], non_blocking=True)
    tt = t(chunks)
    print(f"{chunk_mb} MB chunks: {n/tt/1e9:.1f} GB/s ({tt*1e3:.1f} ms)")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def two():
    half = n // 2
    with torch.cuda.stream(s1): d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2): d[half:].copy_(h[half:], non_blocking=True)
tt = t(two)
print(f"two streams: {n/tt/1e9:.1f} GB/s ({tt*1e3:.1f} ms)")
