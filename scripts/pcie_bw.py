import torch, time
n = 1 << 30  # 4 GiB of u32
h = torch.empty(n, dtype=torch.int32, pin_memory=True)
h2 = torch.empty(n, dtype=torch.int32, pin_memory=True)
d = torch.empty(n, dtype=torch.int32, device='cuda')
d2 = torch.empty(n, dtype=torch.int32, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); return time.perf_counter() - t0
for _ in range(2):
    a = t(lambda: d.copy_(h, non_blocking=True))
    b = t(lambda: h.copy_(d, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    c = t(both)
print(f"H2D {4/a:.1f} GiB/s  D2H {4/b:.1f} GiB/s  duplex {8/c:.1f} GiB/s total")
