"""Per-buffer pinned-copy rates: do some pinned 1 GiB host buffers copy slower than others? (development aid)"""
import torch, time
n = 1 << 28
d = torch.empty(n, dtype=torch.int32, device="cuda"); d2 = torch.empty(n, dtype=torch.int32, device="cuda")
bufs = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(12)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=3):
    fn(); torch.cuda.synchronize(); best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    return best
for i, h in enumerate(bufs):
    a = t(lambda: d.copy_(h, non_blocking=True)); b = t(lambda: h.copy_(d, non_blocking=True))
    print(i, "H2D %.1f GB/s  D2H %.1f GB/s" % (4 * n / a / 1e9, 4 * n / b / 1e9), flush=True)
# duplex pairs
for i in range(0, 12, 2):
    def both():
        with torch.cuda.stream(s1): d.copy_(bufs[i], non_blocking=True)
        with torch.cuda.stream(s2): bufs[i + 1].copy_(d2, non_blocking=True)
    x = t(both)
    print("pair", i, i + 1, "both %.1f GB/s (%.1f ms)" % (8 * n / x / 1e9, x * 1e3), flush=True)
# four copies at once: 2 H2D + 2 D2H on four streams
ss = [torch.cuda.Stream() for _ in range(4)]
dd = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(4)]
def four():
    with torch.cuda.stream(ss[0]): dd[0].copy_(bufs[0], non_blocking=True)
    with torch.cuda.stream(ss[1]): dd[1].copy_(bufs[1], non_blocking=True)
    with torch.cuda.stream(ss[2]): bufs[2].copy_(dd[2], non_blocking=True)
    with torch.cuda.stream(ss[3]): bufs[3].copy_(dd[3], non_blocking=True)
x = t(four)
print("2 H2D + 2 D2H at once: %.1f GB/s (%.1f ms for 4 GiB)" % (16 * n / x / 1e9, x * 1e3))
