"""Pinned-memory PCIe bandwidth: H2D alone, D2H alone, both at once (development aid)."""
import torch, time
n = 1 << 28  # 1 GiB of int32
h1 = torch.empty(n, dtype=torch.int32).pin_memory(); h2 = torch.empty(n, dtype=torch.int32).pin_memory()
d1 = torch.empty(n, dtype=torch.int32, device="cuda"); d2 = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    return best
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
for name, fn in (("H2D", h2d), ("D2H", d2h), ("both", both)):
    t = timed(fn)
    gb = (2 if name == "both" else 1) * n * 4 / 1e9
    print(f"{name}: {t*1e3:.1f} ms, {gb / t:.1f} GB/s")
