"""H2D/D2H bandwidth: pageable numpy vs pinned torch buffers (1 GiB)."""
import time, numpy as np, torch
n = 1 << 28
h = np.random.randint(0, 2**31, n, dtype=np.int32)
pin = torch.from_numpy(h).pin_memory()
d = torch.empty(n, dtype=torch.int32, device="cuda")
def t(f, k=3):
    f(); torch.cuda.synchronize(); ts = []
    for _ in range(k):
        a = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - a)
    return min(ts)
hp = torch.from_numpy(h)
print("pageable H2D GB/s", 4 * n / t(lambda: d.copy_(hp)) / 1e9)
print("pinned   H2D GB/s", 4 * n / t(lambda: d.copy_(pin, non_blocking=True)) / 1e9)
print("pageable D2H GB/s", 4 * n / t(lambda: hp.copy_(d)) / 1e9)
print("pinned   D2H GB/s", 4 * n / t(lambda: pin.copy_(d, non_blocking=True)) / 1e9)
a = np.empty_like(h)
print("host memcpy 1 thread GB/s", 4 * n / t(lambda: np.copyto(a, h)) / 1e9)
