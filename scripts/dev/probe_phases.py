"""One-sweep phase breakdown (BSG_OS_DBG=8): cycles per phase summed over CTAs."""
import sys, os, ctypes
os.environ["BSG_OS_DBG"] = str(int(os.environ.get("BSG_OS_DBG", "0")) | 8)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1708_09495_b200 import _lib
n = 1 << int(os.environ.get("LGN", "28"))
t = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device='cuda')
out = torch.empty_like(t)
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
L.bsg_debug_phase_cycles.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 16)()
_lib.check(L.bsg_count_sort_round_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 1, 8, 1, st)); torch.cuda.synchronize()
L.bsg_debug_phase_cycles(buf, 1)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ctx.set_timing(True)
for _ in range(3):
    _lib.check(L.bsg_count_sort_round_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 1, 8, 1, st))
torch.cuda.synchronize()
ms, cnt = ctx.kernel_time(_lib.K_ONESWEEP)
L.bsg_debug_phase_cycles(buf, 1)
names = ["tma_wait", "count", "barrier_after_count", "scan+syncs", "rank+staging(+early count for warp 8)",
         "barrier_after_lookback", "write", "lookback walk (warp 0)"]
tot = sum(buf[:8])
ctas = min(148, (n + 8191) // 8192) * 3  # approximate for small n
print(f"kernel {ms/cnt:.3f} ms/launch; cycles per CTA per launch ~ {ms/cnt*1e-3*1.95e9:.0f}")
tot2 = sum(buf[8:16]) or 1
print(f"{'phase':40s} {'thread 0':>10s} {'thread 256':>10s}")
for i in (0, 1, 2, 3, 4, 7, 5, 6):
    print(f"{names[i]:40s} {buf[i]/tot*100:9.1f}% {buf[8+i]/tot2*100:9.1f}%")
