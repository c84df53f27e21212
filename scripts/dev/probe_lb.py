"""Look-back statistics of one 2^28-key pass (needs a build with -DBSG_LB_STATS=1)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1708_09495_b200 import _lib
n = 1 << int(os.environ.get("LGN", "28"))
t = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device='cuda')
out = torch.empty_like(t)
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
buf = (ctypes.c_ulonglong * 4)()
for _ in range(2):
    _lib.check(L.bsg_count_sort_round_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 1, 8, 1, st))
torch.cuda.synchronize()
L.bsg_debug_lb_stats(buf, 1)
for _ in range(3):
    _lib.check(L.bsg_count_sort_round_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 1, 8, 1, st))
torch.cuda.synchronize()
L.bsg_debug_lb_stats(buf, 1)
w = max(buf[3], 1)
print(f"{os.environ.get('BSG_LIB','default')}: per look-back warp-tile: rounds {buf[0]/w:.2f}, predecessors {buf[1]/w:.2f}, unpublished stops {buf[2]/w:.2f} (warp-tiles {w})")
