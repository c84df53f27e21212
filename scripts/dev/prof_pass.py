"""Runs a few 2^28-key count-sort passes and sorts (profiling target)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
what = sys.argv[2] if len(sys.argv) > 2 else "pass"
keys = bsg.generate_uniform_keys(n, 1)
t = torch.from_numpy(keys.view(np.int32)).cuda().view(torch.uint32)
out = torch.empty_like(t)
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    if what == "pass":
        _lib.check(L.bsg_count_sort_round_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 1, 8, 1, st))
    else:
        _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 8, 1, st))
torch.cuda.synchronize()
print("done")
