import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
n = 1 << 28
keys = bsg.generate_uniform_keys(n + 4, 1)
t = torch.from_numpy(keys.view(np.int32)).cuda()
o = torch.empty_like(t)
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
for off in (0, 1):
    f = lambda: _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr() + 4 * off, o.data_ptr() + 4 * off, n, 8, 1, st))
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    print("offset", off, "words:", e0.elapsed_time(e1) / 10, "ms")
