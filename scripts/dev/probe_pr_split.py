"""Kernel-class time split of one in-process PR sort (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
n = int(os.environ.get("N", str(1 << 28))); p = int(os.environ.get("P", "8"))
t = bsg.generate_uniform_keys_device(n, 1); out = torch.empty_like(t)
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
for bits in (8, 16):
    f = lambda: _lib.check(L.bsg_parallel_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, p, bits, -1, None, 1, st))
    f(); torch.cuda.synchronize(); ctx.set_timing(True)
    for _ in range(3): f()
    torch.cuda.synchronize()
    res = {name: ctx.kernel_time(k) for name, k in (("onesweep", _lib.K_ONESWEEP), ("hist", _lib.K_HIST), ("pr", 3))}
    ctx.set_timing(False)
    print(bits, {k: (round(v[0] / 3, 3), v[1] // 3) for k, v in res.items()})
