"""One in-process PR sort (for ncu of the segmented one-sweep pass).  Development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
n = int(os.environ.get("N", str(1 << 28))); p = int(os.environ.get("P", "8")); bits = int(os.environ.get("BITS", "8"))
t = bsg.generate_uniform_keys_device(n, 1); out = torch.empty_like(t)
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    _lib.check(L.bsg_parallel_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, p, bits, -1, None, 1, st))
torch.cuda.synchronize(); print("done")
