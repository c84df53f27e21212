"""One SR4 sort of config 3's Zipf(1.1) 2^28 keys (for ncu: histogram contention,
rank-first skew passes).  Development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
kind = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = 1 << 28
keys = bsg.generate_skewed_keys(n, bsg.derive_seed(1, 0), kind, 1.1)
t = torch.from_numpy(keys.view(np.int32)).cuda(); o = torch.empty_like(t)
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), o.data_ptr(), n, 8, 1, st))
torch.cuda.synchronize(); print("done")
