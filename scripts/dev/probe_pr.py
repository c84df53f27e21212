"""In-process PR timing at one (n, p, radix) (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
n = 1 << int(os.environ.get("LGN", "26")); p = int(os.environ.get("P", "2")); bits = int(os.environ.get("BITS", "8"))
keys = bsg.generate_uniform_keys(n, 1)
t = torch.from_numpy(keys.view(np.int32)).cuda(); o = torch.empty_like(t)
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
f = lambda: _lib.check(L.bsg_parallel_radix_sort_u32(ctx.handle, t.data_ptr(), o.data_ptr(), n, p, bits, -1, None, 1, st))
for _ in range(int(os.environ.get("REPS", "5"))): f()
torch.cuda.synchronize(); print("done")
