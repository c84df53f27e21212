import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
net = int(sys.argv[1]) if len(sys.argv) > 1 else 0
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
num, ln = 1 << 16, 4096
t = torch.randint(-2**31, 2**31 - 1, (num * ln,), dtype=torch.int32, device='cuda')
out = torch.empty_like(t)
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _lib.check(L.bsg_block_network_batched_u32(ctx.handle, net, t.data_ptr(), out.data_ptr(), num, ln, p, -1, None, 1, st))
torch.cuda.synchronize(); print("done")
