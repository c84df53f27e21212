"""Quick GPU timing probe (development aid, not the bench contract)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib

def timeit(fn, reps=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return min(ts), sorted(ts)[len(ts)//2]

n = 1 << 28
keys = bsg.generate_uniform_keys(n, 1)
t = torch.from_numpy(keys.view(np.int32)).cuda().view(torch.uint32)
out = torch.empty_like(t)
ctx = _lib.context(0)
L = _lib.lib()
st = torch.cuda.current_stream().cuda_stream
def sort8():
    _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 8, 1, st))
def pass8():
    _lib.check(L.bsg_count_sort_round_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 1, 8, 1, st))
res = {}
res['sort_r256_ms'] = timeit(sort8)
res['pass_r256_ms'] = timeit(pass8)
ti = t.view(torch.int32)
res['torch_sort_int32_ms'] = timeit(lambda: torch.sort(ti))
res['copy_ms'] = timeit(lambda: out.copy_(t))
torch.cuda.synchronize()
o = out.cpu().numpy(); sort8(); torch.cuda.synchronize(); ok = bool((out.cpu().numpy() == np.sort(keys)).all())
res['sorted_ok'] = ok
for k, v in res.items():
    print(k, v)
gb = n * 4 * 2 / 1e9
print('pass GB/s', gb / (res['pass_r256_ms'][0] / 1e3), 'sort Gkeys/s', n / res['sort_r256_ms'][0] / 1e6)
# batched networks
A = 1 << 16; ln = 4096
arr = torch.from_numpy(bsg.generate_uniform_keys(A * ln, 7).view(np.int32)).cuda().view(torch.uint32)
o2 = torch.empty_like(arr)
for net in (0, 1):
    for p in (2, 4, 8):
        f = lambda: _lib.check(L.bsg_block_network_batched_u32(ctx.handle, net, arr.data_ptr(), o2.data_ptr(), A, ln, p, -1, None, 1, st))
        print('net', net, 'p', p, timeit(f, reps=5))
