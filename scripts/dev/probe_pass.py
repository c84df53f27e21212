"""Times one 8-bit count-sort pass and a full SR4 sort at 2^28 (config/dbg via env)."""
import sys, os, faulthandler
faulthandler.dump_traceback_later(int(os.environ.get("PROBE_TO", "45")), exit=True)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
n = 1 << 28
g = torch.Generator(device='cuda'); g.manual_seed(1)
t = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device='cuda', generator=g)
keys = t.cpu().numpy().view(np.uint32)
t = t.view(torch.uint32)
out = torch.empty_like(t)
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
def timeit(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return round(min(ts), 4), round(sorted(ts)[len(ts) // 2], 4)
print("start", flush=True)
pss = timeit(lambda: _lib.check(L.bsg_count_sort_round_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 1, 8, 1, st)))
print("pass", pss, flush=True)
srt = timeit(lambda: _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 8, 1, st)))
ok = None
if os.environ.get('BSG_OS_DBG', '0') == '0':
    ok = bool(np.array_equal(out.cpu().numpy(), np.sort(keys)))
print(f"cfg={os.environ.get("BSG_OS_CFG","0")} rank={os.environ.get("BSG_OS_RANK","0")} dbg={os.environ.get('BSG_OS_DBG','0')} pass_ms={pss} sort_ms={srt} ok={ok}", flush=True)
