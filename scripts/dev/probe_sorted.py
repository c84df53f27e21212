"""Sort time of structured 2^28 inputs (sorted, reverse-sorted, runs) -- development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1708_09495_b200 import _lib
n = 1 << 28
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
g = torch.Generator(device='cuda'); g.manual_seed(3)
base = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device='cuda', generator=g)
srt = torch.empty_like(base)
_lib.check(L.bsg_radix_sort_u32(ctx.handle, base.data_ptr(), srt.data_ptr(), n, 8, 1, st))
inputs = {"uniform": base, "sorted": srt, "reversed": srt.flip(0).contiguous(),
          "runs4k": srt.view(-1, 4096)[torch.randperm(n // 4096, device='cuda', generator=g)].reshape(-1).contiguous()}
out = torch.empty_like(base)
for name, t in inputs.items():
    f = lambda: _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 8, 1, st))
    for _ in range(2): f()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True); ts = []
    for _ in range(5):
        s.record(); f(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    ok = bool(torch.equal(out, srt))
    print(f"rank={os.environ.get('BSG_OS_RANK','0')} {name:9s} {min(ts):.3f} ms ok={ok}", flush=True)
