"""A/B of full in-process PR runs: value-stable rounds vs strictly stable (development aid)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
L = _lib.lib(); ctx = _lib.context(0); st = torch.cuda.current_stream().cuda_stream
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
t = torch.empty(n, dtype=torch.int32, device="cuda")
_lib.check(L.bsg_generate_uniform_device_u32(ctx.handle, t.data_ptr(), n, bsg.derive_seed(1, 0), st))
out = torch.empty_like(t)
exp = torch.sort(t.view(torch.uint32).to(torch.int64))[0].to(torch.uint32).view(torch.int32)
for bits in (8, 16):
    for p in (2, 8):
        f = lambda: _lib.check(L.bsg_parallel_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, p, bits, -1, None, 1, st))
        for rel in (1, 0, 1, 0):
            L.bsg_debug_set_relaxed_passes(rel)
            for _ in range(2): f()
            torch.cuda.synchronize()
            s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True); ts = []
            for _ in range(7):
                s.record(); f(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
            print("bits", bits, "p", p, "relaxed", rel, "ms %.4f" % sorted(ts)[3], "equal", bool(torch.equal(out, exp)), flush=True)
L.bsg_debug_set_relaxed_passes(1)
