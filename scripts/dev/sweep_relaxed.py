"""Full-sort time by n with value-stable passes on/off (development aid)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
L = _lib.lib(); ctx = _lib.context(0); st = torch.cuda.current_stream().cuda_stream
for lg in range(22, 29):
    for extra in (0,):
        n = (1 << lg) + extra
        t = torch.empty(n, dtype=torch.int32, device="cuda")
        _lib.check(L.bsg_generate_uniform_device_u32(ctx.handle, t.data_ptr(), n, bsg.derive_seed(1, 0), st))
        out = torch.empty_like(t)
        f = lambda: _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 8, 1, st))
        res = {0: [], 1: []}
        for rnd in range(5):
            for rel in (1, 0):
                L.bsg_debug_set_relaxed_passes(rel)
                for _ in range(2): f()
                torch.cuda.synchronize()
                s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
                reps = max(5, min(50, (1 << 30) // n))
                s.record()
                for _ in range(reps): f()
                e.record(); torch.cuda.synchronize()
                res[rel].append(s.elapsed_time(e) / reps)
        L.bsg_debug_set_relaxed_passes(1)
        print("2^%d relaxed %.4f strict %.4f  (%.1f%%)" % (lg, sorted(res[1])[2], sorted(res[0])[2],
              100 * (sorted(res[1])[2] / sorted(res[0])[2] - 1)), flush=True)
