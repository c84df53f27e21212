"""A/B of passes k > 0 of a full sort: value-stable ranking vs the stable K3 (development aid)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
L = _lib.lib(); ctx = _lib.context(0); st = torch.cuda.current_stream().cuda_stream
per = lambda a: a[0] / max(a[1], 1)
for n in [int(x) for x in (sys.argv[1:] or [str(1 << 28)])]:
    t = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.check(L.bsg_generate_uniform_device_u32(ctx.handle, t.data_ptr(), n, bsg.derive_seed(1, 0), st))
    out = torch.empty_like(t)
    f = lambda: _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 8, 1, st))
    res = {}
    for rnd in range(3):
        for rel in (1, 0):
            L.bsg_debug_set_relaxed_passes(rel)
            for _ in range(3): f()
            torch.cuda.synchronize()
            s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True); ts = []
            for _ in range(10):
                s.record(); f(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
            res.setdefault(rel, []).append(sorted(ts)[len(ts) // 2])
    for rel in (1, 0):
        L.bsg_debug_set_relaxed_passes(rel)
        ctx.set_timing(False); ctx.set_timing(True)
        f(); f()
        print(n, "relaxed", rel, "K3 ms/launch %.4f (%d)" % (per(ctx.kernel_time(_lib.K_ONESWEEP)), ctx.kernel_time(_lib.K_ONESWEEP)[1]),
              "K3r ms/launch %.4f (%d)" % (per(ctx.kernel_time(_lib.K_RELAXED_PASS)), ctx.kernel_time(_lib.K_RELAXED_PASS)[1]),
              "K3f ms/launch %.4f" % per(ctx.kernel_time(_lib.K_FIRST_PASS)))
    ctx.set_timing(False)
    L.bsg_debug_set_relaxed_passes(1)
    f(); torch.cuda.synchronize()
    ok = bool(torch.equal(out, torch.sort(t.view(torch.uint32).to(torch.int64))[0].to(torch.uint32).view(torch.int32))) if n <= (1 << 28) else None
    print(n, {k: ["%.4f" % x for x in v] for k, v in res.items()}, "equal torch.sort", ok, flush=True)
