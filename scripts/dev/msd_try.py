"""Hybrid route (msd.cu) vs the LSD sort: correctness and per-class times (development aid)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
L = _lib.lib(); ctx = _lib.context(0); st = torch.cuda.current_stream().cuda_stream
per = lambda a: a[0] / max(a[1], 1)
sizes = [int(x) for x in sys.argv[1:]] or [5, 100003, 1 << 20, (1 << 24) + 7, 1 << 26, 1 << 28]
for n in sizes:
    t = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.check(L.bsg_generate_uniform_device_u32(ctx.handle, t.data_ptr(), n, bsg.derive_seed(1, 0), st))
    exp = torch.sort(t.view(torch.uint32).to(torch.int64))[0].to(torch.uint32).view(torch.int32)
    out = torch.empty_like(t)
    f = lambda: _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 8, 1, st))
    for mode in (2, 1):
        L.bsg_debug_set_msd(mode)
        out.zero_()
        f(); torch.cuda.synchronize()
        ok = bool(torch.equal(out, exp))
        for _ in range(2): f()
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        reps = 10
        s.record()
        for _ in range(reps): f()
        e.record(); torch.cuda.synchronize()
        tot = s.elapsed_time(e) / reps
        ctx.set_timing(False); ctx.set_timing(True)
        for _ in range(3): f()
        kt = {k: ctx.kernel_time(getattr(_lib, k)) for k in ("K_MSD_HIST", "K_MSD_PARTITION", "K_MSD_LOCAL", "K_HIST", "K_FIRST_PASS", "K_RELAXED_PASS", "K_ONESWEEP")}
        ctx.set_timing(False)
        print("n=%d mode=%d equal=%s sort %.4f ms |" % (n, mode, ok, tot), " ".join("%s %.4f(x%d)" % (k[2:], v[0] / 3, v[1] // 3) for k, v in kt.items()), flush=True)
L.bsg_debug_set_msd(0)
