"""Per-kernel-class ms per launch of full 2^28-key sorts for the library in BSG_LIB (development aid)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
L = _lib.lib(); ctx = _lib.context(0); st = torch.cuda.current_stream().cuda_stream
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
t = torch.empty(n, dtype=torch.int32, device="cuda")
_lib.check(L.bsg_generate_uniform_device_u32(ctx.handle, t.data_ptr(), n, bsg.derive_seed(1, 0), st))
out = torch.empty_like(t)
f = lambda: _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 8, 1, st))
for _ in range(3): f()
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): f()
e.record(); torch.cuda.synchronize()
tot = s.elapsed_time(e) / 10
ctx.set_timing(True)
for _ in range(5): f()
per = lambda a: a[0] / max(a[1], 1)
exp = torch.sort(t.view(torch.uint32).to(torch.int64))[0].to(torch.uint32).view(torch.int32)
print(os.environ.get("BSG_LIB", "default").split("/")[-2], "sort %.4f  K3f %.4f K3r %.4f K3 %.4f hist %.4f equal %s" % (
    tot, per(ctx.kernel_time(_lib.K_FIRST_PASS)), per(ctx.kernel_time(_lib.K_RELAXED_PASS)),
    per(ctx.kernel_time(_lib.K_ONESWEEP)), per(ctx.kernel_time(_lib.K_HIST)), bool(torch.equal(out, exp))))
