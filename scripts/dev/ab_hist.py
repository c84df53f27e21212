"""Same-session A/B of the digit-histogram kernel (K1) across builds (development aid)."""
import os, subprocess, sys
CHILD = r'''
import os, sys, torch
sys.path.insert(0, os.environ["REPO"])
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
n = 1 << 28
t = bsg.generate_uniform_keys_device(n, 1); out = torch.empty_like(t)
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
f = lambda: _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 8, 1, st))
for _ in range(3): f()
torch.cuda.synchronize(); ctx.set_timing(True)
for _ in range(10): f()
torch.cuda.synchronize(); ms, cnt = ctx.kernel_time(_lib.K_HIST); print("RESULT", ms / cnt)
'''
repo = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
for rnd in range(3):
    for lib in sys.argv[1:]:
        r = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, REPO=repo, BSG_LIB=os.path.abspath(lib)),
                           capture_output=True, text=True)
        print(rnd, lib, [l for l in r.stdout.splitlines() if l.startswith("RESULT")], r.stderr[-300:] if r.returncode else "")
