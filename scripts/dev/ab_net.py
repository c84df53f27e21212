"""Same-session A/B of block-network builds (development aid).
usage: python scripts/ab_net.py LIB ...  (C4: 2^16 arrays x 4096 keys; BTN/OET p=2,8)"""
import os, subprocess, sys

CHILD = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.environ["REPO"])
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
num, ln = int(os.environ.get("AB_NUM", 1 << 16)), int(os.environ.get("AB_LEN", 4096))
keys = bsg.generate_uniform_keys(num * ln, 7)
t = torch.from_numpy(keys.view(np.int32)).cuda().view(torch.uint32)
out = torch.empty_like(t)
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
ref = torch.sort(t.view(torch.int32).to(torch.int64).view(num, ln) & 0xFFFFFFFF, dim=1).values
for net in (0, 1):
    for p in (2, 8):
        f = lambda: _lib.check(L.bsg_block_network_batched_u32(ctx.handle, net, t.data_ptr(), out.data_ptr(), num, ln, p, -1, None, 1, st))
        for _ in range(2): f()
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True); ts = []
        for _ in range(10):
            s.record(); f(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
        ok = bool(torch.equal(out.view(torch.int32).to(torch.int64).view(num, ln) & 0xFFFFFFFF, ref))
        print("RESULT", net, p, min(ts), ok)
'''
repo = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
for rnd in range(2):
    for lib in sys.argv[1:]:
        env = dict(os.environ, REPO=repo, BSG_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        for l in r.stdout.splitlines():
            if l.startswith("RESULT"):
                _, net, p, ms, ok = l.split()
                print(rnd, lib, ("BTN", "OET")[int(net)], "p=" + p, "%.3f ms" % float(ms), ok, flush=True)
        if r.returncode:
            print(lib, "FAILED", r.stderr[-1500:])
