"""Same-session A/B of in-process PR (segmented one-sweep rounds) across library
builds (development aid).  usage: python scripts/dev/ab_pr.py LIB ...  (AB_CASES="n:p:bits,...")"""
import os, subprocess, sys

CHILD = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.environ["REPO"])
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
for case in os.environ.get("AB_CASES", "268435456:8:8,2147483648:2:8").split(","):
    n, p, bits = (int(x) for x in case.split(":"))
    t = bsg.generate_uniform_keys_device(n, 3).view(torch.int32)
    out = torch.empty_like(t)
    f = lambda: _lib.check(L.bsg_parallel_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, p, bits, -1, None, 1, st))
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); f(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    o = out[: min(n, 1 << 26)]
    ok = bool((o[1:].to(torch.int64) & 0xFFFFFFFF >= o[:-1].to(torch.int64) & 0xFFFFFFFF).all())
    print("RESULT", case, min(ts), ok, flush=True)
    del t, out; torch.cuda.empty_cache(); ctx.release()
'''
repo = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
for rnd in range(int(os.environ.get("AB_ROUNDS", "2"))):
    for lib in sys.argv[1:]:
        env = dict(os.environ, REPO=repo, BSG_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        for l in r.stdout.splitlines():
            if l.startswith("RESULT"):
                print(rnd, lib, l[7:], flush=True)
        if r.returncode:
            print(lib, "FAILED", r.stderr[-1500:])
