"""Same-session A/B of onesweep builds/configs (development aid).

usage: python scripts/ab.py LIB[:CFG] ...   (LIB = path to a libbsg.so build,
CFG = BSG_OS_CFG value).  Each combination runs in its own process, rounds
interleaved so clock drift hits all variants alike.
"""
import json, os, subprocess, sys

CHILD = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.environ["REPO"])
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
n = int(os.environ.get("AB_N", str(1 << 28)))
keys = bsg.generate_uniform_keys(n, 1)
t = torch.from_numpy(keys.view(np.int32)).cuda().view(torch.uint32)
out = torch.empty_like(t)
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
f = lambda: _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 8, 1, st))
for _ in range(3): f()
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True); ts = []
for _ in range(20):
    s.record(); f(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
ok = bool((out.cpu().numpy() == np.sort(keys)).all()) if n <= (1 << 26) else None
if ok is None:
    o = out.cpu().numpy(); ok = bool((o[1:] >= o[:-1]).all()) and int(o.astype(np.uint64).sum()) == int(keys.astype(np.uint64).sum())
ts.sort(); print("RESULT", min(ts), ts[len(ts) // 2], ok)
'''

repo = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
res = {}
for rnd in range(int(os.environ.get("AB_ROUNDS", "3"))):
    for spec in sys.argv[1:]:
        lib, _, cfg = spec.partition(":")
        env = dict(os.environ, REPO=repo, BSG_LIB=os.path.abspath(lib))
        if cfg:
            env["BSG_OS_CFG"] = cfg
        try:
            p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True,
                               timeout=float(os.environ.get("AB_TIMEOUT", "120")))
        except subprocess.TimeoutExpired:
            print(rnd, spec, "TIMEOUT", flush=True); continue
        line = [l for l in p.stdout.splitlines() if l.startswith("RESULT")]
        if not line:
            print(spec, "FAILED", p.stderr[-2000:]); continue
        _, mn, md, ok = line[0].split()
        res.setdefault(spec, []).append((float(mn), float(md), ok))
        print(rnd, spec, mn, md, ok, flush=True)
for spec, v in res.items():
    print("SUMMARY", spec, "best-min %.4f" % min(x[0] for x in v), "median-med %.4f" % sorted(x[1] for x in v)[len(v) // 2], {x[2] for x in v})
