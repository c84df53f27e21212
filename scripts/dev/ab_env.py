"""Same-session A/B of one-sweep variants selected by environment variables
(development aid).  usage: python scripts/dev/ab_env.py "BSG_OS_RANK=0" "BSG_OS_RANK=4,BSG_LIB=build/var/x/libbsg.so"
Each spec runs in its own process; rounds are interleaved so clock drift hits
all variants alike.  AB_N keys (default 2^28), AB_RADIX bits (default 8)."""
import os, subprocess, sys

CHILD = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.environ["REPO"])
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
n = int(os.environ.get("AB_N", str(1 << 28))); bits = int(os.environ.get("AB_RADIX", "8"))
t = bsg.generate_uniform_keys_device(n, 1)
out = torch.empty_like(t)
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
f = lambda: _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, bits, 1, st))
for _ in range(3): f()
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True); ts = []
for _ in range(20):
    s.record(); f(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
ctx.set_timing(True); f(); f(); f(); torch.cuda.synchronize()
os_ms, os_cnt = ctx.kernel_time(_lib.K_ONESWEEP); ctx.set_timing(False)
exp = torch.sort(t.view(torch.int32).to(torch.int64) & 0xFFFFFFFF)[0] if n <= (1 << 28) else None
ok = bool(torch.equal(out.view(torch.int32).to(torch.int64) & 0xFFFFFFFF, exp)) if exp is not None else None
ts.sort(); print("RESULT", min(ts), ts[len(ts) // 2], os_ms / max(os_cnt, 1), ok)
'''

repo = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
res = {}
for rnd in range(int(os.environ.get("AB_ROUNDS", "3"))):
    for spec in sys.argv[1:]:
        env = dict(os.environ, REPO=repo)
        for kv in filter(None, spec.split(",")):
            k, _, v = kv.partition("=")
            env[k] = os.path.abspath(v) if k == "BSG_LIB" else v
        try:
            p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True,
                               timeout=float(os.environ.get("AB_TIMEOUT", "180")))
        except subprocess.TimeoutExpired:
            print(rnd, spec, "TIMEOUT", flush=True); continue
        line = [l for l in p.stdout.splitlines() if l.startswith("RESULT")]
        if not line:
            print(spec, "FAILED", p.stderr[-2000:]); continue
        _, mn, md, pas, ok = line[0].split()
        res.setdefault(spec, []).append((float(mn), float(md), float(pas), ok))
        print(rnd, spec, mn, md, pas, ok, flush=True)
for spec, v in res.items():
    print("SUMMARY %-40s best %.4f  median %.4f  pass %.4f ms" % (spec, min(x[0] for x in v),
          sorted(x[1] for x in v)[len(v) // 2], min(x[2] for x in v)), {x[3] for x in v})
