"""Host enqueue time vs device time of back-to-back sorts (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
import bench

n = 1 << 28
keys = bsg.generate_uniform_keys(n, bsg.derive_seed(1, 0))
d_in = torch.from_numpy(keys.view(np.int32)).cuda(); d_out = torch.empty_like(d_in)
ctx = _lib.context(0); ctx.reserve(n); L = _lib.lib(); st = torch.cuda.current_stream(); sh = st.cuda_stream
step = lambda: _lib.check(L.bsg_radix_sort_u32(ctx.handle, d_in.data_ptr(), d_out.data_ptr(), n, 8, 1, sh))
for _ in range(3): step()
torch.cuda.synchronize()
for label in ("plain", "sampler", "plain"):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cm = bench.ClockSampler(0) if label == "sampler" else None
    if cm: cm.__enter__()
    torch.cuda.synchronize()
    t0 = time.perf_counter(); e0.record(st)
    hs = []
    for _ in range(10):
        a = time.perf_counter(); step(); hs.append(time.perf_counter() - a)
    e1.record(st); t1 = time.perf_counter()
    torch.cuda.synchronize()
    if cm: cm.__exit__(None, None, None)
    print(label, "device ms/sort %.3f" % (e0.elapsed_time(e1) / 10), "host enqueue ms/call", ["%.2f" % (h * 1e3) for h in hs])
