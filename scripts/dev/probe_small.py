"""Small-n SR4 latency probe: CUDA-event time per sort (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
ctx = _lib.context(0); L = _lib.lib(); st = torch.cuda.current_stream().cuda_stream
for lg in [int(x) for x in os.environ.get("SIZES", "16,18,20,22").split(",")]:
    n = 1 << lg
    keys = bsg.generate_uniform_keys(n, bsg.derive_seed(1, 0))
    t = torch.from_numpy(keys.view(np.int32)).cuda(); o = torch.empty_like(t)
    f = lambda: _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), o.data_ptr(), n, 8, 1, st))
    for _ in range(5): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = int(os.environ.get("REPS", "50"))
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    ok = bool((o.cpu().numpy().view(np.uint32) == np.sort(keys)).all())
    print(f"n=2^{lg}: {e0.elapsed_time(e1)/reps*1e3:.1f} us per sort (back-to-back), ok={ok}", flush=True)
