"""On-GPU generate_uniform_keys: parity with the host stream + throughput (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
L = _lib.lib(); ctx = _lib.context(0); st = torch.cuda.current_stream().cuda_stream
for n, seed in ((1, 5), (313, 5), (100003, 7), ((1 << 20) + 7, bsg.derive_seed(1, 0)), (1 << 26, bsg.derive_seed(1, 0))):
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    t0 = time.time()
    _lib.check(L.bsg_generate_uniform_device_u32(ctx.handle, out.data_ptr(), n, seed, st))
    torch.cuda.synchronize()
    t1 = time.time()
    host = bsg.generate_uniform_keys(n, seed)
    print(n, "equal" if np.array_equal(out.cpu().numpy().view(np.uint32), host) else "MISMATCH", f"first call {t1-t0:.3f}s", flush=True)
n = 1 << 28
out = torch.empty(n, dtype=torch.int32, device="cuda")
for _ in range(2):
    _lib.check(L.bsg_generate_uniform_device_u32(ctx.handle, out.data_ptr(), n, 1, st))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); _lib.check(L.bsg_generate_uniform_device_u32(ctx.handle, out.data_ptr(), n, 1, st)); e1.record(); torch.cuda.synchronize()
print(f"2^28 keys on device: {e0.elapsed_time(e1):.2f} ms (host generator ~1.6 s)")
t = time.time(); h = bsg.generate_uniform_keys(n, 1); th = time.time() - t
print("2^28 equal:", np.array_equal(out.cpu().numpy().view(np.uint32), h), f"host {th:.2f}s")
