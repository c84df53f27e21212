"""serial_radix_sort through BSG_MEM_HOST with pageable vs pinned 2^28-key buffers."""
import sys, time, numpy as np, torch
sys.path.insert(0, __import__("os").environ.get("REPO", "."))
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib
n = 1 << 28
keys = bsg.generate_uniform_keys(n, 1)
out = np.empty_like(keys)
ctx = _lib.context(0); L = _lib.lib()
pin_in = torch.from_numpy(keys.view(np.int32)).pin_memory(); pin_out = torch.empty_like(pin_in).pin_memory()
def run(a, b):
    _lib.check(L.bsg_radix_sort_u32(ctx.handle, a, b, n, 8, _lib.MEM_HOST, None))
for name, a, b in (("pageable", keys.ctypes.data, out.ctypes.data), ("pinned", pin_in.data_ptr(), pin_out.data_ptr())):
    run(a, b); ts = []
    for _ in range(3):
        t = time.perf_counter(); run(a, b); ts.append(time.perf_counter() - t)
    print(name, "ms %.1f" % (min(ts) * 1e3), "Gkeys/s %.2f" % (n / min(ts) / 1e9))
assert np.array_equal(out[::4096], np.sort(keys)[::4096])
