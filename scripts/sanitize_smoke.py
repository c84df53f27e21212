"""Small invocations of every kernel family with result checks: a quick
all-paths sanity run (run it under compute-sanitizer --tool memcheck/racecheck/synccheck).  Development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import _lib, distributed as D

L = _lib.lib(); ctx = _lib.context(0); st = torch.cuda.current_stream().cuda_stream
def dev(a): return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()
for n in (1, 1000, 70001):
    keys = bsg.generate_uniform_keys(n, n)
    assert np.array_equal(bsg.radix.serial_radix_sort(keys, 256), np.sort(keys))
    assert np.array_equal(bsg.radix.serial_radix_sort(keys, 65536), np.sort(keys))
    bsg.radix.count_sort_round(keys, 1, 16)
# multi-launch path + config rows + misaligned pointers
L.bsg_debug_set_small_sort(0)
keys = bsg.generate_uniform_keys(100003, 3)
for cfg in (1, 2, 4, 6):
    L.bsg_debug_set_onesweep_cfg(cfg)
    assert np.array_equal(bsg.radix.serial_radix_sort(keys, 256), np.sort(keys))
L.bsg_debug_set_onesweep_cfg(0); L.bsg_debug_set_small_sort(1)
t = dev(np.concatenate([[0], keys])); o = torch.empty_like(t)
_lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr() + 4, o.data_ptr() + 4, keys.size, 8, 1, st))
# PR (segmented r=2^8, r=2^16 path), networks, merge_split
for p in (1, 3, 8):
    for r in (256, 65536):
        res = bsg.radix.run_parallel_radix(bsg.radix.prepare_parallel_radix(keys[:20000], p, r))
        assert np.array_equal(res.output, np.sort(keys[:20000]))
arrs = keys[:64 * 300].reshape(64, 300)
for net in (0, 1):
    out, _ = bsg.netsort.block_network_batched(arrs, 4, net)
    assert np.array_equal(out, np.sort(arrs, axis=1))
# register networks (power-of-two blocks): in-warp, layout-B and cross-warp paths
for ln, p in ((4096, 8), (1024, 2), (16384, 2), (256, 16)):
    arrs = keys[:8 * ln].reshape(8, ln) if 8 * ln <= keys.size else np.tile(keys[:ln], 8).reshape(8, ln)
    for net in (0, 1):
        out, _ = bsg.netsort.block_network_batched(arrs, p, net)
        assert np.array_equal(out, np.sort(arrs, axis=1))
        S = len(D.network_schedule(net, p))
        bsg.netsort.block_network_batched(arrs, p, net, S // 2)
big = keys[:40000]
assert np.array_equal(bsg.netsort.oet_sort(bsg.SortInstance(big, 5, bsg.Algorithm.OET)), np.sort(big))
lo, hi = bsg.netsort.merge_split(np.sort(keys[:500]), np.sort(keys[500:1100]))
# peer-store exchange with logical workers
ops = D.CudaStepOps(torch.device("cuda", 0))
n = 30001; p = 3
blocks = [dev(keys[D.partition_offset_of(n, p, w):D.partition_offset_of(n, p, w) + D.partition_size_of(n, p, w)]) for w in range(p)]
counts_all = torch.cat([ops.count(b, 0, 8) for b in blocks])
nxt = [torch.empty(D.partition_size_of(n, p, w), dtype=torch.int32, device="cuda") for w in range(p)]
for me in range(p):
    ops.fused_round(blocks[me], counts_all, n, p, me, 0, 8, [t.data_ptr() for t in nxt])
    ops.peer_scatter(ops.local_sort(blocks[me], 0, 8), counts_all, n, p, me, 0, 8, [t.data_ptr() for t in nxt])
# generator
out = torch.empty(300000, dtype=torch.int32, device="cuda")
_lib.check(L.bsg_generate_uniform_device_u32(ctx.handle, out.data_ptr(), 300000, 9, st))
torch.cuda.synchronize()
print("sanitize smoke ok")
