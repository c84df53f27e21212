"""Times the fused peer-store PR4 round path (variant P) with one rank (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, torch.distributed as dist
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import distributed as D
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29535")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
n = 1 << 28
blk = bsg.generate_uniform_keys_device(n, 1).view(torch.int32)
peer = D.PeerBlocks(n)
for _ in range(2):
    out = D.parallel_radix_sort(blk, n, radix=256, exchange="peer", peer=peer)
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True); ts = []
for _ in range(5):
    s.record(); out = D.parallel_radix_sort(blk, n, radix=256, exchange="peer", peer=peer); e.record()
    torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
print(f"{os.environ.get('BSG_LIB', 'default')}: variant P world 1, 2^28 keys: {min(ts):.3f} ms", flush=True)
dist.destroy_process_group()
