"""Times distributed.parallel_radix_sort (variant A) per radix on this rank's
block (development aid; world size from torchrun, default 1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch, torch.distributed as dist
import paper_1708_09495_b200 as bsg
from paper_1708_09495_b200 import distributed as D

os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
rank = int(os.environ["RANK"]); ws = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
dist.init_process_group("nccl")
n_per = int(os.environ.get("N_PER", str(1 << 26)))
keys = bsg.generate_uniform_keys(n_per, bsg.derive_seed(1, rank))
blk = torch.from_numpy(keys.view(np.int32)).cuda()
for radix in (256, 65536):
    ops = D.CudaStepOps(blk.device)
    for _ in range(2):
        out = D.parallel_radix_sort(blk, n_per * ws, radix, ops=ops)
    torch.cuda.synchronize(); dist.barrier()
    ctx = ops.ctx if hasattr(ops, "ctx") else None
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        out = D.parallel_radix_sort(blk, n_per * ws, radix, ops=ops)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    if ws == 1:
        ok = bool(torch.equal(out.to(torch.int64) & 0xFFFFFFFF, torch.sort(blk.to(torch.int64) & 0xFFFFFFFF).values))
    else:
        ok = None
    if rank == 0:
        print(f"radix {radix}: {ms:.3f} ms per sort of {n_per} keys/rank, verified={ok}", flush=True)
dist.destroy_process_group()
