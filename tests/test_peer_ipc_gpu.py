"""The fused NVLink round's multi-process plumbing on one GPU: two ranks
(processes) on cuda:0 coordinate over gloo, map each other's next-round
blocks by CUDA IPC (torch reduce_tensor) and store keys into the other
process's memory.  The kernels never wait on each other (rounds are ordered by
host-side barriers), so this checks the IPC mapping, cross-process stores and
round ordering -- not multi-GPU performance."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, n, radix, rounds, result_q):
    import torch
    import torch.distributed as dist
    import paper_1708_09495_b200 as bsg
    from paper_1708_09495_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        keys = bsg.generate_uniform_keys(n, 321)
        off, size = D.partition_offset_of(n, world, rank), D.partition_size_of(n, world, rank)
        blk = torch.from_numpy(keys[off:off + size].view(np.int32)).cuda()
        peer = D.PeerBlocks(n, device=torch.device("cuda", 0))
        out = D.parallel_radix_sort(blk, n, radix=radix, rounds=rounds, exchange="peer", peer=peer)
        result_q.put((rank, out.cpu().numpy().view(np.uint32).copy()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("radix,rounds", [(256, 1), (256, None), (65536, None)])
def test_two_processes_peer_exchange(cuda, orc, radix, rounds):
    import torch.multiprocessing as mp

    n, world = 200003, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, n, radix, rounds, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = dict(q.get(timeout=240) for _ in range(world))
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    keys = orc.generate_uniform_keys(n, 321)
    exp, _ = orc.parallel_radix(keys, world, radix, -1 if rounds is None else rounds)
    np.testing.assert_array_equal(np.concatenate([got[0], got[1]]), exp)
