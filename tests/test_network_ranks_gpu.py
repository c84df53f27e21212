"""The paper's BTN / OET across ranks (netsort.hpp:157-199 with
one worker per rank) on the device path: p processes on cuda:0 coordinate
over gloo, each runs its block's local sort and every merge_split stage with
the product's kernels (CudaNetworkOps: serial radix sort + bsg_merge_split_u32);
the blocks in rank order after every truncated stage table equal the oracle's
block-network state (orc.block_network(., stages_limit))."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, n, network, result_q):
    import torch
    import torch.distributed as dist
    from paper_1708_09495_b200 import distributed as D
    from oracle.pyoracle import Oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        keys = Oracle().generate_uniform_keys(n, 900 + world)
        L = (n + world - 1) // world
        padded = np.full(L * world, 0xFFFFFFFF, np.uint32)    # prepare_blocks (netsort.hpp:131-139)
        padded[:n] = keys
        blk = torch.from_numpy(padded[rank * L:(rank + 1) * L].view(np.int32).copy()).cuda()
        ops = D.CudaNetworkOps(torch.device("cuda", 0))
        S = len(D.network_schedule(network, world))
        for s in range(S + 1):
            out = D.block_network_sort(blk, network=network, stages=s, ops=ops)
            result_q.put((s, rank, out.cpu().numpy().view(np.uint32).copy()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("network,world,n", [(0, 2, 20000), (0, 4, 40000), (1, 3, 30001), (1, 4, 40003)])
def test_block_network_across_ranks_per_stage(cuda, orc, network, world, n):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, n, network, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    S = orc.schedule(network, world)[0].shape[0]
    got = {}
    for _ in range((S + 1) * world):
        s, r, blk = q.get(timeout=300)
        got[(s, r)] = blk
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    keys = orc.generate_uniform_keys(n, 900 + world)
    for s in range(S + 1):
        state = np.concatenate([got[(s, r)] for r in range(world)])
        exp, _ = orc.block_network(network, keys, world, s)
        np.testing.assert_array_equal(state[:exp.size], exp, err_msg=f"stage {s}")
    assert np.array_equal(np.concatenate([got[(S, r)] for r in range(world)])[:n], np.sort(keys))
