"""CPU: the multi-process PR orchestration (paper_1708_09495_b200.distributed)
under gloo with world_size 2 and 3.  The per-worker steps are host stand-ins
(oracle count/sort, the product's host planner bsg_pr_plan_host, a numpy
rebuild) so the collective sequence, split sizes and buffer handling of the
product orchestration are exercised without a GPU.  Every rank's block after
k rounds must equal worker `rank`'s block of the reference's
run_parallel_radix with plan.rounds = k."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class HostOps:
    def __init__(self):
        from oracle.pyoracle import Oracle
        import paper_1708_09495_b200 as bsg

        self.orc = Oracle()
        self.L = bsg._lib.lib()

    def keys(self, n):
        return torch.empty(n, dtype=torch.int32)

    def count(self, block, rnd, bits):
        k = block.numpy().view(np.uint32)
        d = (k.astype(np.uint64) >> np.uint64(rnd * bits)) & np.uint64((1 << bits) - 1)
        return torch.from_numpy(np.bincount(d.astype(np.int64), minlength=1 << bits).astype(np.int64))

    def local_sort(self, block, rnd, bits):
        out = self.orc.count_sort_round(block.numpy().view(np.uint32), rnd, 1 << bits)
        return torch.from_numpy(out.view(np.int32).copy())

    def plan(self, counts_all, n, p, me, rnd, bits):
        c = np.ascontiguousarray(counts_all.numpy().astype(np.uint64))
        send = np.zeros(p, np.uint64)
        recv = np.zeros(p, np.uint64)
        delta = np.zeros(p << bits, np.int64)
        rc = self.L.bsg_pr_plan_host(c.ctypes.data, n, p, me, bits, send.ctypes.data, recv.ctypes.data,
                                     delta.ctypes.data)
        assert rc == 0
        return [int(x) for x in send], [int(x) for x in recv], recv, delta

    def sort(self, keys):
        return torch.from_numpy(np.sort(keys.numpy().view(np.uint32)).view(np.int32))

    def merge_keep(self, mine, theirs, keep_low):
        lo, hi = self.orc.merge_split(mine.numpy().view(np.uint32), theirs.numpy().view(np.uint32))
        return torch.from_numpy((lo if keep_low else hi).view(np.int32).copy())

    def rebuild(self, recv, recv_counts, p, rnd, bits, delta, out_len):
        k = recv.numpy().view(np.uint32)
        src = np.repeat(np.arange(p), recv_counts.astype(np.int64))
        d = ((k.astype(np.uint64) >> np.uint64(rnd * bits)) & np.uint64((1 << bits) - 1)).astype(np.int64)
        pos = delta[src * (1 << bits) + d] + np.arange(k.size)
        out = np.empty(out_len, np.uint32)
        out[pos] = k
        assert np.array_equal(np.sort(pos), np.arange(out_len))
        return torch.from_numpy(out.view(np.int32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cases, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1708_09495_b200 import distributed as D

        ops = HostOps()
        res = []
        for keys, radix, rounds in cases:
            n = keys.size
            off = D.partition_offset_of(n, world, rank)
            sz = D.partition_size_of(n, world, rank)
            blk = torch.from_numpy(keys[off:off + sz].view(np.int32).copy())
            out = D.parallel_radix_sort(blk, n, radix=radix, rounds=rounds, ops=ops)
            res.append(out.numpy().view(np.uint32).copy())
        q.put((rank, res, None))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback

        q.put((rank, None, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_pr_matches_reference_rounds(world, orc):
    keys_u = orc.generate_uniform_keys(4001, 17)
    keys_d = orc.generate_uniform_keys(3000, 5) % 31
    cases = []
    for keys in (keys_u, keys_d):
        for radix in (256, 65536):
            for rounds in sorted({0, 1, 32 // (radix.bit_length() - 1)}):
                cases.append((keys, radix, rounds))
    cases.append((np.array([5, 1, 4], np.uint32), 256, 4))  # fewer keys than... p=3 edge
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = {}
    for _ in range(world):
        rank, res, err = q.get(timeout=300)
        assert err is None, err
        out[rank] = res
    for pr in procs:
        pr.join(timeout=60)
    for ci, (keys, radix, rounds) in enumerate(cases):
        exp, _ = orc.parallel_radix(keys, world, radix, rounds)
        got = np.concatenate([out[r][ci] for r in range(world)])
        np.testing.assert_array_equal(got, exp, err_msg=f"case {ci} radix={radix} rounds={rounds}")


def _worker_b(rank, world, port, cases, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1708_09495_b200 import distributed as D

        ops = HostOps()
        res = []
        for keys in cases:
            n = keys.size
            off = D.partition_offset_of(n, world, rank)
            sz = D.partition_size_of(n, world, rank)
            blk = torch.from_numpy(keys[off:off + sz].view(np.int32).copy())
            out = D.parallel_radix_sort_single_exchange(blk, ops=ops)
            res.append(out.numpy().view(np.uint32).copy())
        q.put((rank, res, None))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback

        q.put((rank, None, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_single_exchange_variant(world, orc):
    cases = [orc.generate_uniform_keys(40001, 3), orc.generate_uniform_keys(20000, 4) % 7,
             np.array([5, 1, 4], np.uint32), np.array([], np.uint32)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_b, args=(r, world, port, cases, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = {}
    for _ in range(world):
        rank, res, err = q.get(timeout=300)
        assert err is None, err
        out[rank] = res
    for pr in procs:
        pr.join(timeout=60)
    for ci, keys in enumerate(cases):
        got = np.concatenate([out[r][ci] for r in range(world)])
        np.testing.assert_array_equal(got, np.sort(keys))
        sizes = [out[r][ci].size for r in range(world)]
        assert max(sizes) - min(sizes) <= 2 * int(np.bincount(keys >> 24, minlength=256).max()) + 1


def test_digit_cuts_balanced():
    from paper_1708_09495_b200.distributed import digit_cuts

    assert digit_cuts([10] * 256, 4) == [0, 64, 128, 192, 256]
    assert digit_cuts([0] * 256, 3)[0] == 0 and digit_cuts([0] * 256, 3)[-1] == 256
    c = digit_cuts([1000] + [0] * 255, 2)
    assert c[0] == 0 and c[-1] == 256


def _worker_net(rank, world, port, cases, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1708_09495_b200 import distributed as D

        ops = HostOps()
        res = []
        for keys, network, stages in cases:
            L = keys.size // world
            blk = torch.from_numpy(keys[rank * L:(rank + 1) * L].view(np.int32).copy())
            out = D.block_network_sort(blk, network, stages, ops=ops)
            res.append(out.numpy().view(np.uint32).copy())
        q.put((rank, res, None))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback

        q.put((rank, None, traceback.format_exc()))


@pytest.mark.parametrize("world,networks", [(2, (0, 1)), (3, (1,)), (4, (0, 1))])
def test_gloo_block_networks_match_reference_stages(world, networks, orc):
    """BTN/OET with one worker per rank; after every stage the
    rank-ordered blocks equal run_block_network's block states."""
    keys = orc.generate_uniform_keys(1200, 11)
    cases = []
    for network in networks:
        S = orc.schedule(network, world)[0].shape[0]
        for stages in range(S + 1):
            cases.append((keys, network, stages))
    ctx = mp.get_context("spawn")
    qq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_net, args=(r, world, port, cases, qq)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = {}
    for _ in range(world):
        rank, res, err = qq.get(timeout=300)
        assert err is None, err
        out[rank] = res
    for pr in procs:
        pr.join(timeout=60)
    for ci, (k, network, stages) in enumerate(cases):
        exp, _ = orc.block_network(network, k, world, stages)
        got = np.concatenate([out[r][ci] for r in range(world)])
        np.testing.assert_array_equal(got, exp, err_msg=f"network {network} stages {stages}")


def test_exchange_sizes_checked_before_any_byte_moves():
    """bsp_error equivalents on the host side of the orchestration
    (radix.hpp:207-220, 283-286): a rank must send every key of its block
    exactly once and, in PR, receive exactly its partition's size."""
    from paper_1708_09495_b200 import _lib, distributed as D

    D._check_exchange([3, 4], [2, 5], 7, 7, 0, 0)  # consistent
    with pytest.raises(_lib.BspError, match="send counts"):
        D._check_exchange([3, 3], [2, 5], 7, 7, 1, 2)
    with pytest.raises(_lib.BspError, match="receive counts"):
        D._check_exchange([3, 4], [2, 4], 7, 7, 1, 2)
    D._check_exchange([3, 4], [9, 9], 7, None, 0, 0)  # single exchange: receive size is data-dependent
