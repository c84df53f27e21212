"""GPU parity of the parallel radix sort (PR4 / PR2) with p logical workers
(radix_test.cpp:121-163, acceptance.cpp criterion 2) including per-round
intermediate states."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def pr(bsg, keys, p, radix, rounds=None):
    prep = bsg.radix.prepare_parallel_radix(keys, p, radix)
    if rounds is not None:
        prep.plan.rounds = rounds
    return bsg.radix.run_parallel_radix(prep)


def test_single_worker_matches_serial(cuda, bsg, orc):
    keys = orc.generate_uniform_keys(10000, 5)
    for radix in (256, 65536):
        np.testing.assert_array_equal(pr(bsg, keys, 1, radix).output, orc.serial_radix_sort(keys, radix))


@pytest.mark.parametrize("p", [2, 3, 4, 5, 8, 16])
def test_matches_oracle_across_worker_counts(cuda, bsg, orc, p):
    keys = orc.generate_uniform_keys(100000, 9)
    for radix in (256, 65536):
        res = pr(bsg, keys, p, radix)
        np.testing.assert_array_equal(res.output, np.sort(keys))
        _, est = orc.parallel_radix(keys, p, radix)
        assert res.stats == est


@pytest.mark.parametrize("mod", [16, 31])
def test_duplicate_heavy(cuda, bsg, orc, mod):
    keys = orc.generate_uniform_keys(20000, 13) % mod
    for p in (1, 2, 3, 4, 5, 7, 8, 16):
        np.testing.assert_array_equal(pr(bsg, keys, p, 256).output, np.sort(keys))


def test_more_workers_than_keys(cuda, bsg):
    res = pr(bsg, np.array([5, 1, 4], np.uint32), 8, 256)
    assert res.output.tolist() == [1, 4, 5]
    assert pr(bsg, np.array([], np.uint32), 4, 256).output.size == 0


@pytest.mark.parametrize("radix", [256, 65536])
@pytest.mark.parametrize("p", [1, 2, 3, 5, 8])
def test_per_round_states(cuda, bsg, orc, radix, p):
    keys = orc.generate_uniform_keys(1003, 77) % 5000
    rounds = 32 // (radix.bit_length() - 1)
    for k in range(rounds + 1):
        res = pr(bsg, keys, p, radix, k)
        exp, est = orc.parallel_radix(keys, p, radix, k)
        np.testing.assert_array_equal(res.output, exp)
        assert res.stats == est


def test_superstep_counts(cuda, bsg, orc):
    keys = orc.generate_uniform_keys(5000, 21)
    assert pr(bsg, keys, 4, 256).stats["supersteps"] == 9
    assert pr(bsg, keys, 4, 65536).stats["supersteps"] == 5


@pytest.mark.parametrize("bits", [8, 16])
@pytest.mark.parametrize("p", [1, 2, 3, 8])
def test_device_plan_equals_host_plan(cuda, bsg, orc, bits, p):
    torch = cuda
    rng = np.random.default_rng(bits * 100 + p)
    r = 1 << bits
    counts = rng.integers(0, 50, size=p * r).astype(np.uint64)
    counts[rng.integers(0, p * r, size=5)] = 0
    n = int(counts.sum())
    L = bsg._lib.lib()
    ctx = bsg._lib.context(0)
    dc = torch.from_numpy(counts.view(np.int64)).cuda()
    for me in range(p):
        sr = torch.empty(2 * p, dtype=torch.int64, device="cuda")
        delta = torch.empty(p * r, dtype=torch.int64, device="cuda")
        assert L.bsg_pr_plan(ctx.handle, dc.data_ptr(), n, p, me, 0, bits, sr.data_ptr(), sr[p:].data_ptr(),
                             delta.data_ptr(), torch.cuda.current_stream().cuda_stream) == 0
        hs, hr, hd = np.zeros(p, np.uint64), np.zeros(p, np.uint64), np.zeros(p * r, np.int64)
        assert L.bsg_pr_plan_host(counts.ctypes.data, n, p, me, bits, hs.ctypes.data, hr.ctypes.data,
                                  hd.ctypes.data) == 0
        torch.cuda.synchronize()
        assert sr[:p].cpu().numpy().astype(np.uint64).tolist() == hs.tolist()
        assert sr[p:].cpu().numpy().astype(np.uint64).tolist() == hr.tolist()
        np.testing.assert_array_equal(delta.cpu().numpy(), hd)


def test_distributed_nccl_world1(cuda, bsg, orc):
    """The NCCL orchestration with one rank on the GPU (all-gather and
    all-to-all-v degenerate to copies) equals the serial sort, per round."""
    torch = cuda
    import os
    import torch.distributed as dist
    from paper_1708_09495_b200 import distributed as D

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        keys = orc.generate_uniform_keys(100003, 9)
        blk = torch.from_numpy(keys.view(np.int32)).cuda()
        out = D.parallel_radix_sort_single_exchange(blk)
        np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), np.sort(keys))
        # SURVEY §8(f)1 block network with one worker per rank (p = 1 here:
        # local sort only, zero stages)
        for network in (0, 1):
            blk = torch.from_numpy(keys[:4096].view(np.int32)).cuda()
            out = D.block_network_sort(blk, network)
            np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), np.sort(keys[:4096]))
        for radix in (256, 65536):
            for rounds in (1, None):
                blk = torch.from_numpy(keys.view(np.int32)).cuda()
                out = D.parallel_radix_sort(blk, keys.size, radix=radix, rounds=rounds)
                exp, _ = orc.parallel_radix(keys, 1, radix, -1 if rounds is None else rounds)
                np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), exp)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p", [3, 8, 64])
def test_large_blocks_per_round(cuda, bsg, orc, p):
    """Multi-tile worker blocks: per-round states and RunStats vs the oracle."""
    keys = orc.generate_uniform_keys((1 << 20) + 777, 1000 + p)
    for radix in (256, 65536):
        rounds = 32 // (radix.bit_length() - 1)
        for k in sorted({1, rounds}):
            res = pr(bsg, keys, p, radix, k)
            exp, est = orc.parallel_radix(keys, p, radix, k)
            np.testing.assert_array_equal(res.output, exp)
            assert res.stats == est
