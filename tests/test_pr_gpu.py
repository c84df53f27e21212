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
    from paper_1708_09495_b200 import distributed as D

    rng = np.random.default_rng(bits * 100 + p)
    r = 1 << bits
    n = 25 * p * r + 7
    # row v: worker v's digit counts, summing to Partition(n, p).size_of(v)
    counts = np.concatenate([rng.multinomial(D.partition_size_of(n, p, v), np.full(r, 1.0 / r))
                             for v in range(p)]).astype(np.uint64)
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
        # exchange + rebuild as one peer-store kernel (IPC-mapped
        # next-round blocks; with one rank every store is local)
        peer = D.PeerBlocks(keys.size)
        for radix in (256, 65536):
            for rounds in (1, None):
                blk = torch.from_numpy(keys.view(np.int32)).cuda()
                out = D.parallel_radix_sort(blk, keys.size, radix=radix, rounds=rounds, exchange="peer", peer=peer)
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


@pytest.mark.parametrize("p", [2, 3, 5, 8])
def test_peer_scatter_logical_workers(cuda, bsg, orc, p):
    """bsg_pr_peer_scatter with p logical workers in one process (all
    next-round blocks local): every round's concatenated blocks equal
    run_parallel_radix with plan.rounds = k (radix.hpp:260-303)."""
    torch = cuda
    import ctypes
    from paper_1708_09495_b200 import distributed as D

    ops = D.CudaStepOps(torch.device("cuda", 0))
    n = 100003 if p != 2 else (1 << 21) + 5  # p = 2: multi-tile blocks
    keys = orc.generate_uniform_keys(n, 40 + p) % np.uint32(1 << 30)
    sizes = [D.partition_size_of(n, p, w) for w in range(p)]
    offs = [D.partition_offset_of(n, p, w) for w in range(p)]
    for radix in (256, 65536):
        bits = radix.bit_length() - 1
        blocks = [torch.from_numpy(keys[offs[w]:offs[w] + sizes[w]].view(np.int32)).cuda() for w in range(p)]
        for rnd in range(32 // bits):
            counts_all = torch.cat([ops.count(b, rnd, bits) for b in blocks])
            exp, _ = orc.parallel_radix(keys, p, radix, rnd + 1)
            # (a) local pass, then the peer-store exchange kernel
            nxt = [torch.empty(max(sz, 1), dtype=torch.int32, device="cuda") for sz in sizes]
            ptrs = [t.data_ptr() for t in nxt]
            for me in range(p):
                ops.peer_scatter(ops.local_sort(blocks[me], rnd, bits), counts_all, n, p, me, rnd, bits, ptrs)
            np.testing.assert_array_equal(torch.cat([nxt[w][:sizes[w]] for w in range(p)]).cpu().numpy()
                                          .view(np.uint32), exp)
            # (b) the whole round as one pass writing into the owners' blocks
            fused = [torch.empty(max(sz, 1), dtype=torch.int32, device="cuda") for sz in sizes]
            fptrs = [t.data_ptr() for t in fused]
            for me in range(p):
                ops.fused_round(blocks[me], counts_all, n, p, me, rnd, bits, fptrs)
            blocks = [fused[w][:sizes[w]] for w in range(p)]
            np.testing.assert_array_equal(torch.cat(blocks).cpu().numpy().view(np.uint32), exp)
    L = bsg._lib.lib()
    arr = (ctypes.c_void_p * 2)(0, 0)
    ctx = bsg._lib.context(0)
    # size mismatch and bad worker index fail loudly
    assert L.bsg_pr_peer_scatter(ctx.handle, 0, 5, 0, n, 2, 0, 0, 8, arr, None) != 0
    assert L.bsg_pr_peer_scatter(ctx.handle, 0, 0, 0, n, 2, 2, 0, 8, arr, None) != 0
    assert L.bsg_pr_fused_round(ctx.handle, 0, 5, 0, n, 2, 0, 0, 8, arr, None) != 0
    assert L.bsg_pr_fused_round(ctx.handle, 0, 0, 0, n, 2, 0, 9, 8, arr, None) != 0


@pytest.mark.parametrize("p", [8])
def test_c5_full_size_in_process(cuda, bsg, p):
    """BASELINE config 5 at its full size on one GPU: n = 2^33 keys of
    generate_uniform_keys(n, derive_seed(1, 0)) (generated on the device,
    bit-identical to the host stream), PR4 with p logical workers
    (block-distributed n/p: each block 2^30 keys).  At this size the CPU oracle
    is replaced by size-independent properties: globally sorted concatenation
    and multiset checksums (sum, sum of squares mod a prime) equal to the
    input's.  ~128 GiB of device buffers."""
    torch = cuda
    from test_radix_gpu import _chunked_properties

    n = 1 << 33
    free, _ = torch.cuda.mem_get_info()
    if free < 17 * n:
        pytest.skip("not enough device memory")
    keys = bsg.generate_uniform_keys_device(n, bsg.derive_seed(1, 0)).view(torch.int32)
    # the device stream is the host generator's stream: spot-check a window
    # far into it against the host random-access generator
    off = n - 4099
    exp = bsg.generate_uniform_keys_at(4096, bsg.derive_seed(1, 0), off)
    np.testing.assert_array_equal(keys[off:off + 4096].cpu().numpy().view(np.uint32), exp)
    out = torch.empty_like(keys)
    ctx = bsg._lib.context(0)
    L = bsg._lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    assert L.bsg_parallel_radix_sort_u32(ctx.handle, keys.data_ptr(), out.data_ptr(), n, p, 8, -1, None, 1, st) == 0, \
        bsg._lib.last_error()
    torch.cuda.synchronize()
    _chunked_properties(torch, keys, out)
    del keys, out
    bsg._lib.release_all()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("radix_log2", [8, 16])
def test_large_segments_wide_rows(cuda, bsg, radix_log2):
    """Worker blocks above 2^29 keys (p = 2, n = 2^31 + 12345): the segmented
    one-sweep runs its 64-bit status/position rows.  After one round the
    concatenated blocks equal one count_sort_round of the whole array
    (radix.hpp:260-303 with plan.rounds = 1), and the full run equals the
    serial sort; both compared on the device chunk by chunk."""
    torch = cuda
    n, p = (1 << 31) + 12345, 2
    free, _ = torch.cuda.mem_get_info()
    if free < 40 * n:
        pytest.skip("not enough device memory")
    keys = bsg.generate_uniform_keys_device(n, 77).view(torch.int32)
    keys[:5000] = 12345  # ties across the first tiles of block 0
    got = torch.empty_like(keys)
    exp = torch.empty_like(keys)
    ctx = bsg._lib.context(0)
    L = bsg._lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    step = 1 << 27

    def same():
        torch.cuda.synchronize()
        return all(bool(torch.equal(got[a:a + step], exp[a:a + step])) for a in range(0, n, step))

    assert L.bsg_parallel_radix_sort_u32(ctx.handle, keys.data_ptr(), got.data_ptr(), n, p, radix_log2, 1, None, 1,
                                         st) == 0, bsg._lib.last_error()
    assert L.bsg_count_sort_round_u32(ctx.handle, keys.data_ptr(), exp.data_ptr(), n, 0, radix_log2, 1, st) == 0
    assert same()
    assert L.bsg_parallel_radix_sort_u32(ctx.handle, keys.data_ptr(), got.data_ptr(), n, p, radix_log2, -1, None, 1,
                                         st) == 0, bsg._lib.last_error()
    assert L.bsg_radix_sort_u32(ctx.handle, keys.data_ptr(), exp.data_ptr(), n, radix_log2, 1, st) == 0
    assert same()
    del keys, got, exp
    bsg._lib.release_all()
    torch.cuda.empty_cache()


def test_fused_round_large_blocks(cuda, bsg):
    """bsg_pr_fused_round with blocks above 2^29 keys (config 5 puts 2^30-2^32
    keys on each GPU): the 64-bit one-sweep rows store into the owners'
    blocks.  Two logical workers in one process; one round on the input
    equals one count_sort_round of the whole array (a PR round is a stable
    count sort of the block concatenation, radix.hpp:260-303)."""
    torch = cuda
    from paper_1708_09495_b200 import distributed as D

    n, p = (1 << 30) + 4101, 2
    free, _ = torch.cuda.mem_get_info()
    if free < 24 * n:
        pytest.skip("not enough device memory")
    ops = D.CudaStepOps(torch.device("cuda", 0))
    keys = bsg.generate_uniform_keys_device(n, 99).view(torch.int32)
    sizes = [D.partition_size_of(n, p, w) for w in range(p)]
    offs = [D.partition_offset_of(n, p, w) for w in range(p)]
    blocks = [keys[offs[w]:offs[w] + sizes[w]] for w in range(p)]
    ctx = bsg._lib.context(0)
    L = bsg._lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    exp = torch.empty_like(keys)
    for bits, rnd in ((8, 1), (16, 1)):
        counts_all = torch.cat([ops.count(b, rnd, bits) for b in blocks])
        nxt = [torch.empty(sz, dtype=torch.int32, device="cuda") for sz in sizes]
        ptrs = [t.data_ptr() for t in nxt]
        for me in range(p):
            ops.fused_round(blocks[me], counts_all, n, p, me, rnd, bits, ptrs)
        assert L.bsg_count_sort_round_u32(ctx.handle, keys.data_ptr(), exp.data_ptr(), n, rnd, bits, 1, st) == 0
        torch.cuda.synchronize()
        for w in range(p):
            assert bool(torch.equal(nxt[w], exp[offs[w]:offs[w] + sizes[w]])), (bits, w)
        del nxt
    del keys, exp, blocks
    bsg._lib.release_all()
    torch.cuda.empty_cache()


def test_fused_round_global_positions_above_2_32(cuda, bsg):
    """bsg_pr_fused_round where the BLOCKS are small (< 2^29 keys, the
    32-bit look-back rows would do) but the global positions are not:
    n = 2^32 + 2^20 + 7 keys over p = 17 logical workers (~2^28 keys per
    block, the weak-scaled 2^28-per-GPU shape at p >= 17).  Digit bases of the
    high digits exceed 2^32, so the write-out must run the 64-bit position rows
    (a 32-bit position would wrap and store keys at the wrong owner/offset).
    All workers' round-0 passes together equal one count_sort_round of the
    whole array (radix.hpp:44-65; a PR round is a stable count sort of the
    block concatenation, radix.hpp:260-303)."""
    torch = cuda
    from paper_1708_09495_b200 import distributed as D

    n, p = (1 << 32) + (1 << 20) + 7, 17
    free, _ = torch.cuda.mem_get_info()
    if free < 18 * n:
        pytest.skip("not enough device memory")
    ops = D.CudaStepOps(torch.device("cuda", 0))
    keys = bsg.generate_uniform_keys_device(n, 1234).view(torch.int32)
    sizes = [D.partition_size_of(n, p, w) for w in range(p)]
    offs = [D.partition_offset_of(n, p, w) for w in range(p)]
    assert max(sizes) < (1 << 29)
    blocks = [keys[offs[w]:offs[w] + sizes[w]] for w in range(p)]
    counts_all = torch.cat([ops.count(b, 0, 8) for b in blocks])
    nxt = torch.empty_like(keys)
    ptrs = [nxt[offs[w]:].data_ptr() for w in range(p)]
    for me in range(p):
        ops.fused_round(blocks[me], counts_all, n, p, me, 0, 8, ptrs)
    ctx = bsg._lib.context(0)
    L = bsg._lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    exp = torch.empty_like(keys)
    assert L.bsg_count_sort_round_u32(ctx.handle, keys.data_ptr(), exp.data_ptr(), n, 0, 8, 1, st) == 0
    torch.cuda.synchronize()
    step = 1 << 28
    for a in range(0, n, step):
        assert bool(torch.equal(nxt[a:a + step], exp[a:a + step])), a
    del keys, nxt, exp, blocks
    bsg._lib.release_all()
    torch.cuda.empty_cache()


def test_distributed_world1_large_block(cuda, bsg):
    """The multi-GPU orchestration (distributed.py) at a config-5 block size:
    one rank holding 2^30 + 7 keys (every per-rank kernel past 2^29 keys runs
    its 64-bit rows).  Variants A (NCCL all-to-all-v, r = 2^8 and 2^16), B
    (single exchange) and P (peer-store rounds) all equal the serial sort."""
    torch = cuda
    import os
    import torch.distributed as dist
    from paper_1708_09495_b200 import distributed as D

    n = (1 << 30) + 7
    free, _ = torch.cuda.mem_get_info()
    if free < 40 * n:
        pytest.skip("not enough device memory")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = "29533"
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        keys = bsg.generate_uniform_keys_device(n, 5).view(torch.int32)
        exp = torch.empty_like(keys)
        ctx = bsg._lib.context(0)
        L = bsg._lib.lib()
        st = torch.cuda.current_stream().cuda_stream
        assert L.bsg_radix_sort_u32(ctx.handle, keys.data_ptr(), exp.data_ptr(), n, 8, 1, st) == 0
        step = 1 << 27

        def check(out):
            torch.cuda.synchronize()
            assert out.numel() == n
            assert all(bool(torch.equal(out[a:a + step], exp[a:a + step])) for a in range(0, n, step))

        for radix in (256, 65536):
            check(D.parallel_radix_sort(keys.clone(), n, radix=radix))
        check(D.parallel_radix_sort_single_exchange(keys.clone()))
        peer = D.PeerBlocks(n)
        check(D.parallel_radix_sort(keys.clone(), n, radix=256, exchange="peer", peer=peer))
        del peer, keys, exp
        bsg._lib.release_all()
        torch.cuda.empty_cache()
    finally:
        dist.destroy_process_group()


def test_protocol_errors_raise_bsp_error(cuda, bsg):
    """bsp_error equivalents (radix.hpp:207-220, 283-286): count matrices whose
    rows do not sum to the workers' block sizes, and received slices that do
    not fill the rebuilt block, fail with BSG_EPROTO -- and no kernel stores
    outside its blocks (canaries after every block stay intact)."""
    torch = cuda
    import ctypes
    from paper_1708_09495_b200 import distributed as D

    L = bsg._lib.lib()
    ctx = bsg._lib.context(0)
    st = torch.cuda.current_stream().cuda_stream
    p, bits, n = 4, 8, 40003
    ops = D.CudaStepOps(torch.device("cuda", 0))
    keys = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda")
    sizes = [D.partition_size_of(n, p, w) for w in range(p)]
    offs = [D.partition_offset_of(n, p, w) for w in range(p)]
    blocks = [keys[offs[w]:offs[w] + sizes[w]] for w in range(p)]
    good = torch.cat([ops.count(b, 0, bits) for b in blocks])
    bad = good.clone()
    bad[3] += 1                                   # worker 0 claims one key too many
    sr = torch.empty(2 * p, dtype=torch.int64, device="cuda")
    delta = torch.empty(p << bits, dtype=torch.int64, device="cuda")
    assert L.bsg_pr_plan(ctx.handle, good.data_ptr(), n, p, 1, 0, bits, sr.data_ptr(), sr[p:].data_ptr(),
                         delta.data_ptr(), st) == 0
    assert L.bsg_pr_plan(ctx.handle, bad.data_ptr(), n, p, 1, 0, bits, sr.data_ptr(), sr[p:].data_ptr(),
                         delta.data_ptr(), st) == bsg._lib.BSG_EPROTO
    assert "bsp_error" in bsg._lib.last_error()
    hb = bad.cpu().numpy().view(np.uint64).copy()
    hs, hr, hd = np.zeros(p, np.uint64), np.zeros(p, np.uint64), np.zeros(p << bits, np.int64)
    assert L.bsg_pr_plan_host(hb.ctypes.data, n, p, 1, bits, hs.ctypes.data, hr.ctypes.data,
                              hd.ctypes.data) == bsg._lib.BSG_EPROTO
    with pytest.raises(bsg._lib.BspError):
        ops.plan(bad, n, p, 1, 0, bits)

    CAN = 0x5A5A5A5A
    def canaried():
        bufs = [torch.full((sz + 64,), CAN, dtype=torch.int32, device="cuda") for sz in sizes]
        return bufs, [t.data_ptr() for t in bufs]
    def intact(bufs):
        return all(bool((b[sz:] == CAN).all()) for b, sz in zip(bufs, sizes))
    for fn in ("fused_round", "peer_scatter"):
        bufs, ptrs = canaried()
        with pytest.raises(bsg._lib.BspError):
            src = blocks[0] if fn == "fused_round" else ops.local_sort(blocks[0], 0, bits)
            getattr(ops, fn)(src, bad, n, p, 0, 0, bits, ptrs)
        torch.cuda.synchronize()
        assert intact(bufs), fn
        bufs, ptrs = canaried()
        for me in range(p):
            src = blocks[me] if fn == "fused_round" else ops.local_sort(blocks[me], 0, bits)
            getattr(ops, fn)(src, good, n, p, me, 0, bits, ptrs)
        torch.cuda.synchronize()
        assert intact(bufs), fn

    # rebuild: receive counts that do not add up to the received keys
    send, recv, recv_dev, dl = ops.plan(good, n, p, 1, 0, bits)
    recv_buf = torch.randint(-2**31, 2**31 - 1, (sum(recv),), dtype=torch.int32, device="cuda")
    out = torch.full((sum(recv) + 64,), CAN, dtype=torch.int32, device="cuda")
    wrong = recv_dev.clone()
    wrong[0] += 5
    assert L.bsg_pr_rebuild(ctx.handle, recv_buf.data_ptr(), recv_buf.numel(), wrong.data_ptr(), p, 0, bits,
                            dl.data_ptr(), out.data_ptr(), st) == bsg._lib.BSG_EPROTO
    torch.cuda.synchronize()
    assert bool((out[sum(recv):] == CAN).all())
    # exchange sizes checked on the host before any byte moves
    with pytest.raises(bsg._lib.BspError):
        D._check_exchange([1, 2], [3, 4], 4, 7, 0, 0)
    with pytest.raises(bsg._lib.BspError):
        D._check_exchange([1, 2], [3, 3], 3, 7, 0, 0)


@pytest.mark.parametrize("relaxed", [0, 1])
def test_full_run_value_stable_rounds(cuda, bsg, orc, relaxed):
    """The rounds of a FULL in-process PR4/PR2 run whose RunStats are not asked
    for (C ABI, stats = NULL: only the sorted array is returned) may rank
    value-stably from 2^24 keys on; a run that returns RunStats or is
    rounds-limited always ranks strictly, so its count matrices -- and message
    counts -- are the reference's.  Both settings must give the oracle's
    output, below and above 2^24 keys, for ragged blocks, duplicate-heavy and
    skewed keys; RunStats and rounds-limited states stay bit-exact whatever
    the setting."""
    torch = cuda
    L = bsg._lib.lib()
    ctx = bsg._lib.context(0)
    st = torch.cuda.current_stream().cuda_stream
    prev = L.bsg_debug_set_relaxed_passes(relaxed)

    def sort_no_stats(keys, p, bits):
        t = torch.from_numpy(keys.view(np.int32)).cuda()
        out = torch.empty_like(t)
        assert L.bsg_parallel_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), keys.size, p, bits, -1, None,
                                             1, st) == 0, bsg._lib.last_error()
        torch.cuda.synchronize()
        return out.cpu().numpy().view(np.uint32)

    try:
        for n, ps in (((1 << 17) + 5, (1, 3, 8)), ((1 << 22) + 5, (3, 8)), ((1 << 24) + 3, (2, 5)),
                      ((1 << 25) + 1001, (8,))):
            keys = orc.generate_uniform_keys(n, 17 * n + relaxed)
            exp = np.sort(keys)
            for p in ps:
                for bits in (8, 16):
                    np.testing.assert_array_equal(sort_no_stats(keys, p, bits), exp)
                    if n <= (1 << 24) + 3:
                        res = pr(bsg, keys, p, 1 << bits)  # with RunStats: strictly stable rounds
                        np.testing.assert_array_equal(res.output, exp)
                        _, est = orc.parallel_radix(keys, p, 1 << bits)
                        assert res.stats == est
        n = (1 << 24) + 77
        base = orc.generate_uniform_keys(n, 71)
        rng = np.random.default_rng(3)
        for keys in ((base & 0xFFFF0007).astype(np.uint32), rng.choice(base[:500], n).astype(np.uint32),
                     np.minimum(rng.zipf(1.1, n), 0xFFFFFFFF).astype(np.uint32)):
            exp = np.sort(keys)
            for p in (2, 7):
                np.testing.assert_array_equal(sort_no_stats(keys, p, 8), exp)
                np.testing.assert_array_equal(sort_no_stats(keys, p, 16), exp)
        keys = orc.generate_uniform_keys((1 << 20) + 9, 5)
        state = keys
        for r in range(1, 4):
            state = orc.count_sort_round(state, r - 1, 256)
            np.testing.assert_array_equal(pr(bsg, keys, 4, 256, rounds=r).output, state)
        np.testing.assert_array_equal(pr(bsg, keys, 3, 65536, rounds=1).output, orc.count_sort_round(keys, 0, 65536))
    finally:
        L.bsg_debug_set_relaxed_passes(prev)
