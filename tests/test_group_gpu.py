"""Single-process multi-GPU parallel radix sort behind the C ABI
(bsg_ctx_create_group / bsg_pr_group_sort_u32).

The p logical workers of run_parallel_radix (radix.hpp:260-303) are spread
over the members of a group context.  The pool has one GPU, so groups list
cuda:0 several times: every member is its own context with its own stream and
workspace, the count matrix is exchanged between members, the fused rounds
store through the member table and rounds end with cross-member event
barriers -- the multi-GPU code path, with local instead of NVLink stores.
Every round's state is compared with the oracle's run_parallel_radix with
plan.rounds = k, and RunStats with the oracle's."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def groups(cuda, bsg):
    made = {}

    def get(G):
        if G not in made:
            made[G] = bsg._lib.GroupContext([0] * G)
        return made[G]

    yield get
    for g in made.values():
        g.close()


@pytest.mark.parametrize("G", [1, 2, 3, 4])
@pytest.mark.parametrize("radix", [256, 65536])
def test_group_per_round_states(cuda, bsg, orc, groups, G, radix):
    grp = groups(G)
    assert grp.size == G
    keys = orc.generate_uniform_keys(200003, 11 + G) % np.uint32(1 << 31)
    keys[:3000] = 77  # ties spanning several workers' blocks
    rounds = 32 // (radix.bit_length() - 1)
    for p in sorted({G, 2 * G + 1, 8}):
        for k in range(rounds + 1):
            prep = bsg.radix.prepare_parallel_radix(keys, p, radix)
            prep.plan.rounds = k
            res = bsg.radix.run_parallel_radix(prep, group=grp)
            exp, est = orc.parallel_radix(keys, p, radix, k)
            np.testing.assert_array_equal(res.output, exp, err_msg=f"G={G} p={p} round {k}")
            assert res.stats == est, (G, p, k)


def test_group_device_blocks_and_timing(cuda, bsg, orc, groups):
    torch = cuda
    G, p, n = 3, 6, (1 << 22) + 17
    grp = groups(G)
    keys = orc.generate_uniform_keys(n, 5)
    blocks = []
    for g in range(G):
        off, sz = bsg.radix.group_range(n, p, G, g)
        blocks.append(torch.from_numpy(keys[off:off + sz].view(np.int32)).cuda())
    assert sum(b.numel() for b in blocks) == n
    for radix in (256, 65536):
        bl = [b.clone() for b in blocks]
        stats, tm = bsg.radix.group_sort_blocks(grp, bl, n, p, radix, timing=True)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(torch.cat(bl).cpu().numpy().view(np.uint32), np.sort(keys))
        _, est = orc.parallel_radix(keys, p, radix)
        assert stats == est
        assert tm["total_ms"] > 0 and tm["exchange_ms"] > 0 and tm["count_ms"] > 0
        # ~ (G-1)/G of the keys change member every round
        rounds = 32 // (radix.bit_length() - 1)
        assert 0.5 * rounds * 4 * n * (G - 1) / G < tm["remote_bytes"] <= rounds * 4 * n


def test_group_nccl_variant(cuda, bsg, orc):
    """BSG_PR_NCCL: local pass + ncclSend/ncclRecv all-to-all-v + rebuild over
    communicators from ncclCommInitAll (one member: NCCL rejects a device
    listed twice).  p must equal the group size."""
    torch = cuda
    grp = bsg._lib.GroupContext([0])
    try:
        n = 100003
        keys = orc.generate_uniform_keys(n, 8)
        for radix in (256, 65536):
            for k in (1, None):
                b = torch.from_numpy(keys.view(np.int32)).cuda()
                stats, tm = bsg.radix.group_sort_blocks(grp, [b], n, 1, radix, rounds=k, variant=bsg._lib.PR_NCCL,
                                                        timing=True)
                torch.cuda.synchronize()
                exp, est = orc.parallel_radix(keys, 1, radix, -1 if k is None else k)
                np.testing.assert_array_equal(b.cpu().numpy().view(np.uint32), exp)
                assert stats == est
                assert tm["remote_bytes"] == 0
        with pytest.raises(ValueError):
            bsg.radix.group_sort_blocks(grp, [b], n, 2, 256, variant=bsg._lib.PR_NCCL)
    finally:
        grp.close()


def test_group_rejects_bad_arguments(cuda, bsg):
    L = bsg._lib.lib()
    import ctypes

    h = ctypes.c_void_p()
    assert L.bsg_ctx_create_group(None, 0, ctypes.byref(h)) == bsg._lib.BSG_EINVAL
    ctx = bsg._lib.context(0)
    assert L.bsg_ctx_group_size(ctx.handle) == 1
    assert L.bsg_ctx_group_device(ctx.handle, 0) == 0
    # a single-device context is not a group
    arr = (ctypes.c_void_p * 1)(0)
    assert L.bsg_pr_group_sort_u32(ctx.handle, arr, 10, 1, 8, -1, 0, None, None, None) == bsg._lib.BSG_EINVAL
    assert int(L.bsg_group_range_offset(100, 8, 3, 3)) == 100
    assert sum(int(L.bsg_group_range_size(100, 8, 3, g)) for g in range(3)) == 100


def test_group_global_positions_above_2_32(cuda, bsg):
    """n = 2^32 + 5 keys over G = 2 members (p = 4): member ranges are
    ~2^31 keys and global positions exceed 32 bits, so the fused pass runs
    its 64-bit rows.  One round equals one count_sort_round of the whole
    array; the full sort equals the single-GPU sort."""
    torch = cuda
    n, p, G = (1 << 32) + 5, 4, 2
    bsg._lib.release_all()
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    if free < 22 * n:
        pytest.skip("not enough device memory")
    keys = bsg.generate_uniform_keys_device(n, 3).view(torch.int32)
    grp = bsg._lib.GroupContext([0] * G)
    ctx = bsg._lib.Context(0)
    L = bsg._lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    try:
        rng = [bsg.radix.group_range(n, p, G, g) for g in range(G)]
        exp = torch.empty_like(keys)
        for rounds, ref in ((1, "round"), (None, "sort")):
            blocks = [keys[o:o + s].clone() for o, s in rng]
            bsg.radix.group_sort_blocks(grp, blocks, n, p, 256, rounds=rounds)
            if ref == "round":
                assert L.bsg_count_sort_round_u32(ctx.handle, keys.data_ptr(), exp.data_ptr(), n, 0, 8, 1, st) == 0
            else:
                assert L.bsg_radix_sort_u32(ctx.handle, keys.data_ptr(), exp.data_ptr(), n, 8, 1, st) == 0
            torch.cuda.synchronize()
            step = 1 << 28
            for (o, s), b in zip(rng, blocks):
                for a in range(0, s, step):
                    assert bool(torch.equal(b[a:a + step], exp[o + a:o + min(a + step, s)])), (ref, o, a)
            del blocks
    finally:
        grp.close()
        ctx.close()
        del keys
        bsg._lib.release_all()
        torch.cuda.empty_cache()
