"""GPU parity of the count-sort round and the serial LSD sort against the
oracle (radix_test.cpp / acceptance.cpp criteria 1-2 restated)."""
import numpy as np
import pytest

from conftest import stable_digit_sort

pytestmark = pytest.mark.gpu


def test_count_sort_round_kats(cuda, bsg):
    # radix_test.cpp:137-151
    assert bsg.radix.count_sort_round(np.array([], np.uint32), 0, 256).size == 0
    assert bsg.radix.count_sort_round(np.array([], np.uint32), 3, 256).size == 0
    out = bsg.radix.count_sort_round(np.array([0x0103, 0x0201, 0x0102], np.uint32), 0, 256)
    assert out.tolist() == [0x0201, 0x0102, 0x0103]
    inp = np.array([0x0101, 0x0001], np.uint32)
    assert bsg.radix.count_sort_round(inp, 0, 256).tolist() == inp.tolist()


def test_count_sort_round_vs_stable_oracle(cuda, bsg, orc):
    # radix_test.cpp:153-166 (40 random arrays, seed 2024, len < 300)
    draws = orc.mt64_draws(40 * 400, 2024)
    pos = 0
    for _ in range(40):
        n = int(draws[pos] % 300); pos += 1
        keys = (draws[pos:pos + n] & 0xFFFFFFFF).astype(np.uint32); pos += n
        for radix in (256, 65536):
            rounds = 32 // (radix.bit_length() - 1)
            rnd = int(draws[pos] % rounds); pos += 1
            got = bsg.radix.count_sort_round(keys, rnd, radix)
            np.testing.assert_array_equal(got, stable_digit_sort(keys, rnd, radix))
            np.testing.assert_array_equal(got, orc.count_sort_round(keys, rnd, radix))


@pytest.mark.parametrize("radix", [2, 4, 16, 256, 65536])
@pytest.mark.parametrize("n", [1, 2, 3, 10, 1000, 8191, 8192, 8193, 100003])
def test_count_sort_round_every_round(cuda, bsg, orc, radix, n):
    keys = orc.generate_uniform_keys(n, 1000 + n)
    rounds = 32 // (radix.bit_length() - 1)
    for rnd in sorted({0, rounds // 2, rounds - 1}):
        np.testing.assert_array_equal(bsg.radix.count_sort_round(keys, rnd, radix),
                                      orc.count_sort_round(keys, rnd, radix))


@pytest.mark.parametrize("seed", [7, 99])
def test_index_tagged_stability(cuda, bsg, orc, seed):
    # radix_test.cpp:67-83 / acceptance.cpp:124-141
    n = 10000
    draws = orc.mt64_draws(n, seed)
    tagged = (((draws % (1 << 18)).astype(np.uint64) << np.uint64(14)) | np.arange(n, dtype=np.uint64)).astype(np.uint32)
    out = bsg.radix.count_sort_round(tagged, 3, 256)
    d = out >> 24
    assert np.all(d[:-1] <= d[1:])
    same = d[:-1] == d[1:]
    assert np.all((out[:-1] & 0x3FFF)[same] < (out[1:] & 0x3FFF)[same])
    np.testing.assert_array_equal(out, orc.count_sort_round(tagged, 3, 256))


def adversarial(kind, n):
    # acceptance.cpp:60-72
    if kind == 0:
        return np.full(n, 0xABCD1234, np.uint32)
    if kind == 1:
        return (np.arange(n, dtype=np.uint64) * 3).astype(np.uint32)
    return ((n - np.arange(n, dtype=np.uint64)) * 3).astype(np.uint32)


@pytest.mark.parametrize("n", [0, 1, 2, 10, 1000, 100000, 1000000])
def test_serial_radix_sort_grid(cuda, bsg, orc, n):
    # acceptance.cpp:85-120 criterion 1 (SR4 column) + both radixes
    inputs = [orc.generate_uniform_keys(n, s) for s in (11, 22, 33)] + [adversarial(k, n) for k in range(3)]
    for keys in inputs:
        expect = np.sort(keys)
        for radix in (256, 65536, 2, 4, 16):
            np.testing.assert_array_equal(bsg.radix.serial_radix_sort(keys, radix), expect)


def test_serial_equals_composed_rounds(cuda, bsg, orc):
    # radix_test.cpp:93-104
    keys = orc.generate_uniform_keys(5000, 11)
    for radix, rounds in ((256, 4), (65536, 2)):
        comp = keys
        for r in range(rounds):
            comp = bsg.radix.count_sort_round(comp, r, radix)
        np.testing.assert_array_equal(bsg.radix.serial_radix_sort(keys, radix), comp)
        np.testing.assert_array_equal(comp, orc.serial_radix_sort(keys, radix))


def test_device_tensors_and_inplace(cuda, bsg, orc):
    torch = cuda
    keys = orc.generate_uniform_keys(1 << 20, 5)
    t = torch.from_numpy(keys.view(np.int32)).cuda().view(torch.uint32)
    out = bsg.radix.serial_radix_sort(t, 256)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), np.sort(keys))
    # in place through the C ABI
    ctx = bsg._lib.context(0)
    rc = bsg._lib.lib().bsg_radix_sort_u32(ctx.handle, t.data_ptr(), t.data_ptr(), t.numel(), 8, 1,
                                           torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    np.testing.assert_array_equal(t.cpu().numpy(), np.sort(keys))


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_skewed_inputs(cuda, bsg, orc, kind):
    keys = bsg.generate_skewed_keys(1 << 22, 3, kind)
    expect = np.sort(keys)
    for radix in (256, 65536):
        np.testing.assert_array_equal(bsg.radix.serial_radix_sort(keys, radix), expect)
    for rnd in range(4):
        np.testing.assert_array_equal(bsg.radix.count_sort_round(keys, rnd, 256), orc.count_sort_round(keys, rnd, 256))


def test_rejects_bad_arguments(cuda, bsg):
    # radix_test.cpp:189-195
    with pytest.raises(ValueError):
        bsg.radix.count_sort_round(np.array([1], np.uint32), 4, 256)
    with pytest.raises(ValueError):
        bsg.radix.count_sort_round(np.array([1], np.uint32), -1, 256)
    with pytest.raises(ValueError):
        bsg.radix.count_sort_round(np.array([1], np.uint32), 0, 100)
    with pytest.raises(ValueError):
        bsg.radix.count_sort_round(np.array([1], np.uint32), 0, 1 << 32)


def test_full_size_2_28_properties(cuda, bsg):
    # config 2 at full size: sortedness + permutation (checksums) on device
    torch = cuda
    n = 1 << 28
    keys = bsg.generate_uniform_keys(n, bsg.derive_seed(1, 0))
    t = torch.from_numpy(keys.view(np.int32)).cuda()
    out = bsg.radix.serial_radix_sort(t.view(torch.uint32), 256).view(torch.int32)
    o64 = out.to(torch.int64) & 0xFFFFFFFF
    assert bool((o64[1:] >= o64[:-1]).all())
    i64 = t.to(torch.int64) & 0xFFFFFFFF
    assert int(o64.sum()) == int(i64.sum())
    assert int((o64 * o64 % 1000003).sum()) == int((i64 * i64 % 1000003).sum())
    ref_sorted = torch.sort(i64).values
    assert bool(torch.equal(ref_sorted, o64))


@pytest.mark.parametrize("offset", [1, 2, 3, 5])
def test_unaligned_device_pointers(cuda, bsg, orc, offset):
    """Misaligned sub-array pointers take the non-TMA load path."""
    torch = cuda
    n = 3 * 16384 + 777
    keys = orc.generate_uniform_keys(n + offset, 99)
    t = torch.from_numpy(keys.view(np.int32)).cuda()
    sub = t[offset:]
    out = torch.empty(n + offset, dtype=torch.int32, device="cuda")[offset:]
    ctx = bsg._lib.context(0)
    L = bsg._lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    for rnd in range(4):
        assert L.bsg_count_sort_round_u32(ctx.handle, sub.data_ptr(), out.data_ptr(), n, rnd, 8, 1, st) == 0
        torch.cuda.synchronize()
        np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), orc.count_sort_round(keys[offset:], rnd, 256))
    assert L.bsg_radix_sort_u32(ctx.handle, sub.data_ptr(), out.data_ptr(), n, 8, 1, st) == 0
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), np.sort(keys[offset:]))


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5, 6, 7])
def test_every_onesweep_configuration(cuda, bsg, orc, cfg):
    """Each THREADS x ITEMS instantiation (auto picks by n) against the oracle,
    on ragged sizes around its tile: partial last tiles, single tiles, ties."""
    L = bsg._lib.lib()
    prev = L.bsg_debug_set_onesweep_cfg(cfg)
    try:
        for n in (1, 4095, 4097, 24577, 3 * 24576 + 7, 1000003):
            keys = orc.generate_uniform_keys(n, 31 + n + cfg)
            np.testing.assert_array_equal(bsg.radix.serial_radix_sort(keys, 256), orc.serial_radix_sort(keys, 256))
            for rnd in (0, 3):
                np.testing.assert_array_equal(bsg.radix.count_sort_round(keys, rnd, 256),
                                              orc.count_sort_round(keys, rnd, 256))
        narrow = (orc.generate_uniform_keys(200003, 5) & 0x0F0F).astype(np.uint32)  # heavy ties
        np.testing.assert_array_equal(bsg.radix.serial_radix_sort(narrow, 256), orc.serial_radix_sort(narrow, 256))
    finally:
        L.bsg_debug_set_onesweep_cfg(prev)


def test_auto_configuration_boundaries(cuda, bsg, orc):
    """Sizes either side of the auto-selection thresholds (2^21, 2^25)."""
    for n in ((1 << 21), (1 << 21) + 1, (1 << 25), (1 << 25) + 1):
        keys = orc.generate_uniform_keys(n, n)
        np.testing.assert_array_equal(bsg.radix.serial_radix_sort(keys, 256), orc.serial_radix_sort(keys, 256))


@pytest.mark.parametrize("small", [0, 1])
def test_small_n_both_paths(cuda, bsg, orc, small):
    """n <= 2^21 runs the fused cooperative sort (one launch); the multi-launch
    path must agree too.  Includes identity passes (narrow keys) and in-place."""
    L = bsg._lib.lib()
    prev = L.bsg_debug_set_small_sort(small)
    try:
        for n in (1, 2, 31, 8191, 8193, 100000, (1 << 20) + 3, 1 << 21):
            keys = orc.generate_uniform_keys(n, 5 * n + small)
            np.testing.assert_array_equal(bsg.radix.serial_radix_sort(keys, 256), orc.serial_radix_sort(keys, 256))
        for mask in (0xFF, 0xFF00FF, 0):  # 3, 2 and 0 identity passes
            keys = orc.generate_uniform_keys(70001, 3) & np.uint32(mask)
            np.testing.assert_array_equal(bsg.radix.serial_radix_sort(keys, 256), np.sort(keys))
        torch = cuda
        keys = orc.generate_uniform_keys(300007, 11)
        t = torch.from_numpy(keys.view(np.int32)).cuda()
        ctx = bsg._lib.context(0)
        st = torch.cuda.current_stream().cuda_stream
        assert L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), t.data_ptr(), keys.size, 8, 1, st) == 0  # in place
        torch.cuda.synchronize()
        np.testing.assert_array_equal(t.cpu().numpy().view(np.uint32), np.sort(keys))
    finally:
        L.bsg_debug_set_small_sort(prev)


def _chunked_properties(torch, inp, out, step=1 << 27):
    """Sortedness (incl. across chunk seams) and permutation checksums
    (sum, sum of squares mod p) without n-sized int64 temporaries."""
    n = inp.numel()
    m = 1000003
    s_in = s_out = q_in = q_out = 0
    prev_last = None
    for a in range(0, n, step):
        x = inp[a:a + step].to(torch.int64) & 0xFFFFFFFF
        y = out[a:a + step].to(torch.int64) & 0xFFFFFFFF
        assert bool((y[1:] >= y[:-1]).all())
        if prev_last is not None:
            assert int(y[0]) >= prev_last
        prev_last = int(y[-1])
        s_in += int(x.sum()); s_out += int(y.sum())
        q_in += int(((x % m) * (x % m) % m).sum()); q_out += int(((y % m) * (y % m) % m).sum())
        del x, y
    assert s_in == s_out and q_in == q_out


@pytest.mark.parametrize("n", [(1 << 29) + 12345, (1 << 32) + 777])
def test_multi_chunk_and_wide_positions(cuda, bsg, n):
    """n > 2^29: several look-back chunks per pass; n > 2^32: 64-bit positions
    (WIDE one-sweep).  ~48 GiB of device buffers at the larger size."""
    torch = cuda
    free, _ = torch.cuda.mem_get_info()
    if free < 14 * n:
        pytest.skip("not enough device memory")
    g = torch.Generator(device="cuda").manual_seed(n)
    inp = torch.randint(-2**31, 2**31, (n,), dtype=torch.int32, device="cuda", generator=g)
    inp[:1000] = 7  # ties across the first tiles
    out = torch.empty_like(inp)
    ctx = bsg._lib.context(0)
    L = bsg._lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    assert L.bsg_radix_sort_u32(ctx.handle, inp.data_ptr(), out.data_ptr(), n, 8, 1, st) == 0
    torch.cuda.synchronize()
    _chunked_properties(torch, inp, out)
    # one stable pass at the top digit: a count-sort round over all chunks
    assert L.bsg_count_sort_round_u32(ctx.handle, inp.data_ptr(), out.data_ptr(), n, 3, 8, 1, st) == 0
    torch.cuda.synchronize()
    step = 1 << 27
    prev = -1
    for a in range(0, n, step):
        d = (out[a:a + step].to(torch.int64) & 0xFFFFFFFF) >> 24
        assert bool((d[1:] >= d[:-1]).all()) and int(d[0]) >= prev
        prev = int(d[-1])
    del inp, out
    bsg._lib.release_all()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n", [1, 311, 312, 313, 100003, (1 << 18) + 1, (1 << 20) + 7, 3 << 20])
def test_device_generator_matches_host_stream(cuda, bsg, n):
    """generate_uniform_keys on the GPU (segment starts by jump-ahead) is the
    host stream bit for bit; n > 2^18 spans several segments."""
    torch = cuda
    L = bsg._lib.lib()
    ctx = bsg._lib.context(0)
    st = torch.cuda.current_stream().cuda_stream
    for seed in (bsg.derive_seed(1, 0), 7):
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        assert L.bsg_generate_uniform_device_u32(ctx.handle, out.data_ptr(), n, seed, st) == 0
        torch.cuda.synchronize()
        np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), bsg.generate_uniform_keys(n, seed))


@pytest.mark.parametrize("offset", [1, 311, 312, 100003, (1 << 30) + 5, (1 << 32) - 17])
def test_device_generator_at_offset(cuda, bsg, orc, offset):
    """bsg_generate_uniform_device_at_u32: keys [offset, offset + n) of the
    host stream (a rank's block of config 5's block-distributed input)."""
    n = (1 << 19) + 3
    seed = bsg.derive_seed(1, 0)
    got = bsg.generate_uniform_keys_device(n, seed, offset=offset).cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(got, bsg.generate_uniform_keys_at(n, seed, offset))
    if offset < 200000:
        np.testing.assert_array_equal(got, orc.generate_uniform_keys(offset + n, seed)[offset:])


def test_in_place_calls(cuda, bsg, orc):
    """in == out device pointers: count-sort round, block networks and the
    in-process parallel radix sort."""
    torch = cuda
    L = bsg._lib.lib()
    ctx = bsg._lib.context(0)
    st = torch.cuda.current_stream().cuda_stream
    for n in (1000, 70001, (1 << 21) + 3, 3 << 22):
        keys = orc.generate_uniform_keys(n, n + 1)
        t = torch.from_numpy(keys.view(np.int32)).cuda()
        assert L.bsg_count_sort_round_u32(ctx.handle, t.data_ptr(), t.data_ptr(), n, 1, 8, 1, st) == 0
        torch.cuda.synchronize()
        np.testing.assert_array_equal(t.cpu().numpy().view(np.uint32), orc.count_sort_round(keys, 1, 256))
        t = torch.from_numpy(keys.view(np.int32)).cuda()
        assert L.bsg_parallel_radix_sort_u32(ctx.handle, t.data_ptr(), t.data_ptr(), n, 3, 8, -1, None, 1, st) == 0
        torch.cuda.synchronize()
        np.testing.assert_array_equal(t.cpu().numpy().view(np.uint32), np.sort(keys))
        # in place with 1 and 2 rounds (the fused rounds read the input and
        # write the output directly; a single round over in == out goes
        # through the workspace)
        for bits, rounds in ((8, 1), (8, 2), (16, 1), (16, 2)):
            t = torch.from_numpy(keys.view(np.int32)).cuda()
            assert L.bsg_parallel_radix_sort_u32(ctx.handle, t.data_ptr(), t.data_ptr(), n, 3, bits, rounds, None, 1,
                                                 st) == 0
            torch.cuda.synchronize()
            exp, _ = orc.parallel_radix(keys, 3, 1 << bits, rounds)
            np.testing.assert_array_equal(t.cpu().numpy().view(np.uint32), exp)
    arrs = orc.generate_uniform_keys(64 * 4096, 3).reshape(64, 4096)
    t = torch.from_numpy(arrs.reshape(-1).view(np.int32)).cuda()
    assert L.bsg_block_network_batched_u32(ctx.handle, 0, t.data_ptr(), t.data_ptr(), 64, 4096, 8, -1, None, 1,
                                           st) == 0
    torch.cuda.synchronize()
    np.testing.assert_array_equal(t.cpu().numpy().view(np.uint32).reshape(64, 4096), np.sort(arrs, axis=1))


def test_one_context_two_streams(cuda, bsg, orc):
    """Device-mode calls on ONE context issued on two different streams share
    the context's workspace (tmp / status / hist); the context orders each
    call after the previous one (bsg_ctx::last_use), so back-to-back sorts on
    two streams with no host sync in between both come out right."""
    torch = cuda
    ctx = bsg._lib.context(0)
    L = bsg._lib.lib()
    n = (1 << 24) + 3
    a = torch.from_numpy(orc.generate_uniform_keys(n, 71).view(np.int32)).cuda()
    b = torch.from_numpy(orc.generate_uniform_keys(n, 72).view(np.int32)).cuda()
    oa, ob = torch.empty_like(a), torch.empty_like(b)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    for _ in range(3):
        assert L.bsg_radix_sort_u32(ctx.handle, a.data_ptr(), oa.data_ptr(), n, 8, 1, s1.cuda_stream) == 0
        assert L.bsg_radix_sort_u32(ctx.handle, b.data_ptr(), ob.data_ptr(), n, 8, 1, s2.cuda_stream) == 0
        assert L.bsg_count_sort_round_u32(ctx.handle, a.data_ptr(), oa.data_ptr(), n, 1, 8, 1, s1.cuda_stream) == 0
        assert L.bsg_radix_sort_u32(ctx.handle, b.data_ptr(), ob.data_ptr(), n, 8, 1, s2.cuda_stream) == 0
    torch.cuda.synchronize()
    np.testing.assert_array_equal(oa.cpu().numpy().view(np.uint32),
                                  orc.count_sort_round(a.cpu().numpy().view(np.uint32), 1, 256))
    np.testing.assert_array_equal(ob.cpu().numpy().view(np.uint32), np.sort(b.cpu().numpy().view(np.uint32)))


def test_aliased_outputs(cuda, bsg, orc):
    """Partially aliased device arguments give the non-aliased result:
    merge_split with low == a / high == b (netsort.hpp:30-51), and a
    truncated network (padded intermediate state, out_per > len) written over
    its own input."""
    torch = cuda
    L = bsg._lib.lib()
    ctx = bsg._lib.context(0)
    st = torch.cuda.current_stream().cuda_stream
    a = np.sort(orc.generate_uniform_keys(300001, 5))
    b = np.sort(orc.generate_uniform_keys(200003, 6))
    lo_e, hi_e = orc.merge_split(a, b)
    ta = torch.from_numpy(a.view(np.int32)).cuda()
    tb = torch.from_numpy(b.view(np.int32)).cuda()
    assert L.bsg_merge_split_u32(ctx.handle, ta.data_ptr(), a.size, tb.data_ptr(), b.size, ta.data_ptr(),
                                 tb.data_ptr(), 1, st) == 0
    torch.cuda.synchronize()
    np.testing.assert_array_equal(ta.cpu().numpy().view(np.uint32), lo_e)
    np.testing.assert_array_equal(tb.cpu().numpy().view(np.uint32), hi_e)
    # swapped roles: low over b's storage is too small unless |a| == |b|
    a2, b2 = a[:200003], b
    lo_e, hi_e = orc.merge_split(a2, b2)
    ta = torch.from_numpy(a2.view(np.int32)).cuda()
    tb = torch.from_numpy(b2.view(np.int32)).cuda()
    assert L.bsg_merge_split_u32(ctx.handle, ta.data_ptr(), a2.size, tb.data_ptr(), b2.size, tb.data_ptr(),
                                 ta.data_ptr(), 1, st) == 0
    torch.cuda.synchronize()
    np.testing.assert_array_equal(tb.cpu().numpy().view(np.uint32), lo_e)
    np.testing.assert_array_equal(ta.cpu().numpy().view(np.uint32), hi_e)
    # truncated network, len not divisible by p: out_per = padded > len
    num, ln, p = 97, 1001, 8
    arrs = orc.generate_uniform_keys(num * ln, 9).reshape(num, ln)
    Lb = (ln + p - 1) // p
    buf = torch.zeros(num * Lb * p, dtype=torch.int32, device="cuda")
    buf[:num * ln] = torch.from_numpy(arrs.reshape(-1).view(np.int32)).cuda()
    for stages in (0, 2):
        t = buf.clone()
        assert L.bsg_block_network_batched_u32(ctx.handle, 0, t.data_ptr(), t.data_ptr(), num, ln, p, stages, None,
                                               1, st) == 0
        torch.cuda.synchronize()
        got = t.cpu().numpy().view(np.uint32).reshape(num, Lb * p)
        for i in (0, 1, 50, num - 1):
            exp, _ = orc.block_network(0, arrs[i], p, stages)
            np.testing.assert_array_equal(got[i], exp)


def test_pageable_host_staging(cuda, bsg, orc):
    """BSG_MEM_HOST with pageable numpy buffers above the 4 MiB direct-copy
    threshold runs the pinned two-chunk pipeline (staging.cu) both ways:
    odd sizes, several 64 MiB chunks, a misaligned host pointer."""
    for n in ((1 << 20) + 1, (1 << 26) + 12345):
        keys = orc.generate_uniform_keys(n + 1, n)
        view = keys[1:]  # misaligned host start (4-byte offset)
        out = bsg.radix.count_sort_round(view, 2, 256)
        np.testing.assert_array_equal(out, orc.count_sort_round(view, 2, 256))
    keys = orc.generate_uniform_keys((1 << 25) + 7, 3)
    np.testing.assert_array_equal(bsg.radix.serial_radix_sort(keys, 256), np.sort(keys))


@pytest.mark.parametrize("first", [0, 1])
def test_first_pass_both_paths(cuda, bsg, orc, first):
    """Pass 0 of a full sort runs K3f (no order inside a digit run, per-tile
    run reservations by global atomics) or the stable K3: both must give the
    oracle's sorted array.  Ragged sizes for both tile rows (8192 and 12288
    keys), misaligned device pointers (head keys outside the TMA body), skewed
    and two-valued low bytes (counter contention), and a narrow input whose
    pass 0 is an identity pass."""
    torch = cuda
    L = bsg._lib.lib()
    prev_small = L.bsg_debug_set_small_sort(0)
    prev = L.bsg_debug_set_first_pass(first)
    try:
        for n in (1, 5, 8191, 8193, 12289, 100003, (1 << 21) + 1, (1 << 25) + 12345):
            keys = orc.generate_uniform_keys(n, 77 * n + first)
            np.testing.assert_array_equal(bsg.radix.serial_radix_sort(keys, 256), np.sort(keys))
        n = 3 * 12288 + 1001
        base = orc.generate_uniform_keys(n, 4242)
        inputs = [
            (base & 0xFFFFFF01).astype(np.uint32),             # two values of digit 0
            ((base >> 8) << 8 | (base % 3 == 0)).astype(np.uint32),  # digit 0 mostly 0
            (base & 0xFFFFFF00).astype(np.uint32),             # pass 0 is an identity pass
            np.minimum(np.random.default_rng(9).zipf(1.1, n), 0xFFFFFFFF).astype(np.uint32),  # Zipf ranks
        ]
        for keys in inputs:
            np.testing.assert_array_equal(bsg.radix.serial_radix_sort(keys, 256), np.sort(keys))
            np.testing.assert_array_equal(bsg.radix.serial_radix_sort(keys, 65536), np.sort(keys))
        ctx = bsg._lib.context(0)
        st = torch.cuda.current_stream().cuda_stream
        for offset in (1, 2, 3):
            keys = orc.generate_uniform_keys(n + offset, 500 + offset)
            t = torch.from_numpy(keys.view(np.int32)).cuda()
            out = torch.empty(n + offset, dtype=torch.int32, device="cuda")[offset:]
            assert L.bsg_radix_sort_u32(ctx.handle, t[offset:].data_ptr(), out.data_ptr(), n, 8, 1, st) == 0
            torch.cuda.synchronize()
            np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), np.sort(keys[offset:]))
    finally:
        L.bsg_debug_set_first_pass(prev)
        L.bsg_debug_set_small_sort(prev_small)


@pytest.mark.parametrize("relaxed", [0, 1])
def test_relaxed_passes_both_paths(cuda, bsg, orc, relaxed):
    """Passes k > 0 of a full sort rank value-stably (keys equal in the low 8k
    bits and in the digit take their slots by shared-memory atomics; runs of
    items with different low bits fall back to the ballot multisplit) or
    strictly stably: both must give the oracle's sorted array.  The relaxation
    applies from 2^24 keys: sizes below it (strict either way), both tile rows
    above it (2^25: 8192-key tiles, pass 1 only; 2^26: 12288-key tiles, passes
    1-2 with runs of 2^18 and 2^10 keys, so most warps of pass 2 meet a run
    boundary); inputs with few or skewed low-bits values, long runs of fully
    equal keys and run boundaries inside warp items."""
    L = bsg._lib.lib()
    prev_small = L.bsg_debug_set_small_sort(0)
    prev = L.bsg_debug_set_relaxed_passes(relaxed)
    try:
        for n in ((1 << 17) + 3, (1 << 22) + 1, (1 << 25) + 12345, (1 << 26) + 77):
            keys = orc.generate_uniform_keys(n, 31 * n + relaxed)
            np.testing.assert_array_equal(bsg.radix.serial_radix_sort(keys, 256), np.sort(keys))
        n = (1 << 24) + 4099
        base = orc.generate_uniform_keys(n, 990)
        rng = np.random.default_rng(5)
        inputs = [
            (base & 0xFFFF0003).astype(np.uint32),                  # 4 low-byte values, byte 1 constant
            (base & 0xFF00FFFF).astype(np.uint32),                  # byte 2 constant (identity pass in between)
            ((base & 0xFFFFFF00) | (base % 7 == 0)).astype(np.uint32),  # low byte 0 for 6/7 of the keys
            rng.choice(base[:1000], n).astype(np.uint32),           # 1000 distinct keys, long equal runs
            ((base & 0xFFFF0000) | (np.arange(n) % 37)).astype(np.uint32),  # low-bits runs of n/37 keys
            np.minimum(rng.zipf(1.1, n), 0xFFFFFFFF).astype(np.uint32),
        ]
        for keys in inputs:
            np.testing.assert_array_equal(bsg.radix.serial_radix_sort(keys, 256), np.sort(keys))
            np.testing.assert_array_equal(bsg.radix.serial_radix_sort(keys, 65536), np.sort(keys))
    finally:
        L.bsg_debug_set_relaxed_passes(prev)
        L.bsg_debug_set_small_sort(prev_small)


def test_hybrid_route_and_its_fallbacks(cuda, bsg, orc):
    """Full sorts of large evenly spread inputs may take the hybrid route
    (msd.cu: two unordered byte partitions of the top 16 bits, then a local
    sort of every top-16-bit bucket); whatever it cannot take falls back to
    the LSD sort on the device.  Forced on for every size here: uniform keys
    (the route itself, ragged sizes, misaligned pointers), a bucket above the
    local sort's capacity (the plan declines), more than 15 equal keys in one
    bucket (the local sort gives up and the LSD sort re-sorts the untouched
    input), duplicate-heavy and skewed keys, and in-place calls (never routed).
    Every result must equal the oracle's sorted array."""
    torch = cuda
    L = bsg._lib.lib()
    ctx = bsg._lib.context(0)
    st = torch.cuda.current_stream().cuda_stream
    prev = L.bsg_debug_set_msd(2)

    def dev_sort(keys, offset=0, inplace=False):
        t = torch.from_numpy(np.concatenate([np.zeros(offset, np.uint32), keys]).view(np.int32)).cuda()
        src = t[offset:]
        out = src if inplace else torch.empty(keys.size + offset, dtype=torch.int32, device="cuda")[offset:]
        assert L.bsg_radix_sort_u32(ctx.handle, src.data_ptr(), out.data_ptr(), keys.size, 8, 1, st) == 0
        torch.cuda.synchronize()
        if not inplace:
            np.testing.assert_array_equal(src.cpu().numpy().view(np.uint32), keys)  # the input is never written
        return out.cpu().numpy().view(np.uint32)

    try:
        for n in (1, 2, 5, 8191, 100003, (1 << 20) + 1, (1 << 24) + 7, (1 << 26) + 12345):
            keys = orc.generate_uniform_keys(n, 11 * n + 3)
            np.testing.assert_array_equal(dev_sort(keys), np.sort(keys))
        n = 300007
        base = orc.generate_uniform_keys(n, 99)
        rng = np.random.default_rng(12)
        cases = {
            "one top-16 value (bucket above capacity)": ((base & 0xFFFF) | 0x12340000).astype(np.uint32),
            "20 equal keys among uniform ones": np.concatenate([base, np.full(20, base[7], np.uint32)]),
            "every key 16 times": np.repeat(base[: n // 16], 16),
            "every key 17 times": np.repeat(base[: n // 17], 17),
            "1000 distinct keys": rng.choice(base[:1000], n).astype(np.uint32),
            "zipf": np.minimum(rng.zipf(1.1, n), 0xFFFFFFFF).astype(np.uint32),
            "all equal": np.full(n, 0xDEADBEEF, np.uint32),
            "low 16 bits constant": (base & 0xFFFF0000).astype(np.uint32),
            "sorted": np.sort(base),
            "reverse sorted": np.sort(base)[::-1].copy(),
        }
        for name, keys in cases.items():
            np.testing.assert_array_equal(dev_sort(keys), np.sort(keys), err_msg=name)
        keys = orc.generate_uniform_keys((1 << 22) + 5, 8)
        for offset in (1, 2, 3):
            np.testing.assert_array_equal(dev_sort(keys, offset=offset), np.sort(keys))
        np.testing.assert_array_equal(dev_sort(keys, inplace=True), np.sort(keys))
        # host-memory entry (staged through the context's device buffers)
        np.testing.assert_array_equal(bsg.radix.serial_radix_sort(keys, 256), np.sort(keys))
        np.testing.assert_array_equal(bsg.radix.serial_radix_sort(keys, 65536), np.sort(keys))
    finally:
        L.bsg_debug_set_msd(prev)


def test_hybrid_route_in_its_size_window(cuda, bsg):
    """Left to itself the library takes the hybrid route (msd.cu) for full
    sorts of a little more than 2^28 keys: 1.125 x 2^28 uniform keys run
    through it (its kernels are launched and the LSD passes stay idle) and the
    result equals an independent device sort; the same keys with one top-16
    value heavier than a bucket may be are declined by its plan on the device
    and sorted by the LSD passes."""
    torch = cuda
    from paper_1708_09495_b200 import _lib
    L = _lib.lib()
    ctx = _lib.context(0)
    st = torch.cuda.current_stream().cuda_stream
    assert L.bsg_debug_set_msd(-1) == 0  # auto
    n = (1 << 28) + (1 << 25) + 12345
    t = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.check(L.bsg_generate_uniform_device_u32(ctx.handle, t.data_ptr(), n, bsg.derive_seed(7, 1), st))
    out = torch.empty_like(t)

    def run_and_times():
        ctx.set_timing(False)
        ctx.set_timing(True)
        _lib.check(L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), n, 8, 1, st))
        torch.cuda.synchronize()
        r = {k: ctx.kernel_time(getattr(_lib, k)) for k in ("K_MSD_LOCAL", "K_ONESWEEP", "K_RELAXED_PASS", "K_FIRST_PASS")}
        ctx.set_timing(False)
        return r

    def expect():
        return torch.sort(t.view(torch.uint32).to(torch.int64))[0].to(torch.uint32).view(torch.int32)

    kt = run_and_times()
    assert torch.equal(out, expect())
    assert kt["K_MSD_LOCAL"][1] == 1 and kt["K_MSD_LOCAL"][0] > 0.5, kt  # the local sort did the work ...
    lsd_ms = kt["K_ONESWEEP"][0] + kt["K_RELAXED_PASS"][0] + kt["K_FIRST_PASS"][0]
    assert lsd_ms < 0.2, kt  # ... and the LSD passes exited at once
    t[: 10000] = (t[: 10000] & 0xFFFF) | 0x7FFF0000  # bucket 0x7FFF: 4608 + 10000 keys > capacity
    out.zero_()
    kt = run_and_times()
    assert torch.equal(out, expect())
    lsd_ms = kt["K_ONESWEEP"][0] + kt["K_RELAXED_PASS"][0] + kt["K_FIRST_PASS"][0]
    assert kt["K_MSD_LOCAL"][0] < 0.2 and lsd_ms > 1.0, kt  # declined: the LSD passes sorted
    del t, out
    torch.cuda.empty_cache()
