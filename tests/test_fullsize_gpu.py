"""Bit-exact parity at BASELINE.json's FULL config sizes.

The small/mid-size grids in test_radix_gpu / test_netsort_gpu / test_pr_gpu pin
the kernels against the oracle; here every full-size configuration is compared
element for element with a host computation:

- C3: n = 2^28 skewed keys (narrow [0,2^16), Zipf(1.1), all-equal) sorted at
  r = 2^8 and r = 2^16 equal the host sort, and every count_sort_round of the
  Zipf input at full size equals the C oracle's round (radix.hpp:44-65) --
  the rank-first (heavy digit) branch of the one-sweep pass at full tile
  counts.
- C4: all 2^16 arrays x 4096 keys, BTN and OET at p = 2/4/8, equal the
  row-wise host sort; 256 arrays equal the oracle's block states after every
  stage (netsort.hpp:157-199 with a truncated stage table).
- C5: n = 2^33 keys of generate_uniform_keys(n, derive_seed(1,0)), PR4 and PR2
  (p = 8 logical workers), equal the host sort of the same stream, compared
  bucket by bucket (top key byte) -- test_c5_full_size_bit_exact.
"""
import concurrent.futures as cf
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N28 = 1 << 28


def _seed(bsg):
    return bsg.derive_seed(1, 0)


def _sort_dev(torch, bsg, t, bits):
    ctx = bsg._lib.context(0)
    L = bsg._lib.lib()
    out = torch.empty_like(t)
    st = torch.cuda.current_stream().cuda_stream
    assert L.bsg_radix_sort_u32(ctx.handle, t.data_ptr(), out.data_ptr(), t.numel(), bits, 1, st) == 0, \
        bsg._lib.last_error()
    return out


def _round_dev(torch, bsg, t, rnd, bits):
    ctx = bsg._lib.context(0)
    L = bsg._lib.lib()
    out = torch.empty_like(t)
    st = torch.cuda.current_stream().cuda_stream
    assert L.bsg_count_sort_round_u32(ctx.handle, t.data_ptr(), out.data_ptr(), t.numel(), rnd, bits, 1, st) == 0, \
        bsg._lib.last_error()
    return out


def _host(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("kind", [0, 1, 2], ids=["narrow16", "zipf1.1", "all_equal"])
def test_c3_full_size_equals_host_sort(cuda, bsg, kind):
    torch = cuda
    keys = bsg.generate_skewed_keys(N28, _seed(bsg), kind)
    exp = np.sort(keys)
    t = torch.from_numpy(keys.view(np.int32)).cuda()
    for bits in (8, 16):
        np.testing.assert_array_equal(_host(_sort_dev(torch, bsg, t, bits)), exp)


def test_c3_zipf_every_round_vs_oracle(cuda, bsg, orc):
    """Zipf(1.1) at 2^28: P(key = 0) ~ 10.5%, so round 0 (and the rounds whose
    digit is mostly 0) run the rank-first branch; each GPU round is compared
    with the C oracle's count_sort_round on the same input."""
    torch = cuda
    cur = bsg.generate_skewed_keys(N28, _seed(bsg), 1)
    for rnd in range(4):
        t = torch.from_numpy(cur.view(np.int32)).cuda()
        got = _host(_round_dev(torch, bsg, t, rnd, 8))
        exp = orc.count_sort_round(cur, rnd, 256)
        np.testing.assert_array_equal(got, exp, err_msg=f"round {rnd}")
        cur = exp
        del t
    # the 16-bit rounds (r = 2^16, 2 rounds) of the same input
    cur = bsg.generate_skewed_keys(N28, _seed(bsg), 1)
    for rnd in range(2):
        t = torch.from_numpy(cur.view(np.int32)).cuda()
        got = _host(_round_dev(torch, bsg, t, rnd, 16))
        exp = orc.count_sort_round(cur, rnd, 65536)
        np.testing.assert_array_equal(got, exp, err_msg=f"r=2^16 round {rnd}")
        cur = exp
        del t


@pytest.mark.parametrize("network", [0, 1], ids=["BTN", "OET"])
def test_c4_all_arrays_and_stage_states(cuda, bsg, orc, network):
    torch = cuda
    num, ln = 1 << 16, 4096
    keys = bsg.generate_uniform_keys_device(num * ln, _seed(bsg)).view(torch.int32)
    host = _host(keys).reshape(num, ln)
    exp = torch.from_numpy(np.sort(host, axis=1).reshape(-1).view(np.int32)).cuda()
    ctx = bsg._lib.context(0)
    L = bsg._lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    out = torch.empty_like(keys)
    for p in (2, 4, 8):
        out.zero_()
        assert L.bsg_block_network_batched_u32(ctx.handle, network, keys.data_ptr(), out.data_ptr(), num, ln, p, -1,
                                               None, 1, st) == 0, bsg._lib.last_error()
        torch.cuda.synchronize()
        assert bool(torch.equal(out, exp)), f"p={p}: some of the 65536 arrays differ from the host sort"
        # every stage of 256 arrays vs the oracle's block states
        S = orc.schedule(network, p)[0].shape[0]
        sub = 256
        part = torch.empty(sub * ln, dtype=torch.int32, device="cuda")
        for s in range(S):
            assert L.bsg_block_network_batched_u32(ctx.handle, network, keys.data_ptr(), part.data_ptr(), sub, ln,
                                                   p, s, None, 1, st) == 0
            got = _host(part).reshape(sub, ln)
            for i in range(sub):
                want, _ = orc.block_network(network, host[i], p, s)
                np.testing.assert_array_equal(got[i], want, err_msg=f"p={p} stage {s} array {i}")


def _host_bucket_sort(bsg, n, seed, nthreads):
    """The host reference output of config 5, as 256 sorted buckets (top key
    byte): the host generator (core.hpp:93-99) in 2^28-key chunks at stream
    offsets (random access, threads), a stable top-byte partition of each
    chunk, then np.sort per bucket.  Returns the list of sorted buckets."""
    chunk = 1 << 28
    starts = list(range(0, n, chunk))

    def gen_split(a):
        k = bsg.generate_uniform_keys_at(min(chunk, n - a), seed, a)
        k.sort()  # GIL-free; a sorted chunk splits at top-byte boundaries
        cuts = np.searchsorted(k, np.arange(1, 256, dtype=np.uint64) << np.uint64(24))
        return np.split(k, cuts)

    pieces = [[] for _ in range(256)]
    with cf.ThreadPoolExecutor(nthreads) as ex:
        for parts in ex.map(gen_split, starts):
            for b in range(256):
                pieces[b].append(parts[b])

    def sort_bucket(b):
        v = np.concatenate(pieces[b])
        pieces[b] = None
        v.sort()
        return v

    with cf.ThreadPoolExecutor(nthreads) as ex:
        return list(ex.map(sort_bucket, range(256)))


def _host_ram_bytes():
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_AVPHYS_PAGES")
    except (ValueError, OSError):
        return 0


def test_c5_full_size_bit_exact(cuda, bsg):
    """Config 5 at its full size: n = 2^33 keys (32 GiB) of
    generate_uniform_keys(n, derive_seed(1,0)), PR4 (r=2^8) and PR2 (r=2^16)
    with p = 8 logical workers (radix.hpp:260-303), each output compared with
    the host sort of the same stream, bucket by bucket; plus rounds_limit = 1
    equal to one count_sort_round of the whole array.  Uses its own contexts
    (closed at the end) so their ~100 GiB of workspace does not linger."""
    import time

    torch = cuda
    n, p = 1 << 33, 8
    bsg._lib.release_all()  # earlier tests' workspaces (e.g. 2^32-key sorts) must not count against 2^33
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    if free < 17 * n:
        pytest.skip("not enough device memory")
    if _host_ram_bytes() < 12 * n:
        pytest.skip("not enough host memory for the host reference sort")
    seed = _seed(bsg)
    t0 = time.perf_counter()
    exp_buckets = _host_bucket_sort(bsg, n, seed, max(1, min(32, os.cpu_count() or 1)))
    t1 = time.perf_counter()
    keys = bsg.generate_uniform_keys_device(n, seed).view(torch.int32)
    out = torch.empty_like(keys)
    L = bsg._lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    ctx = bsg._lib.Context(0)
    try:
        for bits in (8, 16):
            assert L.bsg_parallel_radix_sort_u32(ctx.handle, keys.data_ptr(), out.data_ptr(), n, p, bits, -1, None,
                                                 1, st) == 0, bsg._lib.last_error()
            torch.cuda.synchronize()
            starts = np.concatenate([[0], np.cumsum([e.size for e in exp_buckets])])
            assert starts[-1] == n

            def check(b):
                got = _host(out[int(starts[b]):int(starts[b + 1])])
                return bool(np.array_equal(got, exp_buckets[b]))

            with cf.ThreadPoolExecutor(8) as ex:
                bad = [b for b, ok in enumerate(ex.map(check, range(256))) if not ok]
            assert not bad, f"r=2^{bits}: buckets {bad[:8]} differ from the host sort"
        del exp_buckets
        t2 = time.perf_counter()
        # rounds_limit = 1: the PR state after one round is one stable
        # count-sort round of the whole concatenation (radix.hpp:44-65, 260-303)
        assert L.bsg_parallel_radix_sort_u32(ctx.handle, keys.data_ptr(), out.data_ptr(), n, p, 8, 1, None, 1,
                                             st) == 0
        torch.cuda.synchronize()
    finally:
        ctx.close()
    ctx2 = bsg._lib.Context(0)
    try:
        exp = torch.empty_like(keys)
        assert L.bsg_count_sort_round_u32(ctx2.handle, keys.data_ptr(), exp.data_ptr(), n, 0, 8, 1, st) == 0
        torch.cuda.synchronize()
        step = 1 << 28
        assert all(bool(torch.equal(out[a:a + step], exp[a:a + step])) for a in range(0, n, step))
    finally:
        ctx2.close()
    print(f"c5: host reference {t1 - t0:.1f} s, GPU sorts + compare {t2 - t1:.1f} s")
    del keys, out, exp
    bsg._lib.release_all()
    torch.cuda.empty_cache()
