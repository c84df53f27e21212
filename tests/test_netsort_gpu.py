"""GPU parity of merge_split and the batched BTN/OET block networks
(netsort_test.cpp, acceptance.cpp criterion 1/3 restated)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_merge_split_kats(cuda, bsg):
    ms = bsg.netsort.merge_split
    u = lambda x: np.array(x, np.uint32)
    lo, hi = ms(u([1, 2]), u([3, 4])); assert lo.tolist() == [1, 2] and hi.tolist() == [3, 4]
    lo, hi = ms(u([1, 3, 5]), u([2, 4, 6])); assert lo.tolist() == [1, 2, 3] and hi.tolist() == [4, 5, 6]
    lo, hi = ms(u([7, 7]), u([7, 7])); assert lo.tolist() == [7, 7] and hi.tolist() == [7, 7]
    lo, hi = ms(u([]), u([1, 2])); assert lo.tolist() == [] and hi.tolist() == [1, 2]
    lo, hi = ms(u([1, 9]), u([5])); assert lo.tolist() == [1, 5] and hi.tolist() == [9]


def test_merge_split_vs_oracle(cuda, bsg, orc):
    draws = orc.mt64_draws(60 * 110, 77)
    pos = 0
    for _ in range(60):
        na = int(draws[pos] % 50); nb = int(draws[pos + 1] % 50); pos += 2
        a = np.sort((draws[pos:pos + na] % 1000).astype(np.uint32)); pos += na
        b = np.sort((draws[pos:pos + nb] % 1000).astype(np.uint32)); pos += nb
        lo, hi = bsg.netsort.merge_split(a, b)
        elo, ehi = orc.merge_split(a, b)
        np.testing.assert_array_equal(lo, elo)
        np.testing.assert_array_equal(hi, ehi)
    a = np.sort(orc.generate_uniform_keys(300000, 1)); b = np.sort(orc.generate_uniform_keys(200001, 2))
    lo, hi = bsg.netsort.merge_split(a, b)
    elo, ehi = orc.merge_split(a, b)
    np.testing.assert_array_equal(lo, elo)
    np.testing.assert_array_equal(hi, ehi)


@pytest.mark.parametrize("p", [1, 2, 4, 8, 16])
def test_btn_matches_oracle(cuda, bsg, orc, p):
    keys = orc.generate_uniform_keys(10000, 31)
    inst = bsg.SortInstance(keys, p, bsg.Algorithm.BTN)
    np.testing.assert_array_equal(bsg.netsort.btn_sort(inst), np.sort(keys))


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 7, 8, 16])
def test_oet_matches_oracle(cuda, bsg, orc, p):
    keys = orc.generate_uniform_keys(10000, 23)
    inst = bsg.SortInstance(keys, p, bsg.Algorithm.OET)
    np.testing.assert_array_equal(bsg.netsort.oet_sort(inst), np.sort(keys))


def test_oet_reverse_blocks(cuda, bsg):
    # netsort_test.cpp:211-224
    inst = bsg.SortInstance(np.array([7, 8, 5, 6, 3, 4, 1, 2], np.uint32), 4, bsg.Algorithm.OET)
    assert bsg.netsort.oet_sort(inst).tolist() == [1, 2, 3, 4, 5, 6, 7, 8]
    rev = (9000 - np.arange(9000)).astype(np.uint32)
    for p in (3, 5, 8):
        np.testing.assert_array_equal(bsg.netsort.oet_sort(bsg.SortInstance(rev, p, bsg.Algorithm.OET)), np.sort(rev))


def test_padding_and_max_keys(cuda, bsg, orc):
    # netsort_test.cpp:234-249
    keys = orc.generate_uniform_keys(1003, 19)
    keys[0] = 0xFFFFFFFF; keys[500] = 0xFFFFFFFF
    for p in (2, 4, 8):
        np.testing.assert_array_equal(bsg.netsort.btn_sort(bsg.SortInstance(keys, p, bsg.Algorithm.BTN)), np.sort(keys))
    for p in (3, 6):
        np.testing.assert_array_equal(bsg.netsort.oet_sort(bsg.SortInstance(keys, p, bsg.Algorithm.OET)), np.sort(keys))
    allmax = np.full(37, 0xFFFFFFFF, np.uint32)
    assert bsg.netsort.btn_sort(bsg.SortInstance(allmax, 4, bsg.Algorithm.BTN)).tolist() == allmax.tolist()
    assert bsg.netsort.oet_sort(bsg.SortInstance(allmax, 5, bsg.Algorithm.OET)).tolist() == allmax.tolist()


@pytest.mark.parametrize("network,ps", [(0, [2, 4, 8, 16]), (1, [2, 3, 4, 5, 8])])
def test_per_stage_states(cuda, bsg, orc, network, ps):
    # truncated stage tables give the intermediate block states
    for p in ps:
        n = 4096 - 4096 % p
        keys = orc.generate_uniform_keys(n, 5 + p)
        S = orc.schedule(network, p)[0].shape[0]
        for s in range(S + 1):
            got, st = bsg.netsort.block_network_batched(keys.reshape(1, n), p, network, s)
            exp, est = orc.block_network(network, keys, p, s)
            np.testing.assert_array_equal(got.reshape(-1), exp)
            assert st == est


@pytest.mark.parametrize("length", [256, 1000, 4096, 16384])
@pytest.mark.parametrize("p", [2, 4, 8])
def test_batched_vs_oracle(cuda, bsg, orc, length, p):
    num = 64
    keys = orc.generate_uniform_keys(num * length, 1234 + length)
    arrs = keys.reshape(num, length)
    for network in (0, 1):
        got, _ = bsg.netsort.block_network_batched(arrs, p, network)
        for i in (0, 17, num - 1):
            exp, _ = orc.block_network(network, arrs[i], p)
            np.testing.assert_array_equal(got[i], exp)
        np.testing.assert_array_equal(got, np.sort(arrs, axis=1))


@pytest.mark.parametrize("n,p", [(100000, 16), (1000000, 8), (16385, 2), (100003, 5)])
def test_large_arrays_global_path(cuda, bsg, orc, n, p):
    """Arrays larger than the shared-memory path (p*ceil(n/p) > 16384):
    netsort_test.cpp:174-180 (10^5 keys, p up to 16) and acceptance sizes."""
    keys = orc.generate_uniform_keys(n, 31 + p)
    if (p & (p - 1)) == 0:
        np.testing.assert_array_equal(bsg.netsort.btn_sort(bsg.SortInstance(keys, p, bsg.Algorithm.BTN)), np.sort(keys))
    np.testing.assert_array_equal(bsg.netsort.oet_sort(bsg.SortInstance(keys, p, bsg.Algorithm.OET)), np.sort(keys))


@pytest.mark.parametrize("network,p", [(0, 4), (0, 8), (1, 3), (1, 6)])
def test_large_arrays_per_stage_states(cuda, bsg, orc, network, p):
    n = 40000 - 40000 % p
    keys = orc.generate_uniform_keys(n, 7 + p)
    S = orc.schedule(network, p)[0].shape[0]
    for s in range(S + 1):
        got, st = bsg.netsort.block_network_batched(keys.reshape(1, n), p, network, s)
        exp, est = orc.block_network(network, keys, p, s)
        np.testing.assert_array_equal(got.reshape(-1), exp)
        assert st == est


@pytest.mark.parametrize("network,p", [(0, 2), (0, 8), (1, 3), (1, 7)])
def test_resident_1024_thread_path_per_stage(cuda, bsg, orc, network, p):
    """Padded arrays of 8193..16384 keys run on the 1024-thread instantiation;
    ragged lengths (pads inside the last block), every truncated stage."""
    for n in (8193 + p, 12001, 16384 - 16384 % p):
        if n // p * p != n and network == 0:
            n -= n % p
        keys = orc.generate_uniform_keys(n, 99 + n + p)
        S = orc.schedule(network, p)[0].shape[0]
        for s in sorted({0, 1, S // 2, S}):
            got, st = bsg.netsort.block_network_batched(keys.reshape(1, n), p, network, s)
            exp, est = orc.block_network(network, keys, p, s)
            np.testing.assert_array_equal(got.reshape(-1), exp)
            assert st == est


@pytest.mark.parametrize("network,p,L", [(1, 3, 16), (1, 3, 512), (1, 5, 64), (1, 7, 2048), (0, 4, 16),
                                         (0, 2, 8192), (1, 6, 256), (0, 16, 32)])
def test_register_network_shapes_per_stage(cuda, bsg, orc, network, p, L):
    """The register network runs every power-of-two block length, including
    non-power-of-two OET worker counts (CTAs padded with idle dummy threads,
    e.g. p = 3, L = 16: 85 arrays of 48 keys on 256 threads) and ragged last
    arrays of a batch; every truncated stage table vs the oracle."""
    n = p * L
    num = 37
    keys = orc.generate_uniform_keys(num * n, 1000 + p * L + network)
    arrs = keys.reshape(num, n)
    S = orc.schedule(network, p)[0].shape[0]
    for s in sorted({0, 1, S // 2, S}):
        got, st = bsg.netsort.block_network_batched(arrs, p, network, s)
        for i in (0, num // 2, num - 1):
            exp, est = orc.block_network(network, arrs[i], p, s)
            np.testing.assert_array_equal(got[i], exp)
            assert st == est
    # ragged last block (len not a multiple of p, same power-of-two L)
    m = n - 3
    got, _ = bsg.netsort.block_network_batched(keys[:num * m].reshape(num, m), p, network)
    np.testing.assert_array_equal(got, np.sort(keys[:num * m].reshape(num, m), axis=1))
