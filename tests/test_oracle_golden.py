"""CPU: pins the oracle (oracle/bsg_oracle.c) against the reference's own
known-answer tests and against golden vectors produced by the reference
itself (tests/golden/golden.npz, tests/golden/make_golden.py)."""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def test_frozen_first_draws(orc, golden):
    # core_test.cpp:24-31
    exp = [0x6ee5e2d6, 0xb92502a8, 0x0e5e7b0a, 0x8a1ad34e, 0x4d361955, 0x9c7f4f7c]
    assert orc.generate_uniform_keys(6, 42).tolist() == exp
    assert golden["draws/42/6"].tolist() == exp
    assert orc.generate_uniform_keys(0, 12345).size == 0


def test_generator_determinism_and_uniformity(orc):
    # core_test.cpp:14-20, 36-47
    a = orc.generate_uniform_keys(1000, 42)
    assert (a == orc.generate_uniform_keys(1000, 42)).all()
    assert not (a == orc.generate_uniform_keys(1000, 43)).all()
    keys = orc.generate_uniform_keys(1000000, 7)
    for d in range(4):
        h = np.bincount((keys >> (8 * d)) & 0xFF, minlength=256)
        assert h.min() >= 3595 and h.max() <= 4218


def test_derive_seed(orc):
    # bench_test.cpp:27-31 + splitmix64 restated
    assert orc.derive_seed(42, 0) == orc.derive_seed(42, 0)
    assert orc.derive_seed(42, 0) != orc.derive_seed(42, 1)
    assert orc.derive_seed(42, 0) != orc.derive_seed(43, 0)


def test_count_sort_round_kats(orc):
    # radix_test.cpp:137-151
    assert orc.count_sort_round(np.array([0x0103, 0x0201, 0x0102]), 0, 256).tolist() == [0x0201, 0x0102, 0x0103]
    assert orc.count_sort_round(np.array([0x0101, 0x0001]), 0, 256).tolist() == [0x0101, 0x0001]
    assert orc.count_sort_round(np.array([], np.uint32), 3, 256).size == 0


def test_checked_digit_bits(orc):
    assert [orc.checked_digit_bits(r) for r in (2, 4, 16, 256, 65536)] == [1, 2, 4, 8, 16]
    assert orc.checked_digit_bits(100) == -1 and orc.checked_digit_bits(8) == -1
    assert orc.checked_digit_bits(1 << 32) == -2


def test_oracle_reproduces_golden(orc, golden):
    n = 0
    for key in golden.files:
        parts = key.split("/")
        if parts[0] == "csr":
            radix, rnd, case = int(parts[1]), int(parts[2]), parts[3]
            np.testing.assert_array_equal(orc.count_sort_round(golden[f"in/{case}"], rnd, radix), golden[key], key)
        elif parts[0] == "srs":
            radix, case = int(parts[1]), parts[2]
            np.testing.assert_array_equal(orc.serial_radix_sort(golden[f"in/{case}"], radix), golden[key], key)
        elif parts[0] == "pr":
            radix, p, k = map(int, parts[1:])
            out, st = orc.parallel_radix(golden["in/pr"], p, radix, k)
            np.testing.assert_array_equal(out, golden[key], key)
            exp = golden[f"prstats/{radix}/{p}/{k}"]
            assert [st["supersteps"], st["messages_sent"], st["messages_delivered"], st["words_sent"],
                    st["words_delivered"]] == exp.tolist(), key
        elif parts[0] == "net":
            net = 0 if parts[1] == "btn" else 1
            p, s = int(parts[2]), int(parts[3])
            out, st = orc.block_network(net, golden["in/net"], p, s)
            np.testing.assert_array_equal(out, golden[key], key)
            exp = golden[f"netstats/{parts[1]}/{p}/{s}"]
            assert [st["supersteps"], st["messages_sent"], st["messages_delivered"], st["words_sent"],
                    st["words_delivered"]] == exp.tolist(), key
        elif parts[0] == "ms" and parts[2] == "a":
            i = parts[1]
            lo, hi = orc.merge_split(golden[f"ms/{i}/a"], golden[f"ms/{i}/b"])
            np.testing.assert_array_equal(lo, golden[f"ms/{i}/low"])
            np.testing.assert_array_equal(hi, golden[f"ms/{i}/high"])
        else:
            continue
        n += 1
    assert n > 400


def test_merge_split_kats(orc):
    # netsort_test.cpp:52-82
    ms = orc.merge_split
    assert [x.tolist() for x in ms([1, 2], [3, 4])] == [[1, 2], [3, 4]]
    assert [x.tolist() for x in ms([1, 3, 5], [2, 4, 6])] == [[1, 2, 3], [4, 5, 6]]
    assert [x.tolist() for x in ms([], [1, 2])] == [[], [1, 2]]
    assert [x.tolist() for x in ms([1, 9], [5])] == [[1, 5], [9]]


def _apply_scalar(partner, keep, values):
    values = list(values)
    for s in range(partner.shape[0]):
        for i in range(len(values)):
            q = partner[s, i]
            if q < 0 or q < i:
                continue
            lo, hi = min(values[i], values[q]), max(values[i], values[q])
            values[i], values[q] = (lo, hi) if keep[s, i] else (hi, lo)
    return values


def test_schedules_zero_one_principle(orc):
    # netsort_test.cpp:108-166, acceptance.cpp:182-213
    for p in (1, 2, 4, 8, 16, 64, 256):
        lg = p.bit_length() - 1
        assert orc.schedule(0, p)[0].shape[0] == lg * (lg + 1) // 2
    for p in (2, 4, 8, 16):
        partner, keep = orc.schedule(0, p)
        for s in range(partner.shape[0]):
            for i in range(p):
                q = partner[s, i]
                assert q != i and partner[s, q] == i and keep[s, q] != keep[s, i]
        for mask in range(1 << p):
            v = _apply_scalar(partner, keep, [(mask >> i) & 1 for i in range(p)])
            assert v == sorted(v)
    for p in range(1, 11):
        partner, keep = orc.schedule(1, p)
        for mask in range(1 << p):
            v = _apply_scalar(partner, keep, [(mask >> i) & 1 for i in range(p)])
            assert v == sorted(v)


def test_oracle_vs_reference_live(orc, ref):
    """Where the compiled reference is present (this container), the oracle
    matches it on fresh random cases, including uneven partitions."""
    if ref is None:
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    keys = orc.generate_uniform_keys(20011, 5)
    for p in (1, 2, 3, 7, 16):
        for radix in (256, 65536):
            for k in (-1, 1):
                a, sa = orc.parallel_radix(keys % 1000, p, radix, k)
                b, sb = ref.parallel_radix(keys % 1000, p, radix, k)
                assert (a == b).all() and sa == sb
    for net, ps in ((0, (2, 4, 8)), (1, (3, 5, 6))):
        for p in ps:
            a, sa = orc.block_network(net, keys[:1003], p)
            b, sb = ref.block_network(net, keys[:1003], p)
            assert (a == b).all() and sa == sb
