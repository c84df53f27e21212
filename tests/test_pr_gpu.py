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
