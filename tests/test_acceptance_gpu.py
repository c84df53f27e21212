"""GPU: acceptance.cpp criteria 1-2 restated through sort_instance /
run_parallel_radix on the device path."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def adversarial(kind, n):
    # acceptance.cpp:60-72
    if kind == 0:
        return np.full(n, 0xABCD1234, np.uint32)
    if kind == 1:
        return (np.arange(n, dtype=np.uint64) * 3).astype(np.uint32)
    return ((n - np.arange(n, dtype=np.uint64)) * 3).astype(np.uint32)


def test_criterion1_oracle_grid(cuda, bsg, orc):
    # acceptance.cpp:85-120: n x (3 seeds + 3 adversarial) x 5 algorithms x p
    A = bsg.Algorithm
    checks = 0
    for n in (0, 1, 2, 10, 1000, 100000, 1000000):
        inputs = [orc.generate_uniform_keys(n, s) for s in (11, 22, 33)] + [adversarial(k, n) for k in range(3)]
        for keys in inputs:
            expected = np.sort(keys)
            for algo in (A.SR4, A.PR4, A.PR2, A.BTN, A.OET):
                ps = [1] if algo == A.SR4 else ([1, 2, 4, 8, 16] if algo == A.BTN else [1, 2, 3, 4, 5, 8, 16])
                for p in ps:
                    inst = bsg.SortInstance(keys, p, algo, 65536 if algo == A.PR2 else 256)
                    out = bsg.sort_instance(inst)
                    assert np.array_equal(out, expected), (algo, n, p)
                    checks += 1
    assert checks == 7 * 6 * (1 + 7 + 7 + 5 + 7)


def test_criterion2_parallel_equals_serial(cuda, bsg, orc):
    # acceptance.cpp:143-161: parallel == serial bit-for-bit over (n, p, r)
    for size in (0, 1, 997, 10000):
        rnd = orc.generate_uniform_keys(size, 5)
        for keys in (rnd, rnd % 31):
            for r in (256, 65536):
                serial = bsg.radix.serial_radix_sort(keys, r)
                for p in (1, 2, 3, 4, 5, 8, 16):
                    prep = bsg.radix.prepare_parallel_radix(keys, p, r)
                    assert np.array_equal(bsg.radix.run_parallel_radix(prep).output, serial), (size, p, r)
