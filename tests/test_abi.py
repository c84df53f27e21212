"""CPU: the C-ABI library loads and exports every symbol include/bsg.h
declares; host-only helpers agree with the oracle; compute entry points fail
loudly (no CPU fallback) when no GPU is present."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "bsg.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bsg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(bsg):
    lib = bsg._lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
        assert s in bsg._lib.SIGNATURES, s
    assert lib.bsg_abi_version() == 2


def test_cpp_header_mirror_compiles():
    """include/bspsort_b200/bspsort.hpp (the C++ mirror of the reference API)
    compiles against bsg.h with the host compiler."""
    import subprocess, tempfile

    src = '#include "bspsort_b200/bspsort.hpp"\nint main(){ bspsort::SortInstance s; s.validate(); return 0; }\n'
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.cpp")
        open(p, "w").write(src)
        r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), p],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


def test_host_generator_matches_oracle(bsg, orc):
    for n, seed in ((6, 42), (1000, 7), (12345, 2 ** 63 + 5)):
        np.testing.assert_array_equal(bsg.generate_uniform_keys(n, seed), orc.generate_uniform_keys(n, seed))
    for rep in range(5):
        assert bsg.derive_seed(1, rep) == orc.derive_seed(1, rep)


def test_skewed_generators(bsg):
    a = bsg.generate_skewed_keys(100000, 3, 0)
    assert a.max() <= 0xFFFF
    z = bsg.generate_skewed_keys(200000, 3, 1, 1.1)
    assert (z == bsg.generate_skewed_keys(200000, 3, 1, 1.1)).all()
    frac0 = (z == 0).mean()
    assert 0.09 < frac0 < 0.12  # P(key=0) ~ 1/H(2^32, 1.1) ~ 10.5%
    assert 0.45 < (z < 256).mean() < 0.57
    assert (bsg.generate_skewed_keys(10, 1, 2) == 0xABCD1234).all()


def test_partition_and_digit_bits(bsg, orc):
    for n in (0, 1, 3, 10, 1003, 2 ** 33 + 7):
        for p in (1, 2, 3, 7, 8, 16):
            part = bsg.radix.Partition(n, p)
            offs, sizes = orc.partition(n, p)
            assert [part.offset_of(w) for w in range(p)] == offs
            assert [part.size_of(w) for w in range(p)] == sizes
            for pos in {0, n // 2, max(0, n - 1)}:
                if n:
                    assert part.owner_of(pos) == int(orc.h.orc_part_owner_of(n, p, pos))
    assert [bsg.radix.checked_digit_bits(r) for r in (2, 4, 16, 256, 65536)] == [1, 2, 4, 8, 16]
    for bad in (100, 8, 1 << 32, 0):
        with pytest.raises(ValueError):
            bsg.radix.checked_digit_bits(bad)


def test_schedules_match_oracle(bsg, orc):
    for p in (1, 2, 4, 8, 16, 32):
        partner, keep = orc.schedule(0, p)
        st = bsg.netsort.bitonic_schedule(p).stages
        assert [[a.partner for a in s] for s in st] == partner.tolist()
        assert [[int(a.keep_low) for a in s] for s in st] == keep.tolist()
    for p in (1, 2, 3, 5, 12):
        partner, keep = orc.schedule(1, p)
        st = bsg.netsort.odd_even_rounds(p)
        assert [[a.partner for a in s] for s in st] == partner.tolist()
    for bad in (3, 12, 0):
        with pytest.raises(ValueError):
            bsg.netsort.bitonic_schedule(bad)


def test_sort_instance_validation(bsg):
    # core_test.cpp:67-96
    A = bsg.Algorithm
    ok = bsg.SortInstance(np.array([3, 2, 1], np.uint32), 4, A.OET)
    ok.validate()
    for kw in ({"processors": 0}, {"algorithm": A.SR4, "processors": 2}, {"algorithm": A.BTN, "processors": 3},
               {"radix": 100}, {"algorithm": A.PR2, "radix": 256}):
        bad = bsg.SortInstance(ok.input, **{**{"processors": 4, "algorithm": A.OET}, **kw})
        with pytest.raises(ValueError):
            bad.validate()
    for a in A:
        assert bsg.algorithm_from_name(bsg.algorithm_name(a)) == a
    assert bsg.algorithm_from_name("quicksort") is None
    assert bsg.algorithm_from_name("BTN") == A.BTN


def test_compute_without_gpu_fails_loudly(bsg):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(bsg.DeviceError):
        bsg.radix.serial_radix_sort(np.array([3, 1, 2], np.uint32), 256)


def test_verify_sorted_permutation(bsg):
    # core_test.cpp:49-56
    v = bsg.verify_sorted_permutation
    u = lambda x: np.array(x, np.uint32)
    assert v(u([3, 1, 2]), u([1, 2, 3]))
    assert not v(u([3, 1, 2]), u([1, 2, 4]))
    assert v(u([]), u([]))
    assert not v(u([1, 2]), u([2, 1]))
    assert not v(u([1, 1, 2]), u([1, 2, 2]))
    assert not v(u([1]), u([]))


@pytest.mark.parametrize("seed", [1, 5489, 0, 2**64 - 1])
def test_generate_uniform_random_access(seed):
    """bsg_generate_uniform_at_u32 (jump-ahead by x^offset mod the MT19937-64
    characteristic polynomial) equals slices of generate_uniform_keys
    (core.hpp:93-99), across the first-twist boundaries and deep offsets."""
    import numpy as np
    from paper_1708_09495_b200 import _lib

    L = _lib.lib()
    n = 300000
    full = np.empty(n, np.uint32)
    assert L.bsg_generate_uniform_u32(full.ctypes.data, n, seed) == 0
    for off in (0, 1, 155, 156, 311, 312, 313, 623, 624, 625, 4096, 99991, 299000):
        m = min(1000, n - off)
        part = np.empty(m, np.uint32)
        assert L.bsg_generate_uniform_at_u32(part.ctypes.data, m, seed, off) == 0
        np.testing.assert_array_equal(part, full[off:off + m])
