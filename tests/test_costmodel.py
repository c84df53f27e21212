"""Cost-model restatement vs the reference's costmodel_test.cpp KATs
(used for the predicted_speedup column of the CSV contract)."""
from fractions import Fraction as F

import pytest

from paper_1708_09495_b200 import costmodel as cm


def cores(p):
    return cm.MachineParams.with_cores(p)


def test_serial_closed_forms():
    # costmodel_test.cpp:17-35
    for n in (1, 1000, 1 << 20):
        assert cm.t_serial(n, cores(1), 256) == 68 * n
        assert cm.t_serial(n, cores(1), 65536) == 34 * n
    assert cm.t_serial(0, cores(1), 256) == 0
    mp = cores(1).set_gap_ratio(7)
    assert cm.t_serial(10, mp, 256) == 4 * (3 * 10 * 7 + 2 * 10)
    assert cm.t_serial(10, mp, 2) == 32 * (3 * 10 * 7 + 2 * 10)


def test_parallel_radix_closed_forms():
    # costmodel_test.cpp:37-53 / costmodel.hpp:13-15
    for p in (1, 2, 4, 8, 16):
        for n in (1 << 10, 1 << 20, 12345):
            assert cm.t_parallel_radix(n, cores(p), 256) == F(88 * n, p) + 40 * 256 * p
            assert cm.t_parallel_radix(n, cores(p), 65536) == F(44 * n, p) + 20 * 65536 * p
    for n in (10, 1000):
        assert cm.t_parallel_radix(n, cores(1), 256) > cm.t_serial(n, cores(1), 256)


def test_network_closed_forms():
    # costmodel_test.cpp:55-89
    for n in (1000, 4096):
        assert cm.t_oet(n, cores(1)) == 88 * n
        assert cm.t_oet(n, cores(4)) == 37 * n
        assert cm.t_btn(n, cores(1)) == 68 * n
        assert cm.t_btn(n, cores(4)) == 32 * n
        assert cm.t_btn(n, cores(16)) == F(67, 4) * n
        for p in (2, 4, 8, 16):
            assert cm.t_oet(n, cores(p)) >= cm.t_btn(n, cores(p))
            lg = p.bit_length() - 1
            assert cm.t_btn(n, cores(p)) == F(68 * n, p) + F(10 * n * lg * (lg + 1), p)
            assert cm.t_oet(n, cores(p)) == F(68 * n, p) + 20 * n
    with pytest.raises(ValueError):
        cm.t_btn(100, cores(6))


def test_predicted_speedups():
    # costmodel_test.cpp:91-134
    assert cm.asymptotic_speedup("pr4", cores(4)) == F(34, 11)
    assert cm.asymptotic_speedup("pr4", cores(8)) == F(68, 11)
    assert cm.asymptotic_speedup("pr4", cores(16)) == F(136, 11)
    assert cm.predicted_speedup("btn", 1000, cores(2)) == F(17, 11)
    assert cm.predicted_speedup("btn", 1000, cores(4)) == F(17, 8)
    assert cm.predicted_speedup("btn", 1000, cores(8)) == F(136, 47)
    assert cm.predicted_speedup("btn", 1000, cores(16)) == F(272, 67)
    prev = F(0)
    bound = cm.asymptotic_speedup("pr4", cores(8))
    for n in (1 << 10, 1 << 14, 1 << 18, 1 << 22, 1 << 26):
        s = cm.predicted_speedup("pr4", n, cores(8))
        assert prev < s < bound
        prev = s
    assert cm.predicted_speedup("sr4", 12345, cores(1)) == 1
    with pytest.raises(ValueError):
        cm.predicted_speedup("pr4", 0, cores(4))


def test_oet_btn_ratio():
    # costmodel_test.cpp:136-143
    assert cm.predicted_ratio_oet_btn(16, True) == F(388, 228)
    assert cm.predicted_ratio_oet_btn(4, True) == F(148, 108)
    assert cm.predicted_ratio_oet_btn(16, False) == F(388, 268)
    with pytest.raises(ValueError):
        cm.predicted_ratio_oet_btn(6, True)


def test_validation():
    # costmodel_test.cpp:157-165
    with pytest.raises(ValueError):
        cm.t_serial(10, cores(1).set_gap_ratio(-1), 256)
    with pytest.raises(ValueError):
        cm.t_oet(10, cores(0))


def test_csv_contract_formatting():
    # bench.hpp:213-252: header, shortest decimals, integral values with ".0"
    assert cm.CSV_HEADER == "algorithm,n,p,mean_seconds,speedup,predicted_speedup,verified"
    assert cm.format_number(2.0) == "2.0"
    assert cm.format_number(0.25) == "0.25"
    assert cm.format_number(1e-05) == "1e-05"
    assert cm.csv_row("pr4", 1024, 4, 0.5, 2.0, 1.5, True) == "pr4,1024,4,0.5,2.0,1.5,true"
    assert cm.predicted_for("pr4", 0, 4) == 1.0
