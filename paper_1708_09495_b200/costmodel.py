"""Exact restatement of the reference's analytical cost model
(proj/include/bspsort/costmodel.hpp), used to fill the `predicted_speedup`
column of the reference CSV contract (bench.hpp:221-252) for GPU rows.

Costs are exact rationals in units of the fast-memory gap G
(``fractions.Fraction`` stands in for boost::multiprecision::cpp_rational).
With the default g = 5G and radix 256 the closed forms are
(costmodel.hpp:10-18):

    serial          68*N
    parallel radix  (32/lg r)*(4(n/p)(g/G) + 2(n/p) + 2pr(g/G))
    odd-even        68*n/p + 20*n
    bitonic         68*n/p + 10*n*lg(p)(lg(p)+1)/p
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

KEY_BITS = 32
ALGORITHMS = ("sr4", "pr4", "pr2", "btn", "oet")


def _is_pow2(x: int) -> bool:
    return x > 0 and (x & (x - 1)) == 0


@dataclass
class MachineParams:
    """costmodel.hpp:37-67: the septuplet (p, l, g, m, L, G, M); only p, g
    and G enter the formulas."""
    cores: int = 1
    sync_latency: Fraction = Fraction(0)
    slow_gap: Fraction = Fraction(5)
    memory_units: int = 0
    memory_latency: Fraction = Fraction(0)
    fast_gap: Fraction = Fraction(1)
    fast_capacity: int = -1

    @staticmethod
    def with_cores(p: int) -> "MachineParams":
        return MachineParams(cores=p)

    def set_gap_ratio(self, g_over_G) -> "MachineParams":
        self.slow_gap = Fraction(g_over_G)
        self.fast_gap = Fraction(1)
        return self

    def validate(self) -> None:
        if self.cores < 1:
            raise ValueError("MachineParams: p must be >= 1")
        if self.fast_gap <= 0:
            raise ValueError("MachineParams: G must be positive")
        if self.slow_gap < 0 or self.sync_latency < 0 or self.memory_latency < 0:
            raise ValueError("MachineParams: costs must be non-negative")

    def gap_ratio(self) -> Fraction:
        return Fraction(self.slow_gap) / Fraction(self.fast_gap)


def rounds_for(radix: int) -> int:
    """costmodel.hpp:72-79."""
    if not _is_pow2(radix):
        raise ValueError("cost model: radix must be a power of two")
    bits = radix.bit_length() - 1
    if bits == 0 or KEY_BITS % bits != 0:
        raise ValueError("cost model: lg(radix) must divide 32")
    return KEY_BITS // bits


def _serial_cost(keys_per_core: Fraction, mp: MachineParams, radix: int) -> Fraction:
    """costmodel.hpp:84-89: per round 3N g + 2N G."""
    return rounds_for(radix) * (3 * keys_per_core * mp.gap_ratio() + 2 * keys_per_core)


def stage_count_btn(p: int) -> int:
    """costmodel.hpp:91-97."""
    if p < 1 or not _is_pow2(p):
        raise ValueError("cost model: bitonic requires a power-of-two p")
    lg = p.bit_length() - 1
    return lg * (lg + 1) // 2


def t_serial(keys: int, mp: MachineParams, radix: int = 256) -> Fraction:
    """costmodel.hpp:101-104."""
    mp.validate()
    return _serial_cost(Fraction(keys), mp, radix)


def t_parallel_radix(n: int, mp: MachineParams, radix: int = 256) -> Fraction:
    """costmodel.hpp:109-116."""
    mp.validate()
    gr = mp.gap_ratio()
    per_core = Fraction(n, mp.cores)
    return rounds_for(radix) * (4 * per_core * gr + 2 * per_core + 2 * mp.cores * radix * gr)


def t_oet(n: int, mp: MachineParams) -> Fraction:
    """costmodel.hpp:120-124."""
    mp.validate()
    per_core = Fraction(n, mp.cores)
    return _serial_cost(per_core, mp, 256) + mp.cores * 4 * per_core * mp.gap_ratio()


def t_btn(n: int, mp: MachineParams) -> Fraction:
    """costmodel.hpp:128-133."""
    mp.validate()
    stages = stage_count_btn(mp.cores)
    per_core = Fraction(n, mp.cores)
    return _serial_cost(per_core, mp, 256) + stages * 4 * per_core * mp.gap_ratio()


def t_algorithm(algo: str, n: int, mp: MachineParams) -> Fraction:
    """costmodel.hpp:135-145."""
    if algo == "sr4":
        return t_serial(n, mp, 256)
    if algo == "pr4":
        return t_parallel_radix(n, mp, 256)
    if algo == "pr2":
        return t_parallel_radix(n, mp, 65536)
    if algo == "btn":
        return t_btn(n, mp)
    if algo == "oet":
        return t_oet(n, mp)
    raise ValueError("t_algorithm: unknown algorithm")


def predicted_speedup(algo: str, n: int, mp: MachineParams) -> Fraction:
    """costmodel.hpp:147-152: over the serial radix-256 baseline at the same n."""
    if n == 0:
        raise ValueError("predicted_speedup: undefined for n = 0")
    if algo == "sr4":
        return Fraction(1)
    return t_serial(n, mp, 256) / t_algorithm(algo, n, mp)


def asymptotic_speedup(algo: str, mp: MachineParams) -> Fraction:
    """costmodel.hpp:158-176: the n -> infinity limit."""
    mp.validate()
    gr = mp.gap_ratio()
    serial_per_key = rounds_for(256) * (3 * gr + 2)
    if algo == "sr4":
        return Fraction(1)
    if algo in ("pr4", "pr2"):
        radix = 256 if algo == "pr4" else 65536
        return serial_per_key * mp.cores / (rounds_for(radix) * (4 * gr + 2))
    if algo in ("btn", "oet"):
        return predicted_speedup(algo, 1, mp)
    raise ValueError("asymptotic_speedup: unknown algorithm")


def predicted_ratio_oet_btn(p: int, printed_form: bool) -> Fraction:
    """costmodel.hpp:183-191."""
    if p < 1 or not _is_pow2(p):
        raise ValueError("predicted_ratio_oet_btn: p must be a power of two")
    lg = p.bit_length() - 1
    num = 68 + 20 * Fraction(p)
    den = 68 + 10 * Fraction(lg) * lg if printed_form else 68 + 10 * Fraction(lg) * (lg + 1)
    return num / den


def predicted_for(algo: str, n: int, p: int, g_over_G=5) -> float:
    """bench.hpp:104-110 (`detail::predicted_for`): 1.0 for n = 0."""
    if n == 0:
        return 1.0
    mp = MachineParams.with_cores(p).set_gap_ratio(g_over_G)
    return float(predicted_speedup(algo, n, mp))


def format_number(v: float) -> str:
    """bench.hpp:213-219: shortest round-trip decimal (std::to_chars), with
    a trailing '.0' on integral values.  Python's repr of a float is the
    same shortest round-trip form ('2.0', '1e-05', '1.5e+20')."""
    s = repr(float(v))
    if not any(c in s for c in ".en"):
        s += ".0"
    return s


CSV_HEADER = "algorithm,n,p,mean_seconds,speedup,predicted_speedup,verified"


def csv_row(algo: str, n: int, p: int, mean_seconds: float, speedup: float, predicted: float,
            verified: bool) -> str:
    """One line of bench.hpp:223-252 `emit_csv`."""
    return ",".join([algo, str(n), str(p), format_number(mean_seconds), format_number(speedup),
                     format_number(predicted), "true" if verified else "false"])
