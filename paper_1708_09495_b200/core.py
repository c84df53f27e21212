"""Key types, validation, deterministic inputs, verification.

Python mirror of ``bspsort`` core (core.hpp) plus ``bench::derive_seed``
(bench.hpp:77-88).  Generators run on the host inside libbsg.so (the
reference generator is host-side by definition: the CPU oracle and the GPU
must consume the same bytes).
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib

Key = np.uint32
key_bits = 32  # core.hpp:22


class Algorithm(enum.IntEnum):
    """core.hpp:24 ``enum class Algorithm { SR4, PR4, PR2, BTN, OET }``."""

    SR4 = 0
    PR4 = 1
    PR2 = 2
    BTN = 3
    OET = 4


def algorithm_name(a: Algorithm) -> str:
    """core.hpp:26-35."""
    return {Algorithm.SR4: "sr4", Algorithm.PR4: "pr4", Algorithm.PR2: "pr2", Algorithm.BTN: "btn",
            Algorithm.OET: "oet"}.get(a, "?")


def algorithm_from_name(name: str) -> Optional[Algorithm]:
    """core.hpp:37-47 (case-insensitive)."""
    return {"sr4": Algorithm.SR4, "pr4": Algorithm.PR4, "pr2": Algorithm.PR2, "btn": Algorithm.BTN,
            "oet": Algorithm.OET}.get(name.lower())


def is_power_of_two(x: int) -> bool:
    """core.hpp:49-51."""
    return x > 0 and (x & (x - 1)) == 0


def log2_exact(x: int) -> int:
    """core.hpp:54-56 (bit_width - 1)."""
    return int(x).bit_length() - 1


def digit_bits(radix: int) -> int:
    """core.hpp:60-64: bits per digit, or -1 if the radix does not split 32-bit keys."""
    if not is_power_of_two(radix):
        return -1
    b = log2_exact(radix)
    return b if (b > 0 and key_bits % b == 0) else -1


@dataclass
class SortInstance:
    """core.hpp:67-89."""

    input: object = field(default_factory=lambda: np.empty(0, dtype=np.uint32))
    processors: int = 1
    algorithm: Algorithm = Algorithm.SR4
    radix: int = 256
    seed: int = 0

    def validate(self) -> None:
        """core.hpp:74-88; raises ValueError (std::invalid_argument)."""
        if self.processors < 1:
            raise ValueError("SortInstance: processors must be >= 1")
        if digit_bits(self.radix) < 0:
            raise ValueError("SortInstance: radix must be a power of two whose bit width divides 32")
        if self.algorithm == Algorithm.SR4 and self.processors != 1:
            raise ValueError("SortInstance: sr4 is serial, requires p = 1")
        if self.algorithm == Algorithm.BTN and not is_power_of_two(self.processors):
            raise ValueError("SortInstance: btn requires a power-of-two p")
        if self.algorithm == Algorithm.PR4 and self.radix != 256:
            raise ValueError("SortInstance: pr4 is radix-256 by definition")
        if self.algorithm == Algorithm.PR2 and self.radix != 65536:
            raise ValueError("SortInstance: pr2 is radix-65536 by definition")


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data_as(ctypes.c_void_p).value or 0


def generate_uniform_keys(n: int, seed: int) -> np.ndarray:
    """core.hpp:93-99: n keys, mt19937_64(seed), low 32 bits per draw."""
    out = np.empty(int(n), dtype=np.uint32)
    _lib.check(_lib.lib().bsg_generate_uniform_u32(_ptr(out), int(n), int(seed) & (2**64 - 1)), "generate_uniform_keys")
    return out


def generate_uniform_keys_at(n: int, seed: int, offset: int) -> np.ndarray:
    """Draws [offset, offset + n) of generate_uniform_keys(., seed)'s stream
    (jump-ahead; no need to generate the prefix)."""
    out = np.empty(int(n), dtype=np.uint32)
    _lib.check(_lib.lib().bsg_generate_uniform_at_u32(_ptr(out), int(n), int(seed) & (2**64 - 1), int(offset)),
               "generate_uniform_keys_at")
    return out


def generate_uniform_keys_device(n: int, seed: int, device: int = 0, offset: int = 0):
    """generate_uniform_keys on the GPU: a torch.uint32 CUDA tensor holding the
    same n keys, bit for bit (segment starts by jump-ahead); ``offset`` > 0
    gives keys [offset, offset + n) of the stream (a rank's block of a
    block-distributed input)."""
    import torch

    out = torch.empty(int(n), dtype=torch.int32, device=torch.device("cuda", device))
    ctx = _lib.context(device)
    _lib.check(_lib.lib().bsg_generate_uniform_device_at_u32(ctx.handle, out.data_ptr(), int(n),
                                                             int(seed) & (2**64 - 1), int(offset),
                                                             torch.cuda.current_stream(out.device).cuda_stream),
               "generate_uniform_keys_device")
    return out.view(torch.uint32)


SKEW_NARROW16, SKEW_ZIPF, SKEW_ALL_EQUAL = 0, 1, 2


def generate_skewed_keys(n: int, seed: int, kind: int, zipf_s: float = 1.1) -> np.ndarray:
    """Config-3 inputs (builder-defined): 0 = uniform & 0xFFFF,
    1 = Zipf(s) over ranks 1..2^32 (key = rank - 1), 2 = all 0xABCD1234."""
    out = np.empty(int(n), dtype=np.uint32)
    _lib.check(_lib.lib().bsg_generate_skewed_u32(_ptr(out), int(n), int(seed) & (2**64 - 1), int(kind),
                                                  float(zipf_s)), "generate_skewed_keys")
    return out


def derive_seed(seed: int, rep: int) -> int:
    """bench.hpp:86-88 (splitmix64)."""
    return int(_lib.lib().bsg_derive_seed(int(seed) & (2**64 - 1), int(rep)))


def verify_sorted_permutation(input_keys, output_keys) -> bool:
    """core.hpp:103-109: non-decreasing and a permutation of the input."""
    a = _to_host(input_keys)
    b = _to_host(output_keys)
    if a.shape != b.shape:
        return False
    if b.size and not bool(np.all(b[:-1] <= b[1:])):
        return False
    return bool(np.array_equal(np.sort(a, kind="stable"), b))


def _to_host(x) -> np.ndarray:
    try:
        import torch

        if isinstance(x, torch.Tensor):
            t = x.detach()
            if t.dtype != torch.uint32:
                t = t.view(torch.uint32) if t.element_size() == 4 else t.to(torch.int64)
            return t.cpu().numpy().astype(np.uint32, copy=False)
    except ImportError:  # pragma: no cover
        pass
    return np.ascontiguousarray(x, dtype=np.uint32)
