"""ctypes wrappers for the CPU checkers.  TEST INFRASTRUCTURE ONLY: imported by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs, never by the product package.

- ``Oracle``: oracle/liborc.so, the plain-C restatement (bsg_oracle.c).
- ``Reference``: oracle/_ref/libbspref.so, the reference's own headers compiled
  unmodified (ref_shim.cpp); None when it was not built.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "liborc.so")
REF_PATH = os.path.join(HERE, "_ref", "libbspref.so")


class Stats(ctypes.Structure):
    _fields_ = [("supersteps", ctypes.c_int32), ("messages_sent", ctypes.c_uint64),
                ("messages_delivered", ctypes.c_uint64), ("words_sent", ctypes.c_uint64),
                ("words_delivered", ctypes.c_uint64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


class Oracle:
    """The C restatement (oracle/bsg_oracle.c)."""

    def __init__(self, path: str = ORC_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.h = ctypes.CDLL(path)
        h = self.h
        vp, u64, i = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
        h.orc_generate_uniform_keys.argtypes = [vp, u64, u64]
        h.orc_mt64_draws.argtypes = [vp, u64, u64]
        h.orc_splitmix64.argtypes = [u64]
        h.orc_splitmix64.restype = u64
        h.orc_derive_seed.argtypes = [u64, i]
        h.orc_derive_seed.restype = u64
        h.orc_checked_digit_bits.argtypes = [u64]
        h.orc_count_sort_round.argtypes = [vp, u64, i, u64, vp]
        h.orc_serial_radix_sort.argtypes = [vp, u64, u64, vp]
        h.orc_parallel_radix.argtypes = [vp, u64, i, u64, i, vp, ctypes.POINTER(Stats)]
        h.orc_merge_split.argtypes = [vp, u64, vp, u64, vp, vp]
        h.orc_bitonic_schedule.argtypes = [i, vp, vp, i]
        h.orc_odd_even_rounds.argtypes = [i, vp, vp, i]
        h.orc_block_network.argtypes = [i, vp, u64, i, i, vp, ctypes.POINTER(Stats)]
        h.orc_part_size_of.argtypes = [u64, i, i]
        h.orc_part_size_of.restype = u64
        h.orc_part_offset_of.argtypes = [u64, i, i]
        h.orc_part_offset_of.restype = u64
        h.orc_part_owner_of.argtypes = [u64, i, u64]

    def generate_uniform_keys(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint32)
        self.h.orc_generate_uniform_keys(_p(out), n, seed)
        return out

    def mt64_draws(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        self.h.orc_mt64_draws(_p(out), n, seed)
        return out

    def derive_seed(self, seed: int, rep: int) -> int:
        return int(self.h.orc_derive_seed(seed, rep))

    def checked_digit_bits(self, radix: int) -> int:
        return int(self.h.orc_checked_digit_bits(radix))

    def count_sort_round(self, keys, round: int, radix: int) -> np.ndarray:
        k = _u32(keys)
        out = np.empty_like(k)
        rc = self.h.orc_count_sort_round(_p(k), k.size, round, radix, _p(out))
        if rc:
            raise ValueError(f"oracle count_sort_round rc={rc}")
        return out

    def serial_radix_sort(self, keys, radix: int) -> np.ndarray:
        k = _u32(keys)
        out = np.empty_like(k)
        rc = self.h.orc_serial_radix_sort(_p(k), k.size, radix, _p(out))
        if rc:
            raise ValueError(f"oracle serial_radix_sort rc={rc}")
        return out

    def parallel_radix(self, keys, p: int, radix: int, rounds_limit: int = -1) -> Tuple[np.ndarray, dict]:
        k = _u32(keys)
        out = np.empty_like(k)
        st = Stats()
        rc = self.h.orc_parallel_radix(_p(k), k.size, p, radix, rounds_limit, _p(out), ctypes.byref(st))
        if rc:
            raise ValueError(f"oracle parallel_radix rc={rc}")
        return out, st.as_dict()

    def merge_split(self, a, b) -> Tuple[np.ndarray, np.ndarray]:
        a, b = _u32(a), _u32(b)
        lo, hi = np.empty_like(a), np.empty_like(b)
        self.h.orc_merge_split(_p(a), a.size, _p(b), b.size, _p(lo), _p(hi))
        return lo, hi

    def schedule(self, network: int, p: int):
        cap = 4096
        partner = np.empty(cap * max(p, 1), dtype=np.int32)
        keep = np.empty(cap * max(p, 1), dtype=np.int32)
        fn = self.h.orc_bitonic_schedule if network == 0 else self.h.orc_odd_even_rounds
        S = fn(p, _p(partner), _p(keep), cap)
        if S < 0:
            raise ValueError("bad p")
        return partner[:S * p].reshape(S, p), keep[:S * p].reshape(S, p)

    def block_network(self, network: int, keys, p: int, stages_limit: int = -1) -> Tuple[np.ndarray, dict]:
        k = _u32(keys)
        L = (k.size + p - 1) // p
        out = np.empty(max(L * p, k.size), dtype=np.uint32)
        st = Stats()
        rc = self.h.orc_block_network(network, _p(k), k.size, p, stages_limit, _p(out), ctypes.byref(st))
        if rc:
            raise ValueError(f"oracle block_network rc={rc}")
        S = self.schedule(network, p)[0].shape[0]
        full = stages_limit < 0 or stages_limit >= S
        return (out[:k.size] if full else out[:L * p]), st.as_dict()

    def time_serial_radix_sort(self, keys, radix: int):
        import time

        k = _u32(keys)
        out = np.empty_like(k)
        t0 = time.perf_counter()
        rc = self.h.orc_serial_radix_sort(_p(k), k.size, radix, _p(out))
        t = time.perf_counter() - t0
        if rc:
            raise RuntimeError("oracle serial_radix_sort failed")
        return t, out

    def partition(self, n: int, p: int):
        return ([int(self.h.orc_part_offset_of(n, p, w)) for w in range(p)],
                [int(self.h.orc_part_size_of(n, p, w)) for w in range(p)])


class Reference:
    """The reference's own headers (oracle/_ref/libbspref.so)."""

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        self.h = ctypes.CDLL(path)
        h = self.h
        vp, u64, i = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
        h.ref_generate_uniform_keys.argtypes = [vp, u64, u64]
        h.ref_count_sort_round.argtypes = [vp, u64, i, u64, vp]
        h.ref_serial_radix_sort.argtypes = [vp, u64, u64, vp]
        h.ref_parallel_radix.argtypes = [vp, u64, i, u64, i, i, vp, ctypes.POINTER(Stats)]
        h.ref_block_network.argtypes = [i, vp, u64, i, i, i, vp, ctypes.POINTER(u64), ctypes.POINTER(Stats)]
        h.ref_merge_split.argtypes = [vp, u64, vp, u64, vp, vp]
        h.ref_schedule.argtypes = [i, i, vp, vp, i, ctypes.POINTER(i)]
        h.ref_sort_instance.argtypes = [vp, u64, i, i, u64, vp]
        h.ref_time_serial_radix_sort.argtypes = [vp, u64, u64, vp]
        h.ref_time_serial_radix_sort.restype = ctypes.c_double
        h.ref_time_parallel_radix.argtypes = [vp, u64, i, u64, vp]
        h.ref_time_parallel_radix.restype = ctypes.c_double
        h.ref_time_block_network.argtypes = [i, vp, u64, u64, i, vp]
        h.ref_time_block_network.restype = ctypes.c_double
        h.ref_time_network_once.argtypes = [i, vp, u64, i, vp]
        h.ref_time_network_once.restype = ctypes.c_double

    def generate_uniform_keys(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint32)
        self.h.ref_generate_uniform_keys(_p(out), n, seed)
        return out

    def count_sort_round(self, keys, round: int, radix: int) -> np.ndarray:
        k = _u32(keys)
        out = np.empty_like(k)
        rc = self.h.ref_count_sort_round(_p(k), k.size, round, radix, _p(out))
        if rc:
            raise ValueError(f"reference count_sort_round rc={rc}")
        return out

    def serial_radix_sort(self, keys, radix: int) -> np.ndarray:
        k = _u32(keys)
        out = np.empty_like(k)
        rc = self.h.ref_serial_radix_sort(_p(k), k.size, radix, _p(out))
        if rc:
            raise ValueError(f"reference serial_radix_sort rc={rc}")
        return out

    def parallel_radix(self, keys, p: int, radix: int, rounds_limit: int = -1, sequential: bool = True):
        k = _u32(keys)
        out = np.empty_like(k)
        st = Stats()
        rc = self.h.ref_parallel_radix(_p(k), k.size, p, radix, rounds_limit, int(sequential), _p(out),
                                       ctypes.byref(st))
        if rc:
            raise ValueError(f"reference parallel_radix rc={rc}")
        return out, st.as_dict()

    def block_network(self, network: int, keys, p: int, stages_limit: int = -1, sequential: bool = True):
        k = _u32(keys)
        L = (k.size + p - 1) // p
        out = np.empty(max(L * p, k.size, 1), dtype=np.uint32)
        n_out = ctypes.c_uint64(0)
        st = Stats()
        rc = self.h.ref_block_network(network, _p(k), k.size, p, stages_limit, int(sequential), _p(out),
                                      ctypes.byref(n_out), ctypes.byref(st))
        if rc:
            raise ValueError(f"reference block_network rc={rc}")
        return out[:n_out.value], st.as_dict()

    def merge_split(self, a, b):
        a, b = _u32(a), _u32(b)
        lo, hi = np.empty_like(a), np.empty_like(b)
        self.h.ref_merge_split(_p(a), a.size, _p(b), b.size, _p(lo), _p(hi))
        return lo, hi

    def schedule(self, network: int, p: int):
        cap = 4096
        partner = np.empty(cap * max(p, 1), dtype=np.int32)
        keep = np.empty(cap * max(p, 1), dtype=np.int32)
        S = ctypes.c_int(0)
        rc = self.h.ref_schedule(network, p, _p(partner), _p(keep), cap, ctypes.byref(S))
        if rc:
            raise ValueError("bad p")
        return partner[:S.value * p].reshape(S.value, p), keep[:S.value * p].reshape(S.value, p)

    def time_serial_radix_sort(self, keys, radix: int):
        """bench.hpp run_once timing of serial_radix_sort: (seconds, output)."""
        k = _u32(keys)
        out = np.empty_like(k)
        t = self.h.ref_time_serial_radix_sort(_p(k), k.size, radix, _p(out))
        if t < 0:
            raise RuntimeError("reference serial_radix_sort failed")
        return t, out

    def time_parallel_radix(self, keys, p: int, radix: int):
        """bench.hpp run_once timing of run_parallel_radix (threaded executor)."""
        k = _u32(keys)
        out = np.empty_like(k)
        t = self.h.ref_time_parallel_radix(_p(k), k.size, p, radix, _p(out))
        if t < 0:
            raise RuntimeError("reference parallel radix failed")
        return t, out

    def time_block_network(self, network: int, arrays, p: int):
        a = _u32(arrays)
        out = np.empty_like(a)
        t = self.h.ref_time_block_network(network, _p(a), a.shape[0], a.shape[1], p, _p(out))
        if t < 0:
            raise RuntimeError("reference block network failed")
        return t, out

    def time_network_once(self, network: int, keys, p: int):
        """bench.hpp run_once timing of run_block_network (default executor)."""
        k = _u32(keys)
        out = np.empty_like(k)
        t = self.h.ref_time_network_once(network, _p(k), k.size, p, _p(out))
        if t < 0:
            raise RuntimeError("reference block network failed")
        return t, out

    def sort_instance(self, keys, processors: int, algorithm: int, radix: int) -> np.ndarray:
        k = _u32(keys)
        out = np.empty_like(k)
        rc = self.h.ref_sort_instance(_p(k), k.size, processors, algorithm, radix, _p(out))
        if rc == 1:
            raise ValueError("invalid_argument")
        if rc:
            raise RuntimeError(f"reference sort_instance rc={rc}")
        return out


def maybe_reference() -> Optional[Reference]:
    try:
        return Reference()
    except (FileNotFoundError, OSError):
        return None
