"""Stable LSD radix sorting of uint32 keys -- Python mirror of
``bspsort::radix`` (radix.hpp) running on the B200 through libbsg.so.

Inputs are numpy uint32 arrays (host; staged through the GPU) or torch CUDA
uint32 tensors (device-resident; asynchronous on the current stream).  The
result has the input's kind.  Argument errors raise ValueError exactly where
the reference throws std::invalid_argument.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from ._keys import KeyBuf
from .core import Algorithm, SortInstance, key_bits


def digit_of(key: int, round: int, bits: int) -> int:
    """radix.hpp:28-30: digit of `key` in `round`, low digits first."""
    return (int(key) >> (round * bits)) & ((1 << bits) - 1)


def checked_digit_bits(radix: int) -> int:
    """radix.hpp:32-40: lg r for r in {2,4,16,256,65536}, else ValueError."""
    b = _lib.lib().bsg_checked_digit_bits(int(radix) & (2**64 - 1))
    if b < 0:
        raise ValueError(_lib.last_error())
    return b


def count_sort_round(keys, round: int, radix: int):
    """radix.hpp:44-65: one stable bucket pass over digit `round`."""
    bits = checked_digit_bits(radix)
    if round < 0 or round >= key_bits // bits:
        raise ValueError(f"round {round} outside [0, {key_bits // bits})")
    kb = KeyBuf(keys)
    out = kb.empty(kb.n)
    ctx = kb.ctx()
    _lib.check(_lib.lib().bsg_count_sort_round_u32(ctx.handle, kb.ptr, KeyBuf(out).ptr, kb.n, round, bits, kb.mem,
                                                   kb.stream), "count_sort_round")
    return out


def serial_radix_sort(keys, radix: int):
    """radix.hpp:69-90: 32/lg r stable rounds, low digit first (SR4 = r 256)."""
    bits = checked_digit_bits(radix)
    kb = KeyBuf(keys)
    out = kb.empty(kb.n)
    ctx = kb.ctx()
    _lib.check(_lib.lib().bsg_radix_sort_u32(ctx.handle, kb.ptr, KeyBuf(out).ptr, kb.n, bits, kb.mem, kb.stream),
               "serial_radix_sort")
    return out


@dataclass
class Partition:
    """radix.hpp:96-118 detail::Partition: balanced contiguous cut."""

    n: int = 0
    p: int = 1

    def small(self) -> int:
        return self.n // self.p

    def big_count(self) -> int:
        return self.n % self.p

    def size_of(self, w: int) -> int:
        return int(_lib.lib().bsg_partition_size_of(self.n, self.p, w))

    def offset_of(self, w: int) -> int:
        return int(_lib.lib().bsg_partition_offset_of(self.n, self.p, w))

    def owner_of(self, pos: int) -> int:
        return int(_lib.lib().bsg_partition_owner_of(self.n, self.p, pos))


@dataclass
class RadixPlan:
    """radix.hpp:120-125 detail::RadixPlan."""

    part: Partition = field(default_factory=Partition)
    radix: int = 256
    bits: int = 8
    rounds: int = 4


@dataclass
class PreparedRadix:
    """radix.hpp:228-231.  `keys` holds the input; `blocks` are the per-worker
    views of the balanced partition.  Setting ``plan.rounds = k`` before
    :func:`run_parallel_radix` stops after k rounds, as in the reference."""

    plan: RadixPlan
    keys: object

    @property
    def blocks(self) -> List[object]:
        return [self.keys[self.plan.part.offset_of(w):self.plan.part.offset_of(w) + self.plan.part.size_of(w)]
                for w in range(self.plan.part.p)]


@dataclass
class ParallelSortResult:
    """radix.hpp:251-254 (RunStats as a dict with the bsp.hpp:86-92 fields)."""

    output: object
    stats: dict


def prepare_parallel_radix(keys, p: int, radix: int) -> PreparedRadix:
    """radix.hpp:233-249."""
    if p < 1:
        raise ValueError("parallel radix sort: p must be >= 1")
    bits = checked_digit_bits(radix)
    kb = KeyBuf(keys)
    plan = RadixPlan(Partition(kb.n, p), radix, bits, key_bits // bits)
    return PreparedRadix(plan, kb.obj)


def run_parallel_radix(prep: PreparedRadix, use_sequential_executor: bool = False,
                       group: Optional["_lib.GroupContext"] = None) -> ParallelSortResult:
    """radix.hpp:260-303: PR with p logical workers on the GPU -- or, with a
    ``group`` (:class:`_lib.GroupContext`), spread over the group's GPUs in
    this process (numpy input, or a CUDA tensor on the group's first device).
    The executor flag is accepted for signature parity; results are identical
    either way."""
    del use_sequential_executor
    plan = prep.plan
    full_rounds = key_bits // plan.bits
    rounds_limit = -1 if plan.rounds >= full_rounds else max(0, plan.rounds)
    kb = KeyBuf(prep.keys)
    out = kb.empty(kb.n)
    stats = _lib.RunStats()
    ctx = group if group is not None else kb.ctx()
    _lib.check(_lib.lib().bsg_parallel_radix_sort_u32(ctx.handle, kb.ptr, KeyBuf(out).ptr, kb.n, plan.part.p,
                                                      plan.bits, rounds_limit, ctypes.byref(stats), kb.mem, kb.stream),
               "run_parallel_radix")
    return ParallelSortResult(out, stats.as_dict())


def parallel_radix_sort(instance: SortInstance):
    """radix.hpp:306-312: PR4 / PR2 entry point."""
    instance.validate()
    if instance.algorithm not in (Algorithm.PR4, Algorithm.PR2):
        raise ValueError("parallel_radix_sort handles pr4 and pr2 only")
    prep = prepare_parallel_radix(instance.input, instance.processors, instance.radix)
    return run_parallel_radix(prep).output


def digit_counts(block, round: int, radix: int):
    """radix.hpp:127-132 count_digits on a device block -> uint64 counts (torch)."""
    import torch

    bits = checked_digit_bits(radix)
    kb = KeyBuf(block)
    if kb.mem != _lib.MEM_DEVICE:
        raise ValueError("digit_counts expects a CUDA tensor")
    counts = torch.empty(1 << bits, dtype=torch.int64, device=kb.obj.device)
    _lib.check(_lib.lib().bsg_pr_count_digits(kb.ctx().handle, kb.ptr, kb.n, round, bits, counts.data_ptr(),
                                              kb.stream), "count_digits")
    return counts


def group_sort_blocks(group, blocks, n: int, p: int, radix: int, rounds=None, variant: int = 0,
                      timing: bool = False):
    """bsg_pr_group_sort_u32: the parallel radix sort over a group context
    whose member g holds its key range in ``blocks[g]`` (a CUDA tensor on the
    member's device, sorted in place).  Returns (RunStats dict, timing dict or
    None).  variant: _lib.PR_PEER (fused NVLink rounds) or _lib.PR_NCCL."""
    bits = checked_digit_bits(radix)
    full_rounds = key_bits // bits
    rounds_limit = -1 if rounds is None or rounds >= full_rounds else max(0, int(rounds))
    import torch

    ptrs = (ctypes.c_void_p * len(blocks))(*[b.data_ptr() for b in blocks])
    # each member waits for the torch stream that produced its block
    streams = (ctypes.c_void_p * len(blocks))(*[torch.cuda.current_stream(b.device).cuda_stream for b in blocks])
    stats = _lib.RunStats()
    tm = _lib.PrTiming()
    _lib.check(_lib.lib().bsg_pr_group_sort_u32(group.handle, ptrs, int(n), int(p), bits, rounds_limit, int(variant),
                                                ctypes.byref(stats), ctypes.byref(tm) if timing else None, streams),
               "group sort")
    return stats.as_dict(), (tm.as_dict() if timing else None)


def group_range(n: int, p: int, G: int, g: int):
    """(offset, size) of member g's key range in a G-member group."""
    L = _lib.lib()
    return int(L.bsg_group_range_offset(n, p, G, g)), int(L.bsg_group_range_size(n, p, G, g))
