"""Block-level sorting networks (BTN bitonic, OET odd-even transposition) --
Python mirror of ``bspsort::netsort`` (netsort.hpp) on the B200.

The reference sorts one array per call with p threads; here every call is a
batch of independent arrays, one CTA per array, the p workers living as p
shared-memory blocks (see csrc/netsort.cu).  Single-array calls are batches
of one.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _lib
from ._keys import KeyBuf
from .core import Algorithm, SortInstance
from .radix import ParallelSortResult

local_sort_radix = 256  # netsort.hpp:25


def merge_split(a, b) -> Tuple[object, object]:
    """netsort.hpp:30-51: (|a| smallest, |b| largest) of a U b, both sorted."""
    ka, kb_ = KeyBuf(a), KeyBuf(b)
    if ka.mem != kb_.mem:
        raise ValueError("merge_split: a and b must both be host arrays or both CUDA tensors")
    low, high = ka.empty(ka.n), ka.empty(kb_.n)
    _lib.check(_lib.lib().bsg_merge_split_u32(ka.ctx().handle, ka.ptr, ka.n, kb_.ptr, kb_.n, KeyBuf(low).ptr,
                                              KeyBuf(high).ptr, ka.mem, ka.stream), "merge_split")
    return low, high


@dataclass
class StageAssignment:
    """netsort.hpp:56-59."""

    partner: int = -1
    keep_low: bool = False


@dataclass
class BitonicSchedule:
    """netsort.hpp:61-64."""

    p: int = 1
    stages: List[List[StageAssignment]] = field(default_factory=list)


def _schedule(network: int, p: int) -> List[List[StageAssignment]]:
    S = ctypes.c_int(0)
    _lib.check(_lib.lib().bsg_network_schedule(network, int(p), None, None, 0, ctypes.byref(S)), "schedule")
    partner = np.empty(max(1, S.value * p), dtype=np.int32)
    keep = np.empty(max(1, S.value * p), dtype=np.int32)
    _lib.check(_lib.lib().bsg_network_schedule(network, int(p), partner.ctypes.data, keep.ctypes.data, S.value,
                                               ctypes.byref(S)), "schedule")
    return [[StageAssignment(int(partner[s * p + i]), bool(keep[s * p + i])) for i in range(p)]
            for s in range(S.value)]


def bitonic_schedule(p: int) -> BitonicSchedule:
    """netsort.hpp:70-89."""
    return BitonicSchedule(p, _schedule(_lib.NET_BTN, p))


def odd_even_rounds(p: int) -> List[List[StageAssignment]]:
    """netsort.hpp:95-108."""
    return _schedule(_lib.NET_OET, p)


@dataclass
class PreparedNetwork:
    """netsort.hpp:112-118.  `keys` is the unpadded input; padding to p blocks
    of ceil(n/p) keys happens on the device.  Truncating `stages` to a prefix of
    the schedule stops the network early, as in the reference."""

    p: int
    n: int
    pad: int
    keys: object
    stages: List[List[StageAssignment]]
    network: int

    @property
    def blocks(self) -> List[np.ndarray]:
        L = (self.n + self.p - 1) // self.p if self.p else 0
        host = np.concatenate([np.asarray(_host(self.keys), dtype=np.uint32),
                               np.full(self.pad, 0xFFFFFFFF, dtype=np.uint32)])
        return [host[w * L:(w + 1) * L] for w in range(self.p)]


def _host(x):
    from .core import _to_host

    return _to_host(x)


def _prepare(keys, p: int, network: int, stages) -> PreparedNetwork:
    kb = KeyBuf(keys)
    L = (kb.n + p - 1) // p
    return PreparedNetwork(p, kb.n, L * p - kb.n, kb.obj, stages, network)


def prepare_btn(keys, p: int) -> PreparedNetwork:
    """netsort.hpp:145-147."""
    return _prepare(keys, p, _lib.NET_BTN, bitonic_schedule(p).stages)


def prepare_oet(keys, p: int) -> PreparedNetwork:
    """netsort.hpp:149-151."""
    return _prepare(keys, p, _lib.NET_OET, odd_even_rounds(p))


def block_network_batched(arrays, p: int, network: int, stages_limit: int = -1):
    """Batched BTN/OET over a 2-D (num_arrays, len) uint32 array or tensor.
    Full runs return the same shape; truncated runs (0 <= stages_limit < S)
    return the padded (num_arrays, p*ceil(len/p)) block states."""
    shape = tuple(arrays.shape)
    if len(shape) != 2:
        raise ValueError("block_network_batched expects a 2-D array of arrays")
    num, length = int(shape[0]), int(shape[1])
    kb = KeyBuf(arrays)
    S = ctypes.c_int(0)
    _lib.check(_lib.lib().bsg_network_schedule(network, int(p), None, None, 0, ctypes.byref(S)), "schedule")
    full = stages_limit < 0 or stages_limit >= S.value
    L = (length + p - 1) // p if p > 0 else 0
    per = length if full else L * p
    out = kb.empty(num * per)
    stats = _lib.RunStats()
    _lib.check(_lib.lib().bsg_block_network_batched_u32(kb.ctx().handle, network, kb.ptr, KeyBuf(out).ptr, num,
                                                        length, int(p), int(stages_limit), ctypes.byref(stats), kb.mem,
                                                        kb.stream), "block_network_batched")
    return out.reshape(num, per), stats.as_dict()


def run_block_network(prep: PreparedNetwork, use_sequential_executor: bool = False) -> ParallelSortResult:
    """netsort.hpp:157-199: local sort, then one merge-split stage per
    superstep; concatenation minus the tail padding."""
    del use_sequential_executor
    S = ctypes.c_int(0)
    _lib.check(_lib.lib().bsg_network_schedule(prep.network, prep.p, None, None, 0, ctypes.byref(S)), "schedule")
    limit = len(prep.stages)
    stages_limit = -1 if limit >= S.value else limit
    kb = KeyBuf(prep.keys)
    if kb.n == 0:
        return ParallelSortResult(kb.empty(0), {"supersteps": 1 + S.value, "messages_sent": 0,
                                                "messages_delivered": 0, "words_sent": 0, "words_delivered": 0})
    arrays = kb.obj.reshape(1, kb.n)
    out, stats = block_network_batched(arrays, prep.p, prep.network, stages_limit)
    out = out.reshape(-1)[:prep.n]  # netsort.hpp:197 resize(n)
    return ParallelSortResult(out, stats)


def btn_sort(instance: SortInstance):
    """netsort.hpp:202-207."""
    instance.validate()
    if instance.algorithm != Algorithm.BTN:
        raise ValueError("btn_sort expects a BTN instance")
    return run_block_network(prepare_btn(instance.input, instance.processors)).output


def oet_sort(instance: SortInstance):
    """netsort.hpp:210-215."""
    instance.validate()
    if instance.algorithm != Algorithm.OET:
        raise ValueError("oet_sort expects an OET instance")
    return run_block_network(prepare_oet(instance.input, instance.processors)).output
