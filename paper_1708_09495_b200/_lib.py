"""ctypes binding of the C ABI in include/bsg.h (libbsg.so, built for sm_100a).

This module is the only place that talks to the shared library.  There is no
CPU fallback: if libbsg.so is missing, importing works (so host-only helpers
can report the problem) but every call raises :class:`LibraryNotBuilt`; if no
B200 is present, context creation fails with :class:`DeviceError`.
"""
from __future__ import annotations

import ctypes
import os
import threading
from typing import Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BSG_LIB", os.path.join(_HERE, "libbsg.so"))

BSG_OK, BSG_EINVAL, BSG_EPROTO, BSG_ECUDA, BSG_ENOMEM, BSG_ENCCL = range(6)
MEM_HOST, MEM_DEVICE = 0, 1
NET_BTN, NET_OET = 0, 1
K_ONESWEEP, K_HIST, K_NETWORK, K_PR, K_FIRST_PASS, K_RELAXED_PASS, K_MSD_HIST, K_MSD_PARTITION, K_MSD_LOCAL = range(9)


class LibraryNotBuilt(RuntimeError):
    """libbsg.so is absent: run `make` (or __graft_entry__.build())."""


class BspError(RuntimeError):
    """Protocol failure; the reference's bspsort::bsp::bsp_error (bsp.hpp:38-41)."""


class DeviceError(RuntimeError):
    """CUDA failure or no usable sm_100 GPU (there is no CPU fallback)."""


class RunStats(ctypes.Structure):
    """bsp.hpp:86-92 RunStats."""

    _fields_ = [
        ("supersteps", ctypes.c_int32),
        ("messages_sent", ctypes.c_uint64),
        ("messages_delivered", ctypes.c_uint64),
        ("words_sent", ctypes.c_uint64),
        ("words_delivered", ctypes.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


class PrTiming(ctypes.Structure):
    """bsg_pr_timing: per-phase device time of one group sort (ms, max over members)."""

    _fields_ = [
        ("total_ms", ctypes.c_double),
        ("count_ms", ctypes.c_double),
        ("exchange_ms", ctypes.c_double),
        ("local_ms", ctypes.c_double),
        ("remote_bytes", ctypes.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


PR_PEER, PR_NCCL = 0, 1

_u32p = ctypes.c_void_p
_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64
_i = ctypes.c_int

# name -> (restype, argtypes); the exact symbol set declared in include/bsg.h
SIGNATURES = {
    "bsg_abi_version": (ctypes.c_int, []),
    "bsg_last_error": (ctypes.c_char_p, []),
    "bsg_ctx_launch_count": (ctypes.c_uint64, [_vp]),
    "bsg_ctx_create": (_i, [_i, ctypes.POINTER(_vp)]),
    "bsg_ctx_destroy": (_i, [_vp]),
    "bsg_ctx_release": (_i, [_vp]),
    "bsg_ctx_reserve": (_i, [_vp, _u64]),
    "bsg_ctx_set_timing": (_i, [_vp, _i]),
    "bsg_ctx_get_timing": (_i, [_vp, _i, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)]),
    "bsg_generate_uniform_u32": (_i, [_u32p, _u64, _u64]),
    "bsg_generate_uniform_at_u32": (_i, [_u32p, _u64, _u64, _u64]),
    "bsg_generate_uniform_device_u32": (_i, [_vp, _u32p, _u64, _u64, _vp]),
    "bsg_generate_uniform_device_at_u32": (_i, [_vp, _u32p, _u64, _u64, _u64, _vp]),
    "bsg_derive_seed": (ctypes.c_uint64, [_u64, ctypes.c_int32]),
    "bsg_checked_digit_bits": (_i, [_u64]),
    "bsg_generate_skewed_u32": (_i, [_u32p, _u64, _u64, _i, ctypes.c_double]),
    "bsg_network_schedule": (_i, [_i, _i, _vp, _vp, _i, ctypes.POINTER(_i)]),
    "bsg_partition_size_of": (ctypes.c_uint64, [_u64, _i, _i]),
    "bsg_partition_offset_of": (ctypes.c_uint64, [_u64, _i, _i]),
    "bsg_partition_owner_of": (_i, [_u64, _i, _u64]),
    "bsg_radix_sort_u32": (_i, [_vp, _u32p, _u32p, _u64, _i, _i, _vp]),
    "bsg_count_sort_round_u32": (_i, [_vp, _u32p, _u32p, _u64, _i, _i, _i, _vp]),
    "bsg_merge_split_u32": (_i, [_vp, _u32p, _u64, _u32p, _u64, _u32p, _u32p, _i, _vp]),
    "bsg_block_network_batched_u32": (
        _i, [_vp, _i, _u32p, _u32p, _u64, ctypes.c_uint32, _i, _i, ctypes.POINTER(RunStats), _i, _vp]),
    "bsg_parallel_radix_sort_u32": (
        _i, [_vp, _u32p, _u32p, _u64, _i, _i, _i, ctypes.POINTER(RunStats), _i, _vp]),
    "bsg_sort_instance_u32": (_i, [_vp, _u32p, _u32p, _u64, _i, _i, _u64, _i, _vp]),
    "bsg_pr_count_digits": (_i, [_vp, _u32p, _u64, _i, _i, _vp, _vp]),
    "bsg_pr_plan": (_i, [_vp, _vp, _u64, _i, _i, _i, _i, _vp, _vp, _vp, _vp]),
    "bsg_pr_local_sort": (_i, [_vp, _u32p, _u32p, _u64, _i, _i, _vp]),
    "bsg_pr_plan_host": (_i, [_vp, _u64, _i, _i, _i, _vp, _vp, _vp]),
    "bsg_pr_rebuild": (_i, [_vp, _u32p, _u64, _vp, _i, _i, _i, _vp, _u32p, _vp]),
    "bsg_ctx_enable_peer_access": (_i, [_vp, ctypes.POINTER(_i)]),
    "bsg_pr_peer_scatter": (_i, [_vp, _u32p, _u64, _vp, _u64, _i, _i, _i, _i, ctypes.POINTER(_vp), _vp]),
    "bsg_pr_fused_round": (_i, [_vp, _u32p, _u64, _vp, _u64, _i, _i, _i, _i, ctypes.POINTER(_vp), _vp]),
    "bsg_ctx_create_group": (_i, [ctypes.POINTER(_i), _i, ctypes.POINTER(_vp)]),
    "bsg_ctx_group_size": (_i, [_vp]),
    "bsg_ctx_group_device": (_i, [_vp, _i]),
    "bsg_group_range_offset": (ctypes.c_uint64, [_u64, _i, _i, _i]),
    "bsg_group_range_size": (ctypes.c_uint64, [_u64, _i, _i, _i]),
    "bsg_pr_group_sort_u32": (
        _i, [_vp, ctypes.POINTER(_vp), _u64, _i, _i, _i, _i, ctypes.POINTER(RunStats), ctypes.POINTER(PrTiming),
             ctypes.POINTER(_vp)]),
}

_lib: Optional[ctypes.CDLL] = None
_lock = threading.RLock()


def lib() -> ctypes.CDLL:
    """Loads libbsg.so once and declares every C-ABI signature."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise LibraryNotBuilt(f"{LIB_PATH} not found; build it with `make lib` (no CPU fallback exists)")
        h = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
        return h


def last_error() -> str:
    msg = lib().bsg_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    """Maps C-ABI status codes to the reference's exception types."""
    if status == BSG_OK:
        return
    msg = last_error()
    text = f"{what}: {msg}" if what else msg
    if status == BSG_EINVAL:
        raise ValueError(text)  # std::invalid_argument
    if status == BSG_EPROTO:
        raise BspError(text)
    if status == BSG_ENOMEM:
        raise MemoryError(text)
    raise DeviceError(text)


class Context:
    """Owns one bsg_ctx bound to a CUDA device (workspace cache, launch count)."""

    def __init__(self, device: int = 0):
        h = _vp()
        check(lib().bsg_ctx_create(device, ctypes.byref(h)), "bsg_ctx_create")
        self.handle = h
        self.device = device

    @property
    def launches(self) -> int:
        return int(lib().bsg_ctx_launch_count(self.handle))

    def set_timing(self, enable: bool) -> None:
        """Per-launch CUDA-event timing of kernel classes (K_ONESWEEP, ...)."""
        check(lib().bsg_ctx_set_timing(self.handle, int(enable)), "bsg_ctx_set_timing")

    def kernel_time(self, kernel_class: int):
        """(total ms, launches) of one kernel class since timing was enabled."""
        ms, cnt = ctypes.c_double(0), ctypes.c_uint64(0)
        check(lib().bsg_ctx_get_timing(self.handle, kernel_class, ctypes.byref(ms), ctypes.byref(cnt)),
              "bsg_ctx_get_timing")
        return ms.value, cnt.value

    def reserve(self, n: int) -> None:
        check(lib().bsg_ctx_reserve(self.handle, n), "bsg_ctx_reserve")

    def release(self) -> None:
        """Frees the cached device workspace (the context stays usable)."""
        check(lib().bsg_ctx_release(self.handle), "bsg_ctx_release")

    def close(self) -> None:
        if getattr(self, "handle", None):
            lib().bsg_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


class GroupContext(Context):
    """A multi-GPU group context (bsg_ctx_create_group): p logical workers of
    the parallel radix sort spread over `devices` (may repeat a device)."""

    def __init__(self, devices):
        devs = (_i * len(devices))(*[int(d) for d in devices])
        h = _vp()
        check(lib().bsg_ctx_create_group(devs, len(devices), ctypes.byref(h)), "bsg_ctx_create_group")
        self.handle = h
        self.device = int(devices[0])
        self.devices = [int(d) for d in devices]

    @property
    def size(self) -> int:
        return int(lib().bsg_ctx_group_size(self.handle))


_contexts: dict = {}


def context(device: Optional[int] = None) -> Context:
    """Per-device default context (created lazily)."""
    if device is None:
        device = _current_device()
    ctx = _contexts.get(device)
    if ctx is None:
        with _lock:
            ctx = _contexts.get(device)
            if ctx is None:
                ctx = Context(device)
                _contexts[device] = ctx
    return ctx


def release_all() -> None:
    """Frees the cached workspace of every default context."""
    for ctx in list(_contexts.values()):
        ctx.release()


def _current_device() -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # pragma: no cover
        pass
    return 0
