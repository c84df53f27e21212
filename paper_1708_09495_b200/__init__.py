"""B200-native (sm_100a) integer-sorting hot path of arXiv 1708.09495.

Python mirror of the reference's C++ API (``bspsort::radix``,
``bspsort::netsort``, ``bspsort::sort_instance``) over the C ABI in
include/bsg.h (libbsg.so).  All sorting runs in hand-written CUDA kernels;
there is no CPU fallback.
"""
from . import _lib
from ._lib import BspError, Context, DeviceError, LibraryNotBuilt, RunStats
from .bspsort import sort_instance
from .core import (Algorithm, Key, SortInstance, algorithm_from_name, algorithm_name, derive_seed, digit_bits,
                   generate_skewed_keys, generate_uniform_keys, generate_uniform_keys_at,
                   generate_uniform_keys_device, is_power_of_two, key_bits, log2_exact,
                   verify_sorted_permutation)
from . import netsort, radix

__all__ = [
    "Algorithm", "BspError", "Context", "DeviceError", "Key", "LibraryNotBuilt", "RunStats", "SortInstance",
    "algorithm_from_name", "algorithm_name", "derive_seed", "digit_bits", "generate_skewed_keys",
    "generate_uniform_keys", "generate_uniform_keys_at", "generate_uniform_keys_device", "is_power_of_two", "key_bits", "log2_exact", "netsort", "radix", "sort_instance",
    "verify_sorted_permutation",
]
