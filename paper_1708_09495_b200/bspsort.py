"""bspsort.hpp:15-25 sort_instance: validate, then dispatch on the algorithm."""
from __future__ import annotations

from . import netsort, radix
from .core import Algorithm, SortInstance


def sort_instance(instance: SortInstance):
    """Dispatches a sort instance to its algorithm (bspsort.hpp:15-25)."""
    instance.validate()
    if instance.algorithm == Algorithm.SR4:
        return radix.serial_radix_sort(instance.input, instance.radix)
    if instance.algorithm in (Algorithm.PR4, Algorithm.PR2):
        return radix.parallel_radix_sort(instance)
    if instance.algorithm == Algorithm.BTN:
        return netsort.btn_sort(instance)
    if instance.algorithm == Algorithm.OET:
        return netsort.oet_sort(instance)
    raise ValueError("sort_instance: unknown algorithm")
