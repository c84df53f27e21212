import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")


@pytest.fixture(scope="session")
def orc():
    from oracle.pyoracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    """The reference's own headers compiled (oracle/_ref); None if not built."""
    from oracle.pyoracle import maybe_reference

    return maybe_reference()


@pytest.fixture(scope="session")
def bsg():
    import paper_1708_09495_b200 as pkg

    return pkg


@pytest.fixture(scope="session")
def cuda():
    """GPU tests must run on the CUDA path: fail loudly (never skip) when the
    library or the GPU is missing."""
    import torch

    import paper_1708_09495_b200 as pkg

    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    pkg._lib.lib()  # raises LibraryNotBuilt if the extension is missing
    pkg._lib.context(0)
    return torch


def stable_digit_sort(keys, round, radix):
    """radix_test.cpp:14-20: std::stable_sort on the digit alone."""
    bits = int(radix).bit_length() - 1
    k = np.asarray(keys, dtype=np.uint32)
    d = (k.astype(np.uint64) >> np.uint64(round * bits)) & np.uint64(radix - 1)
    return k[np.argsort(d, kind="stable")]
