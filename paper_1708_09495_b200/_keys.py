"""Key-array plumbing: numpy (host) arrays go through BSG_MEM_HOST, torch CUDA
tensors through BSG_MEM_DEVICE on the tensor's current stream.  Torch is used
only for device memory and streams; all compute is in libbsg.so."""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

try:  # torch is optional for host-only use
    import torch
except ImportError:  # pragma: no cover
    torch = None


def is_device(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


class KeyBuf:
    """A contiguous uint32 key buffer plus how the C ABI should see it."""

    def __init__(self, keys):
        if is_device(keys):
            t = keys
            if t.dtype == torch.int32:
                t = t.view(torch.uint32)
            if t.dtype != torch.uint32:
                raise TypeError(f"device keys must be uint32 (or int32 bit patterns), got {t.dtype}")
            self.obj = t.contiguous().view(-1)
            self.mem = _lib.MEM_DEVICE
            self.device = self.obj.device.index or 0
            self.stream = torch.cuda.current_stream(self.obj.device).cuda_stream
        else:
            if torch is not None and isinstance(keys, torch.Tensor):
                keys = keys.detach().cpu().numpy()
            a = np.asarray(keys)
            if a.dtype != np.uint32:
                if a.size and (a.min() < 0 or a.max() > 0xFFFFFFFF):
                    raise ValueError("keys must be uint32")
                a = a.astype(np.uint32)
            self.obj = np.ascontiguousarray(a).reshape(-1)
            self.mem = _lib.MEM_HOST
            self.device = None
            self.stream = None

    @property
    def n(self) -> int:
        return int(self.obj.numel()) if self.mem == _lib.MEM_DEVICE else int(self.obj.size)

    @property
    def ptr(self) -> int:
        if self.mem == _lib.MEM_DEVICE:
            return int(self.obj.data_ptr())
        return self.obj.ctypes.data_as(ctypes.c_void_p).value or 0

    def empty(self, n: int):
        """A new output buffer of the same kind."""
        if self.mem == _lib.MEM_DEVICE:
            return torch.empty(n, dtype=torch.uint32, device=self.obj.device)
        return np.empty(n, dtype=np.uint32)

    def wrap(self, out) -> "KeyBuf":
        return KeyBuf(out)

    def ctx(self) -> _lib.Context:
        return _lib.context(self.device if self.device is not None else None)


def ptr_of(x) -> int:
    if is_device(x):
        return int(x.data_ptr())
    return x.ctypes.data_as(ctypes.c_void_p).value or 0
