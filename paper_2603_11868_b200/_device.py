"""Host <-> device plumbing for the kernel-dispatch boundary.

Arguments of particle_for / particle_reduce may be host numpy arrays (the
reference's registry views) or CUDA torch tensors.  ``Staging`` uploads host
arrays for one native call and writes the arrays the kernel mutates back in
place, so host callers observe exactly the reference's in-place semantics
(physics bodies mutate the registry storage, variables.py:57-59).
"""

from __future__ import annotations

import numpy as np

from . import _native


def torch_mod():
    import torch
    return torch


def is_tensor(a):
    try:
        import torch
    except ImportError:   # pragma: no cover
        return False
    return isinstance(a, torch.Tensor)


_NP_TO_TORCH = {
    np.dtype(np.float32): "float32", np.dtype(np.float64): "float64",
    np.dtype(np.int64): "int64", np.dtype(np.int32): "int32",
    np.dtype(np.uint32): "int32", np.dtype(np.uint8): "uint8",
}


def device_of(policy):
    torch = torch_mod()
    _native.require_cuda()
    idx = getattr(policy, "device", 0) or 0
    return torch.device("cuda", int(idx))


def stream_ptr(device):
    torch = torch_mod()
    return C_void(torch.cuda.current_stream(device).cuda_stream)


def C_void(v):
    import ctypes
    return ctypes.c_void_p(v)


def ptr(t):
    import ctypes
    if t is None:
        return ctypes.c_void_p(0)
    return ctypes.c_void_p(t.data_ptr())


class Staging:
    """Upload host arrays for one call; write mutated ones back on exit."""

    def __init__(self, device):
        self.device = device
        self._back = []
        self._keep = []

    def to_dev(self, a, writeback=False):
        torch = torch_mod()
        if a is None:
            return None
        if is_tensor(a):
            if a.device != self.device:
                raise TypeError("tensor argument lives on another device")
            if not a.is_contiguous():
                raise TypeError("tensor arguments must be contiguous")
            return a
        arr = np.asarray(a)
        if not arr.flags.c_contiguous:
            if writeback:
                raise TypeError("mutated arrays must be C-contiguous")
            arr = np.ascontiguousarray(arr)
        tname = _NP_TO_TORCH.get(arr.dtype)
        if tname is None:
            raise TypeError(f"unsupported array dtype {arr.dtype}")
        view = arr.view(np.int32) if arr.dtype == np.uint32 else arr
        host = torch.from_numpy(view)
        dev = host.to(self.device, non_blocking=False)
        self._keep.append(dev)
        if writeback:
            self._back.append((arr, dev))
        return dev

    def empty(self, shape, dtype):
        torch = torch_mod()
        t = torch.empty(shape, dtype=dtype, device=self.device)
        self._keep.append(t)
        return t

    def __enter__(self):
        return self

    def __exit__(self, exc_type, exc, tb):
        if exc_type is None:
            for arr, dev in self._back:
                host = dev.cpu().numpy()
                arr[...] = host.view(arr.dtype).reshape(arr.shape)
        self._back.clear()
        self._keep.clear()
        return False


def workspace(device, nbytes):
    torch = torch_mod()
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)
