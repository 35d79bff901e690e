"""Operand plumbing between numpy/torch objects and the C ABI.

numpy inputs travel as host pointers (the library copies them in and the
results out); torch CUDA tensors travel as device pointers on torch's current
stream.  Nothing here computes: it only describes memory.
"""

import ctypes

import numpy as np

from . import _lib


def is_torch(x):
    return type(x).__module__.split(".")[0] == "torch"


def torch_stream_ptr(t):
    import torch
    return torch.cuda.current_stream(t.device).cuda_stream


class HostMatrix:
    """2-D numpy operand: keeps a reference, knows its layout and ld."""

    def __init__(self, a, name="a"):
        from .kernels import ShapeError
        a = np.asarray(a)
        if a.ndim != 2:
            raise ShapeError(f"{name} must be 2-D, got shape {a.shape}")
        code = _lib.dtype_code(a.dtype)
        if not a.dtype.isnative:
            a = a.astype(a.dtype.newbyteorder("="))
        if a.flags.c_contiguous:
            layout, ld = _lib.ROW_MAJOR, max(a.shape[1], 1)
        elif a.flags.f_contiguous:
            layout, ld = _lib.COL_MAJOR, max(a.shape[0], 1)
        else:
            a = np.ascontiguousarray(a)
            layout, ld = _lib.ROW_MAJOR, max(a.shape[1], 1)
        self.a = a
        self.code = code
        self.layout = layout
        self.ld = ld
        self.shape = a.shape
        self.dtype = a.dtype

    @property
    def ptr(self):
        return ctypes.c_void_p(self.a.ctypes.data)


class DeviceMatrix:
    """2-D torch CUDA operand (row- or column-major, dense)."""

    def __init__(self, t, name="a"):
        import torch
        from .kernels import ShapeError
        if t.dim() != 2:
            raise ShapeError(f"{name} must be 2-D, got shape {tuple(t.shape)}")
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor")
        if t.dtype == torch.float64:
            code = _lib.F64
        elif t.dtype == torch.float32:
            code = _lib.F32
        else:
            raise TypeError(f"unsupported dtype {t.dtype}; expected float64 or float32")
        m, n = t.shape
        if t.is_contiguous():
            layout, ld = _lib.ROW_MAJOR, max(n, 1)
        elif t.t().is_contiguous():
            layout, ld = _lib.COL_MAJOR, max(m, 1)
        else:
            t = t.contiguous()
            layout, ld = _lib.ROW_MAJOR, max(n, 1)
        self.t = t
        self.code = code
        self.layout = layout
        self.ld = ld
        self.shape = (m, n)
        self.device = t.device.index or 0

    @property
    def ptr(self):
        return ctypes.c_void_p(self.t.data_ptr())


def host_empty(shape, dtype, order):
    return np.empty(shape, dtype=dtype, order=order)


def np_ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None
