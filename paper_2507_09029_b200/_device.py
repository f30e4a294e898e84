"""Device plumbing shared by the host modules: torch is used only for device
memory, streams and host<->device copies; all compute goes through libsdp."""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .errors import CudaError


def device(dev=None) -> torch.device:
    if not torch.cuda.is_available():
        raise CudaError("no CUDA device: the subnetwork-DP hot path runs only on the GPU")
    if dev is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(dev)
    if dev.type != "cuda":
        raise CudaError(f"expected a CUDA device, got {dev}")
    return dev


def stream_ptr(dev: torch.device | None = None) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def ptr(t: torch.Tensor | None) -> C.c_void_p | None:
    return None if t is None else C.c_void_p(t.data_ptr())


def upload_struct(arr: np.ndarray, dev: torch.device) -> torch.Tensor:
    """Copy a numpy structured/plain array into a 16-B aligned device byte buffer."""
    raw = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
    n = max(16, (raw.size + 15) // 16 * 16)
    host = torch.zeros(n, dtype=torch.uint8)
    if raw.size:
        host[: raw.size] = torch.from_numpy(raw.copy())
    return host.to(dev, non_blocking=False)


def mask_bytes_for(n_workers: int) -> int:
    for b in (1, 2, 4, 8):
        if n_workers <= 8 * b:
            return b
    raise ValueError(f"at most {N.MAX_WORKERS} workers are supported, got {n_workers}")


MASK_TORCH_DTYPE = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}


def slice_dtype(t: torch.dtype) -> int:
    """dtype code of the (typeless) gather kernels: 2-byte types move as bits."""
    if t in (torch.bfloat16, torch.float16):
        return N.DTYPE_U16
    if t == torch.uint8:
        return N.DTYPE_U8
    return sdp_dtype(t)


def sdp_dtype(t: torch.dtype) -> int:
    if t == torch.float32:
        return N.DTYPE_F32
    if t == torch.float64:
        return N.DTYPE_F64
    raise TypeError(f"owner sync runs on float32 or float64 buffers, got {t}")


_INPLACE_DUNDERS = frozenset({"__setitem__", "__iadd__", "__isub__", "__imul__", "__itruediv__",
                              "__ifloordiv__", "__imod__", "__ipow__", "__ilshift__", "__irshift__",
                              "__iand__", "__ior__", "__ixor__", "__imatmul__"})


class ReadOnlyTensor(torch.Tensor):
    """A device array the caller may read but not write: the reference freezes
    an assignment's arrays (masking.py:206-207, `setflags(write=False)`), so an
    in-place op, item assignment or `out=` into one raises ValueError exactly as
    writing a read-only numpy array does.  Views taken from it stay read-only;
    every other result is a plain tensor.  libsdp reads it through data_ptr()."""

    @classmethod
    def __torch_function__(cls, func, types, args=(), kwargs=None):
        kwargs = kwargs or {}
        name = getattr(func, "__name__", "")
        first = args[0] if args else None
        if isinstance(first, ReadOnlyTensor) and (
                name in _INPLACE_DUNDERS or (name.endswith("_") and not name.startswith("_"))):
            raise ValueError(f"assignment array is read-only ({name})")
        out = kwargs.get("out")
        if out is not None and any(isinstance(o, ReadOnlyTensor)
                                   for o in (out if isinstance(out, (tuple, list)) else (out,))):
            raise ValueError("assignment array is read-only (out=)")
        with torch._C.DisableTorchFunctionSubclass():
            ret = func(*args, **kwargs)
        if isinstance(first, ReadOnlyTensor) and isinstance(ret, torch.Tensor) and not \
                isinstance(ret, ReadOnlyTensor) and ret._is_view() and ret.numel() and \
                ret.untyped_storage().data_ptr() == first.untyped_storage().data_ptr():
            ret = ret.as_subclass(ReadOnlyTensor)
        return ret


def read_only(t: torch.Tensor | None) -> torch.Tensor | None:
    if t is None or isinstance(t, ReadOnlyTensor):
        return t
    return t.as_subclass(ReadOnlyTensor)
