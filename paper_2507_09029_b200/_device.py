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
