"""Gradient-alignment diagnostic on the GPU (diagnostics.py:24-78; SURVEY.md
§8f row 4).

`gradient_alignment` runs the worker's masked forward/backward and the
unmasked one on the same batch (models.masked_forward / flat_gradient), then
ONE `sdp_restricted_dots` launch computes, for every requested layer, the dot
product and both squared norms over the worker's support in float64
(warp-shuffle partials, deterministic fixed-order second pass).  Only the
per-layer scalars come back to the host.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._device import ptr, sdp_dtype, stream_ptr, upload_struct
from .models import flat_gradient, masked_forward

REDUCE_DTYPE = np.dtype([("offset", "<i8"), ("length", "<i8"), ("segment", "<i4"), ("pad_", "<i4")])
CHUNK = 16384


@dataclass(frozen=True)
class AlignmentSample:
    step: int
    worker_id: int
    layer: str
    cosine: float | None
    reason: str | None = None  # set when cosine is absent


def restricted_dots(a: torch.Tensor, b: torch.Tensor, support: torch.Tensor | None,
                    segments: list[tuple[int, int]]) -> np.ndarray:
    """[(offset, length)] -> [S, 4] float64 (sum ab, sum aa, sum bb, count)."""
    tasks = []
    for s, (off, length) in enumerate(segments):
        for k in range(0, max(length, 1), CHUNK):
            if length:
                tasks.append((off + k, min(CHUNK, length - k), s, 0))
    t = np.array(tasks, dtype=REDUCE_DTYPE)
    dev = a.device
    t_dev = upload_struct(t, dev)
    partials = torch.empty(max(1, len(t)) * 4, dtype=torch.float64, device=dev)
    out = torch.empty(len(segments) * 4, dtype=torch.float64, device=dev)
    sup = None if support is None else support.view(torch.uint8)
    N.call("sdp_restricted_dots", sdp_dtype(a.dtype), ptr(a), ptr(b), ptr(sup), ptr(t_dev), len(t),
           len(segments), ptr(partials), ptr(out), stream_ptr(dev))
    return out.view(-1, 4).cpu().numpy()


def _cosine(row) -> tuple[float | None, str | None]:
    ab, aa, bb, n = row
    if n == 0:
        return None, "empty-support"
    na, nb = math.sqrt(aa), math.sqrt(bb)
    if na == 0.0 or nb == 0.0:
        return None, "zero-norm"
    return float(ab / (na * nb)), None


def restricted_cosine(g_masked, g_unmasked, support) -> tuple[float | None, str | None]:
    """Cosine over the support only; absent on degenerate input (diagnostics.py:33-47)."""
    a = torch.as_tensor(g_masked)
    b = torch.as_tensor(g_unmasked, device=a.device).to(a.dtype).contiguous()
    s = torch.as_tensor(support, device=a.device).to(torch.bool).contiguous()
    return _cosine(restricted_dots(a.contiguous(), b, s, [(0, a.numel())])[0])


def gradient_alignment(model, worker, xs, ys, layers, g_mask=None, step: int = 0) -> list[AlignmentSample]:
    """Per-layer cosine between masked and unmasked gradients (diagnostics.py:50-78)."""
    if g_mask is None:
        loss_m, tape_m, params_m = masked_forward(model, worker, xs, ys)
        g_mask = flat_gradient(model, tape_m, loss_m, params_m)
    loss_u, tape_u, params_u = masked_forward(model, None, xs, ys)
    g_unmask = flat_gradient(model, tape_u, loss_u, params_u)
    segs = [(model.topology.index[layer].offset, model.topology.index[layer].size) for layer in layers]
    rows = restricted_dots(g_mask.contiguous(), g_unmask.contiguous(), worker.param_mask_bool, segs)
    out = []
    for layer, row in zip(layers, rows):
        cos, reason = _cosine(row)
        out.append(AlignmentSample(step, worker.worker_id, layer, cos, reason))
    return out
