"""Training-step integration: N subnetwork workers + owner-subset sync on B200.

The reference's protocol step (engine.py:202-223) is: every worker runs a
forward/backward on its subnetwork, the gradients are masked-averaged
(`aggregate`), and one SGD-Nesterov update is applied.  Here the per-worker
forward/backward is dense cuDNN/cuBLAS in bf16 autocast (not the optimisation
target), dropped residual blocks are never executed (models.py:161-163), and
the sync + update is ONE k_owner_sync launch with the Nesterov epilogue and
the bf16 weight cast fused (SDP_SYNC_NESTEROV).

`ResNet18Cifar` is the BASELINE configs[1]/[2] model: CIFAR stem, GroupNorm(2),
torchvision BasicBlock (ReLU after the residual add), the 3 downsampling blocks
always active.  Its parameter layout is zoo.resnet18_cifar_topology.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F

from . import _native as N
from . import engine, masking, zoo
from ._device import ptr, stream_ptr
from .errors import ConfigError, NumericalError, UsageError
from .models import _channels_last_bf16, group_norm
from .topology import GlobalModel


class _ChannelScatterAdd(torch.autograd.Function):
    """out = sc with o added into channels idx (the compact block output
    written back into the residual stream), keeping channels-last layouts in
    both directions (torch's index_add / index_select backward would hand
    the next GroupNorm an NCHW gradient and force a transpose copy)."""

    @staticmethod
    def forward(ctx, sc, idx, o):
        ctx.save_for_backward(idx)
        fmt = torch.channels_last if sc.is_contiguous(memory_format=torch.channels_last) else torch.contiguous_format
        ctx.fmt = fmt
        return sc.clone(memory_format=fmt).index_add_(1, idx, o)

    @staticmethod
    def backward(ctx, g):
        (idx,) = ctx.saved_tensors
        b, _, h, w = g.shape
        go = torch.empty((b, idx.numel(), h, w), dtype=g.dtype, device=g.device, memory_format=ctx.fmt)
        torch.index_select(g, 1, idx, out=go)
        return g, None, go


def _channel_scatter_add(sc, idx, o):
    return _ChannelScatterAdd.apply(sc, idx, o)


class ResNet18Cifar:
    def __init__(self, classes: int = 10, norm_groups: int = 2):
        self.classes, self.norm_groups = classes, norm_groups
        self.topology = zoo.resnet18_cifar_topology(classes, norm_groups)
        self.block_plan = []
        cin = 64
        for stage, planes in enumerate((64, 128, 256, 512), start=1):
            for j in range(2):
                stride = 2 if (stage > 1 and j == 0) else 1
                self.block_plan.append((f"layer{stage}.{j}", stride, stride != 1 or cin != planes))
                cin = planes

    def build_topology(self):
        return self.topology

    def _gn(self, x, gamma, beta, worker, layer_id, relu=False):
        """GroupNorm (+ReLU); over the worker's live channels only when some
        are dead (ops.py:140-204: dead channels output exact zeros)."""
        flags = None if worker is None else worker.channel_active.get(layer_id)
        if flags is None or bool(np.all(flags)):
            return group_norm(x, self.norm_groups, gamma, beta, relu=relu)
        from .models import active_group_norm
        act = torch.as_tensor(np.array(flags, dtype=bool), device=x.device)
        out = active_group_norm(x, self.norm_groups, gamma, beta, act)
        return F.relu(out) if relu else out

    @staticmethod
    def _layout(x):
        """Training (bf16 autocast) keeps activations channels-last end to end:
        cuDNN's NHWC kernels and libsdp's GroupNorm need no layout transposes."""
        return x.contiguous(memory_format=torch.channels_last) if torch.is_autocast_enabled("cuda") else x

    def forward(self, params, x, worker=None, block_mode: str = "skip"):
        g = self.norm_groups
        h = F.conv2d(self._layout(x), params["conv1.w"], padding=1)
        h = group_norm(h, g, params["gn1.gamma"], params["gn1.beta"], relu=True)
        for bi, (p, stride, down) in enumerate(self.block_plan):
            live = True if worker is None else bool(worker.block_active[bi])
            if not live and block_mode == "skip":
                continue  # a dropped block is the identity and is never executed
            o = F.conv2d(h, params[f"{p}.conv1.w"], stride=stride, padding=1)
            o = self._gn(o, params[f"{p}.gn1.gamma"], params[f"{p}.gn1.beta"], worker, f"{p}.conv1", relu=True)
            o = F.conv2d(o, params[f"{p}.conv2.w"], padding=1)
            o = self._gn(o, params[f"{p}.gn2.gamma"], params[f"{p}.gn2.beta"], worker, f"{p}.conv2")
            if down:
                sc = downsample(h, params[f"{p}.down.w"], stride)
                sc = group_norm(sc, g, params[f"{p}.down_gn.gamma"], params[f"{p}.down_gn.beta"])
            else:
                sc = h
            if not live:
                o = o * 0.0
            h = F.relu(o + sc)
        return F.linear(h.mean(dim=(2, 3)), params["fc.w"], params["fc.b"])

    def forward_compact(self, cp, x, sub):
        """Width-wise subnetwork (config C3): cp holds only the worker's live
        conv1/conv2 channels (models.SubnetLayout); GroupNorm statistics over
        the live channels of each original group (ragged); the
        block output is scattered back into the residual stream's channels."""
        from .models import ragged_group_norm
        g = self.norm_groups
        h = F.conv2d(self._layout(x), cp["conv1.w"], padding=1)
        h = group_norm(h, g, cp["gn1.gamma"], cp["gn1.beta"], relu=True)
        for p, stride, down in self.block_plan:
            if not sub.present(f"{p}.conv1.w"):
                continue
            planes = self.topology.index[f"{p}.conv1.w"].shape[0]
            gsize = planes // g
            a1 = sub.channels(f"{p}.conv1", planes)
            a2 = sub.channels(f"{p}.conv2", planes)
            o = F.conv2d(h, cp[f"{p}.conv1.w"], stride=stride, padding=1)
            # the channels-last kernel needs only the per-group counts (the
            # channel -> group map would be two index divisions per block)
            fast = _channels_last_bf16(o)
            o = ragged_group_norm(o, None if fast else a1 // gsize, g, cp[f"{p}.gn1.gamma"], cp[f"{p}.gn1.beta"],
                                  counts=sub.group_counts(f"{p}.conv1", planes, g), relu=True)
            o = F.conv2d(o, cp[f"{p}.conv2.w"], padding=1)
            o = ragged_group_norm(o, None if fast else a2 // gsize, g, cp[f"{p}.gn2.gamma"], cp[f"{p}.gn2.beta"],
                                  counts=sub.group_counts(f"{p}.conv2", planes, g))
            if down:
                sc = downsample(h, cp[f"{p}.down.w"], stride)
                sc = group_norm(sc, g, cp[f"{p}.down_gn.gamma"], cp[f"{p}.down_gn.beta"])
            else:
                sc = h
            h = F.relu(_channel_scatter_add(sc, a2, o.to(sc.dtype)))
        return F.linear(h.mean(dim=(2, 3)), cp["fc.w"], cp["fc.b"])


_LN_PARTS: dict = {}


class _LayerNormBF16(torch.autograd.Function):
    """Row LayerNorm of bf16 activations on libsdp's k_ln_fwd / k_ln_bwd (one
    warp per row, fp32 statistics; the weight / bias gradients reduced per CTA
    and folded in CTA order).  torch's bf16 layer_norm backward spent 74 us of
    a [8192, 768] call in its gamma/beta kernel: ~1 ms of a GPT-2 worker step."""

    @staticmethod
    def forward(ctx, x, w, b, eps):
        cols = x.shape[-1]
        rows = x.numel() // cols
        x2 = x.contiguous()
        y = torch.empty_like(x2)
        mean = torch.empty(rows, dtype=torch.float32, device=x.device)
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
        N.call("sdp_layer_norm_fwd", ptr(x2), rows, cols, ptr(w), ptr(b), C.c_float(eps), ptr(y), ptr(mean),
               ptr(rstd), stream_ptr(x.device))
        ctx.save_for_backward(x2, w, mean, rstd)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, w, mean, rstd = ctx.saved_tensors
        cols = x.shape[-1]
        rows = x.numel() // cols
        dy = dy.contiguous()
        if dy.data_ptr() % 16:
            dy = dy.clone()
        key = (rows, cols, x.device)
        parts = _LN_PARTS.get(key)
        if parts is None:
            parts = _LN_PARTS[key] = N.lib().sdp_layer_norm_bwd_parts(rows, cols)
        scratch = torch.empty(2 * cols * parts, dtype=torch.float32, device=x.device)
        dx = torch.empty_like(x)
        dw = torch.empty(cols, dtype=torch.bfloat16, device=x.device)
        db = torch.empty(cols, dtype=torch.bfloat16, device=x.device)
        N.call("sdp_layer_norm_bwd", ptr(dy), ptr(x), rows, cols, ptr(w), ptr(mean), ptr(rstd), ptr(dx), ptr(dw),
               ptr(db), ptr(scratch), parts, stream_ptr(x.device))
        return dx, dw, db, None


class _AddLayerNormBF16(torch.autograd.Function):
    """(s, LN(s)) with s = a + b in bf16, on libsdp's residual-fused row
    kernels: one pass writes the residual stream and its normalisation, and
    the backward adds the residual branch's gradient into dx -- the two
    bf16 adds of an unfused block (forward sum, backward accumulation) go
    away."""

    @staticmethod
    def forward(ctx, a, b, w, bias, eps):
        cols = a.shape[-1]
        rows = a.numel() // cols
        s = torch.empty_like(a)
        y = torch.empty_like(a)
        mean = torch.empty(rows, dtype=torch.float32, device=a.device)
        rstd = torch.empty(rows, dtype=torch.float32, device=a.device)
        N.call("sdp_add_layer_norm_fwd", ptr(a), ptr(b), rows, cols, ptr(w), ptr(bias), C.c_float(eps), ptr(s),
               ptr(y), ptr(mean), ptr(rstd), stream_ptr(a.device))
        ctx.save_for_backward(s, w, mean, rstd)
        return s, y

    @staticmethod
    def backward(ctx, ds, dy):
        s, w, mean, rstd = ctx.saved_tensors
        cols = s.shape[-1]
        rows = s.numel() // cols
        dy = _aligned16(dy if dy is not None else torch.zeros_like(s))
        key = (rows, cols, s.device)
        parts = _LN_PARTS.get(key)
        if parts is None:
            parts = _LN_PARTS[key] = N.lib().sdp_layer_norm_bwd_parts(rows, cols)
        scratch = torch.empty(2 * cols * parts, dtype=torch.float32, device=s.device)
        dx = torch.empty_like(s)
        dw = torch.empty(cols, dtype=torch.bfloat16, device=s.device)
        db = torch.empty(cols, dtype=torch.bfloat16, device=s.device)
        if ds is None:
            N.call("sdp_layer_norm_bwd", ptr(dy), ptr(s), rows, cols, ptr(w), ptr(mean), ptr(rstd), ptr(dx),
                   ptr(dw), ptr(db), ptr(scratch), parts, stream_ptr(s.device))
        else:
            ds = _aligned16(ds)
            N.call("sdp_layer_norm_bwd_res", ptr(dy), ptr(s), ptr(ds), rows, cols, ptr(w), ptr(mean), ptr(rstd),
                   ptr(dx), ptr(dw), ptr(db), ptr(scratch), parts, stream_ptr(s.device))
        return dx, dx, dw, db, None


def _add_layer_norm(a, b, shape, w, bias, eps: float = 1e-5):
    """(a + b, LayerNorm(a + b)); fused on libsdp under bf16 autocast."""
    if a.dtype == torch.bfloat16 and b.dtype == torch.bfloat16 and torch.is_autocast_enabled("cuda"):
        with torch.autocast("cuda", enabled=False):
            wb, bb = w.to(a.dtype), bias.to(a.dtype)
            if (_ln_native(a, wb, bb) and len(shape) == 1 and a.shape == b.shape
                    and a.data_ptr() % 16 == 0 and b.data_ptr() % 16 == 0 and a.is_contiguous() and b.is_contiguous()):
                return _AddLayerNormBF16.apply(a, b, _aligned16(wb), _aligned16(bb), eps)
    s = a + b
    return s, _layer_norm(s, shape, w, bias, eps)


def _ln_native(x, w, b) -> bool:
    cols = x.shape[-1]
    return (x.is_cuda and x.dtype == torch.bfloat16 and cols % 256 == 0 and cols <= 1024
            and w.dtype == torch.bfloat16 and b.dtype == torch.bfloat16)


def _aligned16(t: torch.Tensor) -> torch.Tensor:
    return t if t.is_contiguous() and t.data_ptr() % 16 == 0 else t.contiguous().clone()


def _layer_norm(x, shape, w, b, eps: float = 1e-5):
    """LayerNorm over the last dim; under bf16 autocast bf16 activations stay
    bf16 in and out (fp32 statistics inside the kernel) instead of autocast's
    fp32 upcast, on libsdp's row kernels (_LayerNormBF16)."""
    if x.dtype == torch.bfloat16 and torch.is_autocast_enabled("cuda"):
        with torch.autocast("cuda", enabled=False):
            wb, bb = w.to(x.dtype), b.to(x.dtype)
            if _ln_native(x, wb, bb) and len(shape) == 1:
                x2 = x if x.data_ptr() % 16 == 0 else x.clone()
                return _LayerNormBF16.apply(x2, _aligned16(wb), _aligned16(bb), eps)
            return F.layer_norm(x, shape, wb, bb, eps)
    return F.layer_norm(x, shape, w, b, eps)


class _SplitHeads(torch.autograd.Function):
    """qkv [b*t, 3e] -> q, k, v [b, nh, t, hd] (strided views, as
    `view(b, t, 3, nh, hd).permute(2, 0, 3, 1, 4)`).  The backward writes the
    three head gradients straight into one [b, t, 3, nh, hd] buffer, which IS
    the [b*t, 3e] gradient of qkv; autograd's unbind/permute/view backward
    stacked them ([3, b, nh, t, hd]) and then copied that into the qkv
    layout: a 97 us cat + a copy per block on a GPT-2 worker step.  libsdp
    k_merge_heads interleaves the three in one pass whatever their (batch,
    head, seq) strides (strided torch copies otherwise)."""

    @staticmethod
    def forward(ctx, qkv, b, t, nh, hd):
        ctx.shape = (b, t, nh, hd)
        q, k, v = qkv.view(b, t, 3, nh, hd).permute(2, 0, 3, 1, 4)
        return q, k, v

    @staticmethod
    def backward(ctx, dq, dk, dv):
        b, t, nh, hd = ctx.shape
        ref = next(x for x in (dq, dk, dv) if x is not None)
        g = torch.empty((b, t, 3, nh, hd), dtype=ref.dtype, device=ref.device)
        es = ref.element_size()
        st = ref.stride()
        if (all(x is not None and x.stride() == st and x.dtype == ref.dtype and x.data_ptr() % 16 == 0
                for x in (dq, dk, dv))
                and ref.is_cuda and st[3] == 1 and es in (2, 4) and hd * es % 16 == 0
                and all(s_ * es % 16 == 0 for s_ in st[:3])):  # libsdp k_merge_heads
            N.call("sdp_merge_heads", ptr(dq), ptr(dk), ptr(dv), b, t, nh, hd, es, st[0], st[1], st[2], ptr(g),
                   stream_ptr(ref.device))
            return g.view(b * t, 3 * nh * hd), None, None, None, None
        for i, x in enumerate((dq, dk, dv)):
            dst = g[:, :, i].transpose(1, 2)  # [b, nh, t, hd] view
            if x is None:
                dst.zero_()
            else:
                dst.copy_(x)
        return g.view(b * t, 3 * nh * hd), None, None, None, None


_CS_PARTS: list = []


def _col_sum_parts() -> int:
    if not _CS_PARTS:
        _CS_PARTS.append(N.lib().sdp_col_sum_parts())
    return _CS_PARTS[0]


class _Linear(torch.autograd.Function):
    """addmm(bias, x, w) (HF Conv1D: w is [in, out]) whose backward takes the
    bias gradient with libsdp's column sum (ones @ dy on cuBLAS otherwise)
    instead of dy.sum(0): torch's reduce kernel ran 19 us per [8192, <=3072]
    bf16 gradient, 4 per block."""

    @staticmethod
    def forward(ctx, bias, x, w):
        ctx.save_for_backward(x, w)
        return torch.addmm(bias, x, w)

    @staticmethod
    def backward(ctx, dy):
        x, w = ctx.saved_tensors
        dx = dy @ w.t() if ctx.needs_input_grad[1] else None
        dw = x.t() @ dy if ctx.needs_input_grad[2] else None
        db = None
        if ctx.needs_input_grad[0]:
            n = dy.shape[1]
            if dy.dtype == torch.bfloat16 and dy.is_cuda and n % 8 == 0 and dy.is_contiguous() \
                    and dy.data_ptr() % 16 == 0:  # libsdp column sum (deterministic two-stage)
                db = torch.empty(n, dtype=dy.dtype, device=dy.device)
                scratch = torch.empty(n * _col_sum_parts(), dtype=torch.float32, device=dy.device)
                N.call("sdp_col_sum_bf16", ptr(dy), dy.shape[0], n, ptr(db), ptr(scratch), stream_ptr(dy.device))
            else:
                ones = torch.ones((1, dy.shape[0]), dtype=dy.dtype, device=dy.device)
                db = (ones @ dy).view(-1)
        return db, dx, dw


def _addmm(bias, x, w):
    if x.dtype == torch.bfloat16 and w.dtype == torch.bfloat16 and bias.dtype == torch.bfloat16:
        return _Linear.apply(bias, x, w)
    return torch.addmm(bias, x, w)


class GPT2Small:
    """BASELINE configs[3] (C4): GPT-2 small over zoo.gpt2_small_topology's flat
    layout -- pre-LN blocks, HF Conv1D weights ([in, out]), causal flash SDPA,
    tanh-GELU, tied LM head.  Block dropping skips whole blocks (the residual
    stream passes through), exactly like models.py:161-163 does for CNN blocks."""

    def __init__(self, vocab=50257, n_ctx=1024, d_model=768, n_layer=12, n_head=12):
        self.vocab, self.n_ctx, self.d_model, self.n_layer, self.n_head = vocab, n_ctx, d_model, n_layer, n_head
        self.topology = zoo.gpt2_small_topology(vocab, n_ctx, d_model, n_layer, n_ctx)

    def build_topology(self):
        return self.topology

    def forward(self, params, tokens, worker=None, block_mode: str = "skip"):
        b, t = tokens.shape
        e, nh = self.d_model, self.n_head
        h = F.embedding(tokens, params["wte"]) + params["wpe"][:t][None]
        pend = None  # (r, m): the residual stream is r + m, not yet added
        for i in range(self.n_layer):
            live = True if worker is None else bool(worker.block_active[i])
            if not live and block_mode == "skip":
                continue
            p = f"h{i}"
            if pend is None:
                a = _layer_norm(h, (e,), params[f"{p}.ln_1.w"], params[f"{p}.ln_1.b"])
            else:  # the previous block's residual add fused into this LayerNorm
                h, a = _add_layer_norm(pend[0], pend[1], (e,), params[f"{p}.ln_1.w"], params[f"{p}.ln_1.b"])
                pend = None
            qkv = _addmm(params[f"{p}.attn.c_attn.b"], a.reshape(b * t, e), params[f"{p}.attn.c_attn.w"])
            q, k, v = _SplitHeads.apply(qkv, b, t, nh, e // nh)
            y = F.scaled_dot_product_attention(q, k, v, is_causal=True)
            y = y.transpose(1, 2).reshape(b * t, e)
            y = _addmm(params[f"{p}.attn.c_proj.b"], y, params[f"{p}.attn.c_proj.w"]).view(b, t, e)
            r, m = _add_layer_norm(h, y, (e,), params[f"{p}.ln_2.w"], params[f"{p}.ln_2.b"])
            m = F.gelu(_addmm(params[f"{p}.mlp.c_fc.b"], m.reshape(b * t, e), params[f"{p}.mlp.c_fc.w"]),
                       approximate="tanh")
            m = _addmm(params[f"{p}.mlp.c_proj.b"], m, params[f"{p}.mlp.c_proj.w"]).view(b, t, e)
            if live:
                pend = (r, m)  # h = (h + attn) + mlp, added by the next LayerNorm
            else:  # block_mode "multiply": the dropped block's output scaled by 0
                h = h + (y + m) * 0.0
        if pend is None:
            h = _layer_norm(h, (e,), params["ln_f.w"], params["ln_f.b"])
        else:
            _, h = _add_layer_norm(pend[0], pend[1], (e,), params["ln_f.w"], params["ln_f.b"])
        # tied head, logits h @ wte.T left to lm_loss; "__wte_padded": the
        # head weight padded for the GEMMs, built once per step by the trainer
        return LMHead(h, params["wte"], params.get("__wte_padded"))


@dataclass
class LMHead:
    """Final hidden states [B, T, E] and the tied embedding [V, E].  The
    [B, T, V] logits are never materialised whole: lm_loss fuses the head GEMM
    with the cross-entropy chunk by chunk (logits() builds them for callers
    that want them)."""
    h: torch.Tensor
    wte: torch.Tensor
    padded: torch.Tensor | None = None  # wte padded to the head GEMM's vocabulary (no grad)

    def logits(self) -> torch.Tensor:
        return self.h @ self.wte.t()


class _LinearCrossEntropy(torch.autograd.Function):
    """mean_i CE(h_i @ w.T, t_i) without the [n, V] logits in memory: the
    forward keeps only each row's log-sum-exp, the backward recomputes a chunk
    of logits at a time and feeds the two gradient GEMMs.  Under autocast
    (bf16) the GEMMs write bf16 logit chunks and libsdp's k_ce_fwd / k_ce_bwd
    make one fp32-accumulating pass over each (log-sum-exp; softmax - onehot,
    scaled); other dtypes use torch ops in at least fp32."""

    CHUNK = 2048

    @staticmethod
    def _cdt(h):
        return torch.get_autocast_dtype("cuda") if torch.is_autocast_enabled("cuda") else h.dtype

    PAD = 64  # head GEMMs on a 64-aligned vocabulary (50257 -> 50304)

    @staticmethod
    def _padded(w, cdt):
        """The tied head weight in the GEMM dtype with its rows padded to a
        multiple of PAD (zero rows): an aligned leading dimension keeps cuBLAS
        on its tensor-core kernels (odd 50257 fell back to align-1 mma.sync:
        69% of the GPT-2 step)."""
        v = w.shape[0]
        vp = -(-v // _LinearCrossEntropy.PAD) * _LinearCrossEntropy.PAD
        if vp == v:
            return w.to(cdt)
        wp = torch.empty((vp, w.shape[1]), dtype=cdt, device=w.device)
        wp[:v].copy_(w)
        wp[v:].zero_()
        return wp

    @staticmethod
    def forward(ctx, h, w, t, wp=None):
        cdt = _LinearCrossEntropy._cdt(h)
        t = t.contiguous()
        n, v = h.shape[0], w.shape[0]
        acc = torch.float64 if cdt == torch.float64 else torch.float32
        lse = torch.empty(n, dtype=acc, device=h.device)
        rows = torch.empty(n, dtype=acc, device=h.device)
        hc = h.to(cdt)
        fused = cdt == torch.bfloat16
        if fused and wp is not None and wp.dtype == cdt:  # padded once per step by the trainer
            wc = wp
        else:
            wc = _LinearCrossEntropy._padded(w, cdt) if fused else w.to(cdt)
        ctx.wp = wc if fused and wp is not None and wp.dtype == cdt else None
        with torch.autocast("cuda", enabled=False):
            for s in range(0, n, _LinearCrossEntropy.CHUNK):
                e = min(n, s + _LinearCrossEntropy.CHUNK)
                lg = hc[s:e] @ wc.t()
                if fused:  # libsdp k_ce_fwd: one pass over the bf16 chunk (padding ignored)
                    N.call("sdp_ce_rows_fwd", ptr(lg), e - s, v, lg.shape[1], ptr(t[s:e]), ptr(lse[s:e]),
                           ptr(rows[s:e]), stream_ptr(h.device))
                else:
                    lg = lg.to(acc)
                    lse[s:e] = torch.logsumexp(lg, dim=1)
                    rows[s:e] = lse[s:e] - lg.gather(1, t[s:e, None]).squeeze(1)
        ctx.save_for_backward(h, w, t, lse)
        ctx.cdt = cdt
        return rows.sum() / n

    @staticmethod
    def backward(ctx, g):
        h, w, t, lse = ctx.saved_tensors
        cdt = ctx.cdt
        n, v = h.shape[0], w.shape[0]
        acc = lse.dtype
        fused = cdt == torch.bfloat16
        hc = h.to(cdt)
        if ctx.wp is not None:
            wc = ctx.wp
        else:
            wc = _LinearCrossEntropy._padded(w, cdt) if fused else w.to(cdt)
        gh = torch.empty(h.shape, dtype=cdt, device=h.device)
        gw = torch.zeros(wc.shape, dtype=acc, device=w.device)
        g32 = g.detach().to(torch.float32).reshape(1).contiguous()
        with torch.autocast("cuda", enabled=False):
            for s in range(0, n, _LinearCrossEntropy.CHUNK):
                e = min(n, s + _LinearCrossEntropy.CHUNK)
                lg = hc[s:e] @ wc.t()
                if fused:  # libsdp k_ce_bwd: softmax - onehot, scaled; zero in the padding
                    dl = torch.empty_like(lg)
                    N.call("sdp_ce_rows_bwd", ptr(lg), e - s, v, lg.shape[1], ptr(t[s:e]), ptr(lse[s:e]),
                           ptr(g32), C.c_float(1.0 / n), ptr(dl), stream_ptr(h.device))
                else:
                    p = torch.exp(lg.to(acc) - lse[s:e, None])
                    p[torch.arange(e - s, device=h.device), t[s:e]] -= 1.0
                    dl = (p * (g.to(acc) / n)).to(cdt)
                del lg
                gh[s:e] = dl @ wc
                if fused:  # bf16 x bf16 accumulated straight into the fp32 gradient (cuBLAS C = D)
                    torch.addmm(gw, dl.t(), hc[s:e], out_dtype=torch.float32, out=gw)
                else:
                    gw += (dl.t() @ hc[s:e]).to(acc)
        return gh.to(h.dtype), gw[:v].to(w.dtype), None, None


def lm_loss(out, tokens):
    """Next-token cross entropy over the tied LM head (fused, chunked), or over
    given logits [B, T, V]."""
    if isinstance(out, LMHead):
        e = out.h.shape[-1]
        return _LinearCrossEntropy.apply(out.h[:, :-1].reshape(-1, e), out.wte, tokens[:, 1:].reshape(-1),
                                         out.padded)
    acc = torch.promote_types(out.dtype, torch.float32)  # fp32, or fp64 for fp64 logits
    return F.cross_entropy(out[:, :-1].reshape(-1, out.shape[-1]).to(acc), tokens[:, 1:].reshape(-1))


def build_gpt2(dev, seed: int = 1) -> GlobalModel:
    arch = GPT2Small()
    topo = arch.topology
    m = GlobalModel(arch=arch, topology=topo, theta=torch.zeros(topo.total, device=dev))
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    th = torch.zeros(topo.total, device=dev)
    for spec in topo.params:  # GPT-2 init: N(0, 0.02) weights/embeddings, LN gain 1, biases 0
        sl = slice(spec.offset, spec.offset + spec.size)
        if spec.kind in ("linear_w", "embed"):
            th[sl] = torch.randn(spec.size, generator=gen, device=dev) * 0.02
        elif spec.kind == "norm_w":
            th[sl] = 1.0
    m.theta = th
    return m


def param_views(topology, flat: torch.Tensor) -> dict:
    """Per-parameter views of the flat vector.  One split (the parameters tile
    [0, d) in order, topology.py:66-74): its backward is ONE concatenation of
    the parameter gradients, where per-parameter slicing would zero-fill and
    accumulate a [d] gradient once per parameter (62 x 2 x 44 MB per ResNet-18
    worker step)."""
    parts = flat.split([p.size for p in topology.params])
    return {p.name: t.view(p.shape) for p, t in zip(topology.params, parts)}


def downsample(h: torch.Tensor, w: torch.Tensor, stride: int) -> torch.Tensor:
    """1x1 convolution with stride s == subsample then 1x1 stride-1 convolution
    (the strided 1x1 kernel reads only every s-th position).  cuDNN's strided
    1x1 data-gradient falls back to a direct kernel (~0.44 ms per ResNet-18
    layer4 worker step on B200); the stride-1 form runs on the GEMM path."""
    if stride == 1:
        return F.conv2d(h, w)
    return F.conv2d(h[:, :, ::stride, ::stride], w)


def live_params(topology, view) -> list:
    """Parameters a worker's subnetwork uses (block strategy: not in a dropped
    block; masking.py:160-169)."""
    dead = set()
    for b in topology.blocks:
        if b.maskable and not bool(view.block_active[b.index]):
            dead.update(b.param_names)
    return [p.name for p in topology.params if p.name not in dead]


@dataclass
class StepStats:
    loss_mean: float


class _GradStore:
    """bf16 training-step plumbing shared by SubnetTrainer and PeerTrainer:
    gradients into the fp32 replicas (`self.grads[w]`) with fused copies and
    libsdp's conv-weight OIHW cast, and the width-wise compact step."""

    def _grad_slots(self, w: int) -> dict:
        if not hasattr(self, "_slots"):
            self._slots = {}
        if w not in self._slots:
            self._slots[w] = param_views(self.model.topology, self.grads[w])
        return self._slots[w]

    def _compact_step_bf16(self, w: int, x, y, cache: bool, src: torch.Tensor | None = None,
                           cvec: torch.Tensor | None = None, g_out: torch.Tensor | None = None) -> torch.Tensor:
        """Width-wise worker step under bf16 autocast: the compact parameters
        are per-parameter leaves (conv weights made channels-last once, as
        cuDNN's NHWC kernels want them), so the backward returns per-parameter
        gradients instead of one concatenation; they reach the fp32 replica
        through a bf16 compact scratch (one fused copy), one bf16 -> fp32 cast
        of the whole compact vector, one libsdp launch that puts the conv
        weights back in OIHW order, and the sync-space transfer."""
        sub = self.subs[w]
        src = self.theta_bf16 if src is None else src
        if cvec is None:  # else: the step's batched gather already extracted it
            cvec = self.transfers[w].to_compact(src) if self.slayout else sub.gather(src)
        views = sub.views(cvec)
        if getattr(self, "_cg_max", None) is None:
            self._cg_max = N.lib().sdp_conv_grad_max_block()
        # conv weights to channels-last in ONE launch (sdp_conv_weights_to_ohwi)
        # instead of one cuDNN-side conversion per weight
        conv_w = [k for k, v in views.items()
                  if v.dim() == 4 and v.numel() > 0 and v.shape[1] * v.shape[2] * v.shape[3] <= self._cg_max]
        cl = None
        if conv_w:
            cl = torch.empty_like(cvec)
            descs, max_o = self._conv_table(("w", w, tuple(conv_w)), [views[k] for k in conv_w])
            N.call("sdp_conv_weights_to_ohwi", ptr(descs), len(conv_w), max_o, ptr(cvec), ptr(cl),
                   stream_ptr(cvec.device))
        cset_w = set(conv_w)
        params = {}
        for k, v in views.items():
            if k in cset_w:
                o, i, kh, kw = v.shape
                v = cl.as_strided((o, i, kh, kw), (i * kh * kw, 1, kw * i, i), v.storage_offset())
            elif v.dim() == 4 and v.numel() > 0:
                v = v.contiguous(memory_format=torch.channels_last)
            params[k] = v.requires_grad_(True)
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=True, cache_enabled=cache):
            logits = self.model.arch.forward_compact(params, x, sub)
            loss = self.loss_fn(logits, y)
        del logits
        names = [k for k, v in views.items() if v.numel() > 0]
        gs = torch.autograd.grad(loss, [params[k] for k in names], allow_unused=True)
        n = sub.compact_total
        if getattr(self, "_cbuf", None) is None:
            subs = self.subs.values() if isinstance(self.subs, dict) else self.subs
            m = max(max(1, s_.compact_total) for s_ in subs)
            self._cbuf = torch.empty(m, dtype=torch.bfloat16, device=cvec.device)
            self._cbuf32 = torch.empty(m, dtype=torch.float32, device=cvec.device)
            self._cg_max = N.lib().sdp_conv_grad_max_block()
        slots = sub.views(self._cbuf)
        dst, src, conv = [], [], []
        for k, g in zip(names, gs):
            slot = slots[k]
            if g is None:
                slot.zero_()
                continue
            if g.dim() == 4 and not g.is_contiguous() and g.is_contiguous(memory_format=torch.channels_last) \
                    and g.shape[1] * g.shape[2] * g.shape[3] <= self._cg_max:
                o, i, kh, kw = g.shape
                slot = self._cbuf.as_strided((o, i, kh, kw), (i * kh * kw, 1, kw * i, i), slot.storage_offset())
                conv.append(k)
            dst.append(slot)
            src.append(g)
        torch._foreach_copy_(dst, src)
        g32 = self._cbuf32[:max(1, n)] if g_out is None else g_out
        g32.copy_(self._cbuf[:max(1, n)])  # conv slots are OHWI here; rewritten below
        if conv:
            descs, max_o = self._conv_table(("g", w, tuple(conv)), [slots[k] for k in conv])
            N.call("sdp_conv_grads_to_oihw", ptr(descs), len(conv), max_o, ptr(self._cbuf), ptr(g32),
                   stream_ptr(cvec.device))
        if g_out is None:  # else: the step's batched scatter writes every worker's replica
            if self.slayout:
                self.transfers[w].from_compact(g32, self.grads[w])
            else:
                sub.scatter(g32, self.grads[w])
        return loss.detach()

    def _conv_table(self, key, views: list):
        """Device descriptor table (sdp_conv_grad_desc) of conv weights given as
        views of one flat buffer (offset = storage offset), cached by key."""
        if not hasattr(self, "_ctables"):
            self._ctables = {}
        if key not in self._ctables:
            dt = np.dtype([("offset", "<i8"), ("out", "<i4"), ("inp", "<i4"), ("k", "<i4"), ("pad", "<i4")])
            arr = np.zeros(len(views), dtype=dt)
            for j, v in enumerate(views):
                sh = v.shape
                arr[j] = (v.storage_offset(), sh[0], sh[1], sh[2] * sh[3], 0)
            self._ctables[key] = (torch.from_numpy(arr.view(np.uint8).copy()).to(views[0].device),
                                  int(arr["out"].max()))
        return self._ctables[key]

    def _store_grads(self, w: int, names: list, gs) -> None:
        """Parameter gradients -> worker w's fp32 replica.  bf16 gradients go
        through a bf16 [d] scratch with ONE same-dtype multi-tensor copy (the
        channels-last conv-weight gradients into channels-last views of their
        slots), then one bf16 -> fp32 cast per contiguous run of the other
        live parameters and ONE libsdp launch that casts the conv weights back
        to the reference OIHW order (sdp_conv_grads_to_oihw).  A mixed-dtype
        or mixed-layout multi-tensor copy falls back to one strided copy per
        parameter (~5 us each, 62 per ResNet-18 worker)."""
        topo = self.model.topology
        if all(g.dtype == torch.bfloat16 for g in gs):
            if getattr(self, "_gbuf", None) is None:
                self._gbuf = torch.empty(topo.total, dtype=torch.bfloat16, device=self.grads[w].device)
                self._slots16 = param_views(topo, self._gbuf)
                self._spec = {p.name: p for p in topo.params}
                self._cg_max = N.lib().sdp_conv_grad_max_block()
            conv = [k for k, g in zip(names, gs) if self._cl_grad(g)]
            cset = set(conv)
            dst = [self._cl_slot(k) if k in cset else self._slots16[k] for k in names]
            torch._foreach_copy_(dst, list(gs))
            for a, b in self._live_runs(w, [k for k in names if k not in cset]):
                self.grads[w][a:b].copy_(self._gbuf[a:b])
            if conv:
                descs, max_o = self._conv_descs(tuple(conv))
                N.call("sdp_conv_grads_to_oihw", ptr(descs), len(conv), max_o, ptr(self._gbuf), ptr(self.grads[w]),
                       stream_ptr(self.grads[w].device))
            return
        slots = self._grad_slots(w)
        torch._foreach_copy_([slots[k] for k in names], list(gs))

    def _cl_grad(self, g: torch.Tensor) -> bool:
        """A channels-last (not also contiguous) 4-D gradient the OIHW cast
        kernel takes."""
        return (g.dim() == 4 and not g.is_contiguous() and g.is_contiguous(memory_format=torch.channels_last)
                and g.shape[1] * g.shape[2] * g.shape[3] <= self._cg_max)

    def _cl_slot(self, k: str) -> torch.Tensor:
        """Channels-last (OHWI-ordered) view of parameter k's scratch slot."""
        p = self._spec[k]
        o, i, kh, kw = p.shape
        return self._gbuf.as_strided((o, i, kh, kw), (i * kh * kw, 1, kw * i, i), p.offset)

    def _conv_descs(self, conv: tuple):
        if not hasattr(self, "_cdescs"):
            self._cdescs = {}
        if conv not in self._cdescs:
            dt = np.dtype([("offset", "<i8"), ("out", "<i4"), ("inp", "<i4"), ("k", "<i4"), ("pad", "<i4")])
            arr = np.zeros(len(conv), dtype=dt)
            for j, k in enumerate(conv):
                p = self._spec[k]
                arr[j] = (p.offset, p.shape[0], p.shape[1], p.shape[2] * p.shape[3], 0)
            t = torch.from_numpy(arr.view(np.uint8).copy()).to(self._gbuf.device)
            self._cdescs[conv] = (t, int(arr["out"].max()))
        return self._cdescs[conv]

    def _live_runs(self, w: int, names: list) -> list:
        """Element runs [s, e) covered by the live parameters (merged)."""
        if not hasattr(self, "_runs"):
            self._runs = {}
        if w not in self._runs:
            spec = {p.name: p for p in self.model.topology.params}
            runs: list = []
            for k in sorted(names, key=lambda k: spec[k].offset):
                a, b = spec[k].offset, spec[k].offset + spec[k].size
                if runs and runs[-1][1] == a:
                    runs[-1][1] = b
                else:
                    runs.append([a, b])
            self._runs[w] = [tuple(r) for r in runs]
        return self._runs[w]


OPTIMIZERS = ("sgd-nesterov", "adam")


def _check_optimizer(kind: str) -> str:
    if kind not in OPTIMIZERS:
        raise ConfigError(f"unknown optimizer kind {kind!r}")  # optim.py:120
    return kind


def _fused_optimizer(tr, theta, m, v, theta_bf16) -> dict:
    """owner_sync keyword of a trainer's fused optimizer: Nesterov scalars, or
    Adam with the trainer's device step counter and bias-correction table."""
    if tr.optimizer == "sgd-nesterov":
        return {"nesterov": {"theta": theta, "velocity": m, "lr": tr.lr, "momentum": tr.momentum,
                             "theta_bf16": theta_bf16}}
    if getattr(tr, "_bias_table", None) is None:
        tr._bias_table = engine.adam_bias_table(tr.betas[0], tr.betas[1], tr.adam_step.device)
    return {"adam": {"theta": theta, "m": m, "v": v, "lr": tr.lr, "beta1": tr.betas[0], "beta2": tr.betas[1],
                     "eps": tr.eps, "theta_bf16": theta_bf16, "step": tr.adam_step,
                     "bias_table": tr._bias_table}}


class SubnetTrainer(_GradStore):
    """N logical workers co-resident on one GPU (the reference's in-process
    structure, engine.py:180-245) with the owner-subset sync fused into the
    optimizer step.

    theta / velocity: canonical fp32 master state (engine.py:223 updates one
    shared theta); theta_bf16: the training copy every worker's forward reads,
    written by the sync kernel's epilogue."""

    def __init__(self, model: GlobalModel, assignment, lr: float = 0.1, momentum: float = 0.9,
                 autocast: bool = True, compact: bool | None = None, loss_fn=None,
                 sync_layout: bool = False, graphed: bool = False, optimizer: str = "sgd-nesterov",
                 betas: tuple = (0.9, 0.999), eps: float = 1e-8):
        """optimizer: the reference's kinds (optim.py:115-120), fused into the
        sync launch -- "sgd-nesterov" (momentum) or "adam" (betas, eps; the
        step count lives on the device with a table of the reference's bias
        corrections, so graph replays advance it).

        graphed: capture the whole protocol step (N worker fwd/bwd, gather /
        scatter, the fused sync) in one CUDA graph and replay it -- the eager
        step is host-bound (thousands of small launches), see step()."""
        self.model = model
        self.graphed = graphed
        self._graph = None
        self.assignment = assignment
        self.loss_fn = loss_fn or (lambda logits, y: F.cross_entropy(logits.float(), y))
        self.views = [assignment.worker_view(w) for w in range(assignment.n_workers)]
        # width-wise (neuron) workers run their compact subnetwork: gather ->
        # dense compact fwd/bwd -> scatter into the worker's flat gradient
        self.compact = assignment.strategy == "neuron" if compact is None else compact
        if self.compact:
            from .models import SubnetLayout
            self.subs = [SubnetLayout(assignment, w) for w in range(assignment.n_workers)]
        d = model.topology.total
        dev = model.theta.device
        # sync_layout: keep theta / velocity / gradient replicas permuted into the
        # window-class-major layout (layout.py) so the sync sees uniform tiles
        self.slayout = None
        # master: the fp32 theta the fused update writes.  In the reference
        # layout it IS model.theta (same storage); in the sync layout it is a
        # private permuted copy and model.theta is left in the reference
        # layout (write_back() refreshes it, theta() returns it permuted back),
        # so checkpoint.save_checkpoint(model, ...) never sees a permuted vector.
        self.master = model.theta
        if sync_layout and self.compact:
            from .layout import SyncLayout, WorkerTransfer
            self.slayout = SyncLayout(assignment)
            self.transfers = [WorkerTransfer(self.slayout, s) for s in self.subs]
            self.master = self.slayout.to_sync(model.theta)
        self.velocity = torch.zeros(d, device=dev)  # Nesterov v / Adam m
        self.optimizer = _check_optimizer(optimizer)
        self.betas, self.eps = (float(betas[0]), float(betas[1])), float(eps)
        self.second = torch.zeros(d, device=dev) if optimizer == "adam" else None  # Adam v
        self.adam_step = torch.zeros(1, dtype=torch.int32, device=dev)  # steps taken (device)
        self.theta_bf16 = self.master.to(torch.bfloat16)
        self.grads = [torch.zeros(d, device=dev) for _ in range(assignment.n_workers)]
        self.lr, self.momentum, self.autocast = lr, momentum, autocast
        self.plan = self.slayout.plan() if self.slayout else assignment.sync_plan()
        # status word of the fused sync (SDP_SYNC_CHECK_FINITE): read by check()
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self._prep = None

    def _live_params(self, w: int) -> list:
        if not hasattr(self, "_live"):
            self._live = {}
        if w not in self._live:
            self._live[w] = live_params(self.model.topology, self.views[w])
        return self._live[w]

    def theta(self) -> torch.Tensor:
        """theta in the reference's flat layout."""
        return self.slayout.from_sync(self.master) if self.slayout else self.master

    def write_back(self) -> None:
        """Refresh model.theta (reference layout) from the trainer's master."""
        if self.slayout is not None:
            self.model.theta.copy_(self.slayout.from_sync(self.master))

    def check(self) -> None:
        """Raise NumericalError if any step since the last check produced a
        non-finite mean (the reference raises before updating, optim.py:78-80;
        the fused sync+update cannot roll back, so theta already holds the
        non-finite step when this fires -- call it at every loss read)."""
        st = int(self.status.item())
        if st & N.STATUS_NONFINITE:
            self.status.zero_()
            raise NumericalError("training aborted: the aggregated gradient contains non-finite values")

    def _sync(self):
        if self._prep is None:
            opt = _fused_optimizer(self, self.master, self.velocity, self.second, self.theta_bf16)
            self._prep = engine.PreparedSync(
                self.grads, self.assignment, writeback=False, plan=self.plan, check_finite=True,
                status=self.status, **opt)
        self._prep.args.lr = float(self.lr)
        if self.optimizer == "adam":
            self.adam_step.add_(1)  # optim.py:104: t += 1 before the update
        self._prep.launch()

    def step(self, batches) -> torch.Tensor:
        """batches: list of N (x, y) device tensors; returns the mean loss (device).

        graphed: the first call (and any call after `lr` changed) captures the
        step into a CUDA graph -- after warm-up steps on a side stream whose
        effect on theta / velocity is rolled back -- and every call copies the
        batches into the graph's static inputs and replays it.  Same math, same
        kernels, same order as the eager step."""
        if not self.graphed:
            return self._step_eager(batches)
        if self._graph is None or self._graph_lr != self.lr:
            self._capture(batches)
        for (sx, sy), (x, y) in zip(self._static, batches):
            if sx.data_ptr() != x.data_ptr():
                sx.copy_(x)
            if sy.data_ptr() != y.data_ptr():
                sy.copy_(y)
        self._graph.replay()
        return self._static_loss

    def _capture(self, batches, warmup: int = 2) -> None:
        self._static = [(x.clone(), y.clone()) for x, y in batches]
        state = [self.master, self.velocity, self.theta_bf16, self.adam_step] + \
            ([self.second] if self.second is not None else [])
        saved = [t.clone() for t in state]
        side = torch.cuda.Stream(self.master.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # autograd / cuDNN warm-up outside the capture
            for _ in range(warmup):
                self._step_eager(self._static, cache=False)
        torch.cuda.current_stream().wait_stream(side)
        for t, v in zip(state, saved):  # the warm-up steps never happened
            t.copy_(v)
        del saved
        self._graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self._graph):
            self._static_loss = self._step_eager(self._static, cache=False)
        self._graph_lr = self.lr

    def _step_params(self) -> dict:
        """Leaf parameters of one step's block-strategy workers: views of the
        bf16 copy, with the 4-D convolution weights made channels-last ONCE
        per step (cuDNN's NHWC kernels would otherwise convert every weight
        for every worker).  The leaves are shared by the N workers;
        torch.autograd.grad returns each worker's gradients separately."""
        topo = self.model.topology
        src = (self.theta_bf16 if self.autocast else self.master).detach()
        out = {}
        views = param_views(topo, src)
        conv_w = []
        if self.autocast and src.is_cuda and src.dtype == torch.bfloat16:
            if getattr(self, "_cg_max", None) is None:
                self._cg_max = N.lib().sdp_conv_grad_max_block()
            conv_w = [k for k, v in views.items()
                      if v.dim() == 4 and v.numel() > 0 and v.shape[1] * v.shape[2] * v.shape[3] <= self._cg_max]
        cl = None
        if conv_w:  # every conv weight to channels-last in one launch
            cl = torch.empty_like(src)
            descs, max_o = self._conv_table(("step",), [views[k] for k in conv_w])
            N.call("sdp_conv_weights_to_ohwi", ptr(descs), len(conv_w), max_o, ptr(src), ptr(cl),
                   stream_ptr(src.device))
        cset = set(conv_w)
        for k, v in views.items():
            if k in cset:
                o, i, kh, kw = v.shape
                v = cl.as_strided((o, i, kh, kw), (i * kh * kw, 1, kw * i, i), v.storage_offset())
            elif self.autocast and v.dim() == 4 and v.is_cuda:
                v = v.contiguous(memory_format=torch.channels_last)
            out[k] = v.requires_grad_(True)
        if self.autocast and isinstance(self.model.arch, GPT2Small):  # the tied head, padded once for all workers
            out["__wte_padded"] = _LinearCrossEntropy._padded(views["wte"], torch.bfloat16)
        return out

    def _batches(self):
        """The step's two slice launches over ALL workers (models.SliceBatch):
        extraction of every worker's compact parameters before the first
        forward, write-back of every compact gradient after the last backward."""
        if getattr(self, "_xfer", None) is None:
            from .models import SliceBatch
            dev = self.master.device
            if self.slayout:
                parts = [t.host for t in self.transfers]
                self._xfer = (SliceBatch(parts, dev), SliceBatch(parts, dev))
            else:
                self._xfer = (SliceBatch([s_.host_gather for s_ in self.subs], dev),
                              SliceBatch([s_.host_scatter for s_ in self.subs], dev))
        return self._xfer

    def _extract_all(self, src: torch.Tensor) -> list:
        """Every worker's compact parameters from `src` in ONE launch."""
        gather_b, _ = self._batches()
        outs = [torch.empty(max(1, s_.compact_total), dtype=src.dtype, device=src.device) for s_ in self.subs]
        if self.slayout:  # transfer tables: "full" = the compact tensor, "compact" = the sync block
            gather_b.gather(outs, [src] * len(outs), reverse=True)
        else:
            gather_b.gather([src] * len(outs), outs)
        return outs

    def _write_back_all(self, gs: list) -> None:
        """Every worker's compact gradient into its fp32 replica in ONE launch."""
        _, scatter_b = self._batches()
        if self.slayout:
            scatter_b.gather(gs, self.grads)
        else:
            scatter_b.scatter(gs, self.grads)

    def _step_eager(self, batches, cache: bool = True) -> torch.Tensor:
        topo = self.model.topology
        step_params = None
        losses = []
        if self.compact:
            # the workers train on the bf16 copy the previous sync wrote
            src = self.theta_bf16 if self.autocast else self.master
            cvecs = self._extract_all(src)
            g32s = [torch.empty(max(1, s_.compact_total), dtype=torch.float32, device=src.device)
                    for s_ in self.subs]
        for w, (x, y) in enumerate(batches):
            if self.compact and self.autocast:
                losses.append(self._compact_step_bf16(w, x, y, cache, cvec=cvecs[w], g_out=g32s[w]))
                continue
            if self.compact:
                sub = self.subs[w]
                leaf = cvecs[w][:sub.compact_total].requires_grad_(True)
                with torch.autocast("cuda", dtype=torch.bfloat16, enabled=self.autocast, cache_enabled=cache):
                    logits = self.model.arch.forward_compact(sub.views(leaf), x, sub)
                    loss = self.loss_fn(logits, y)
                del logits
                (g,) = torch.autograd.grad(loss, leaf)
                g32s[w][:sub.compact_total].copy_(g)  # fp32 gradient replica (the sync accumulates in fp32)
                losses.append(loss.detach())
                continue
            # the worker trains on the bf16 weights the previous sync wrote;
            # every parameter is a leaf view and its gradient lands directly
            # in its slot of the fp32 replica (one multi-tensor copy, no [d]
            # concatenation); parameters of dropped blocks keep their zeros
            if step_params is None:  # once per step: every worker reads the same bf16 copy
                step_params = self._step_params()
            params = step_params
            with torch.autocast("cuda", dtype=torch.bfloat16, enabled=self.autocast, cache_enabled=cache):
                logits = self.model.arch.forward(params, x, self.views[w])
                loss = self.loss_fn(logits, y)
            del logits
            names = self._live_params(w)
            gs = torch.autograd.grad(loss, [params[k] for k in names])
            self._store_grads(w, names, gs)
            losses.append(loss.detach())
        if self.compact:
            self._write_back_all(g32s)
        self._sync()
        return torch.stack(losses).mean()

class PeerTrainer(_GradStore):
    """One process per GPU (torchrun): this rank trains its local workers
    (contiguous placement, comm.rank_layout) on their own parameter copies.
    A step is: every local worker's forward/backward writes its fp32 gradient
    into its peer-mapped replica; ONE owner-sync launch per rank (the leader
    of each tile reads every owner's gradient -- local or over NVLink -- in
    ascending worker order and writes the mean into every owner's replica)
    whose last phase applies SGD-Nesterov + the bf16 cast to every local
    worker's own copy (SDP_SYNC_LOCAL_UPDATE; without owned-tile storage, a
    separate sdp_nesterov_update per worker).  Remote traffic is 4 B per
    remote owner per element; updating remote theta / velocity copies from
    the leader instead would cost 10 B.  Every owner applies the same update
    to the same mean, so the owners' copies of an owned parameter stay
    bit-identical to the co-resident trainer's canonical theta
    (engine.py:222-223).

    Width-wise (neuron) assignments keep replicas and parameter copies in the
    window-class-major sync layout (layout.SyncLayout) and train compact
    subnetworks through layout.WorkerTransfer, like SubnetTrainer; on
    owned-tile storage the transfers address the worker's blocks through the
    slot table."""

    def __init__(self, model: GlobalModel, assignment, rank: int, world: int, device, all_gather,
                 lr: float = 0.1, momentum: float = 0.9, autocast: bool = True, loss_fn=None,
                 timeout_cycles: int = 20_000_000_000, graphed: bool = False,
                 compact_storage: bool | None = None, optimizer: str = "sgd-nesterov",
                 betas: tuple = (0.9, 0.999), eps: float = 1e-8):
        """graphed: capture the rank's whole step (local workers' fwd/bwd, the
        peer-mapped sync, the Nesterov updates) in one CUDA graph, as
        SubnetTrainer does.  The sync kernel keeps its cross-rank barrier
        epochs on the device (comm.PeerGroup.epochs), so replays stay in step
        as long as every rank calls step() the same number of times.

        compact_storage (default: on): each local worker keeps theta,
        velocity, the bf16 copy and its gradient replica ONLY for the tiles it
        owns (storage.CompactLayout; dropped blocks / unowned sync blocks have
        no storage), and the step's optimizer runs inside the sync launch as
        its local-update phase (SDP_SYNC_LOCAL_UPDATE): one libsdp launch per
        rank per step for sync + Nesterov + bf16 cast."""
        from . import comm
        self.model, self.assignment = model, assignment
        self.lr, self.momentum, self.autocast = lr, momentum, autocast
        self.graphed = graphed
        self._graph = None
        self.loss_fn = loss_fn or (lambda logits, y: F.cross_entropy(logits.float(), y))
        self.device = torch.device(device)
        self.compact = assignment.strategy == "neuron"
        if compact_storage is None:
            compact_storage = True
        self.compact_storage = bool(compact_storage)
        self.optimizer = _check_optimizer(optimizer)
        self.betas, self.eps = (float(betas[0]), float(betas[1])), float(eps)
        if optimizer == "adam" and not self.compact_storage:
            raise UsageError("the fused Adam update runs in the sync's local-update phase: "
                             "use compact_storage=True")
        self.slayout = None
        theta0 = model.theta.to(self.device)
        if self.compact:
            from .layout import SyncLayout, WorkerTransfer
            from .models import SubnetLayout
            self.slayout = SyncLayout(assignment)
            theta0 = self.slayout.to_sync(theta0)
        self.group = comm.PeerGroup(assignment, rank, world, self.device, all_gather, shadows=False,
                                    timeout_cycles=timeout_cycles,
                                    owner_mask=None if self.slayout is None else self.slayout.owner_mask,
                                    compact=self.compact_storage)
        self.local = self.group.layout.local_workers
        self.views = {w: assignment.worker_view(w) for w in self.local}
        if self.compact:
            self.subs = {w: SubnetLayout(assignment, w) for w in self.local}
            # compact storage: the sync-space buffers hold only the worker's
            # owned tiles and the transfers address them through the slot table
            cl = self.group.compact if self.compact_storage else None
            self.transfers = {w: WorkerTransfer(self.slayout, self.subs[w], compact=cl) for w in self.local}
        if self.compact_storage:
            lay = self.group.compact
            self.theta = {w: lay.gather(w, theta0) for w in self.local}
        else:
            self.theta = {w: theta0.clone() for w in self.local}
        del theta0
        self.velocity = {w: torch.zeros_like(self.theta[w]) for w in self.local}  # Nesterov v / Adam m
        self.second = ({w: torch.zeros_like(self.theta[w]) for w in self.local}
                       if optimizer == "adam" else None)  # Adam v
        self.adam_step = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.theta_bf16 = {w: self.theta[w].to(torch.bfloat16) for w in self.local}
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)
        # the gradient replicas are the peer-mapped ones; parameters of a
        # worker's dropped blocks are never written (the replica keeps zeros
        # there: the sync only writes owned elements)
        self.grads = self.group.replicas
        if not self.compact:
            self._live = {w: live_params(model.topology, self.views[w]) for w in self.local}
        if self.compact_storage:
            from .storage import worker_states
            topo = model.topology
            if not self.compact:
                self._specs = {w: [topo.index[k] for k in self._live[w]] for w in self.local}
            self._states = worker_states([(self.theta[w], self.velocity[w],
                                           None if self.second is None else self.second[w],
                                           self.theta_bf16[w], self.grads[w]) for w in self.local], self.device)
            self._updates, per_cta = lay.update_table(self.local, self.group.plan.leader_cta(), self.group.grid)
            a = self.group.args
            if optimizer == "adam":
                self._bias_table = engine.adam_bias_table(self.betas[0], self.betas[1], self.device)
                a.flags |= N.SYNC_ADAM | N.SYNC_LOCAL_UPDATE | N.SYNC_CHECK_FINITE
                a.beta1, a.beta2 = self.betas
                a.one_minus_beta1, a.one_minus_beta2 = 1 - self.betas[0], 1 - self.betas[1]
                a.eps = self.eps
                a.adam_step = self.adam_step.data_ptr()
                a.adam_bias_table = self._bias_table.data_ptr()
                a.adam_table_len = self._bias_table.numel() // 2
            else:
                a.flags |= N.SYNC_NESTEROV | N.SYNC_LOCAL_UPDATE | N.SYNC_CHECK_FINITE
            a.momentum = float(momentum)
            a.updates = self._updates.data_ptr()
            a.updates_per_cta = per_cta
            a.states = self._states.data_ptr()

    def step(self, batches: dict) -> torch.Tensor:
        """batches: {local worker: (x, y)}; returns the local workers' mean loss."""
        if not self.graphed:
            return self._step_eager(batches)
        if self._graph is None or self._graph_lr != self.lr:
            self._capture(batches)
        for w, (x, y) in batches.items():
            sx, sy = self._static[w]
            if sx.data_ptr() != x.data_ptr():
                sx.copy_(x)
            if sy.data_ptr() != y.data_ptr():
                sy.copy_(y)
        self._graph.replay()
        return self._static_loss

    def _capture(self, batches, warmup: int = 2) -> None:
        """Warm-up steps on a side stream (they run the collective sync, so
        every rank does the same number), rolled back, then one captured step."""
        self._static = {w: (x.clone(), y.clone()) for w, (x, y) in batches.items()}
        state = [t for w in self.local for t in (self.theta[w], self.velocity[w], self.theta_bf16[w])]
        state += [self.adam_step] + ([self.second[w] for w in self.local] if self.second is not None else [])
        saved = [t.clone() for t in state]
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            for _ in range(warmup):
                self._step_eager(self._static, cache=False)
        torch.cuda.current_stream(self.device).wait_stream(side)
        for t, v in zip(state, saved):
            t.copy_(v)
        del saved
        self._graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self._graph):
            self._static_loss = self._step_eager(self._static, cache=False)
        self._graph_lr = self.lr

    def _step_compact_storage(self, batches: dict, cache: bool) -> torch.Tensor:
        """Workers on owned-tile storage.  Block workers: the live parameters
        are views of the worker's compact bf16 copy (one contiguous range
        each) and their gradients go straight into the worker's compact fp32
        replica.  Width-wise workers: their compact subnetwork is extracted
        from / written back into the owned-tile buffers by the slot-mapped
        sync-layout transfers.  Then ONE sync launch per rank averages,
        applies Nesterov to every local owner's compact theta / velocity and
        writes its bf16 copy."""
        lay = self.group.compact
        losses = []
        for w in self.local:
            x, y = batches[w]
            if self.compact:
                losses.append(self._widthwise_step(w, x, y, cache))
                continue
            src = (self.theta_bf16[w] if self.autocast else self.theta[w]).detach()
            params = {}
            for k, v in lay.views(w, src, self._specs[w]).items():
                if self.autocast and v.dim() == 4:  # channels-last conv weights (cuDNN NHWC)
                    v = v.contiguous(memory_format=torch.channels_last)
                params[k] = v.requires_grad_(True)
            if self.autocast and isinstance(self.model.arch, GPT2Small):
                params["__wte_padded"] = _LinearCrossEntropy._padded(params["wte"].detach(), torch.bfloat16)
            with torch.autocast("cuda", dtype=torch.bfloat16, enabled=self.autocast, cache_enabled=cache):
                loss = self.loss_fn(self.model.arch.forward(params, x, self.views[w]), y)
            names = self._live[w]
            gs = torch.autograd.grad(loss, [params[k] for k in names])
            slots = lay.views(w, self.grads[w], self._specs[w])
            torch._foreach_copy_([slots[k] for k in names], list(gs))
            losses.append(loss.detach())
        self.group.args.lr = float(self.lr)
        if self.optimizer == "adam":
            self.adam_step.add_(1)  # optim.py:104: t += 1 before the update
        self.group.launch()  # sync + local Nesterov / Adam + bf16 cast, one launch
        return torch.stack(losses).mean()

    def check(self) -> None:
        """Raise on a cross-rank barrier timeout or a non-finite mean (the
        fused update cannot roll back: call it at every loss read)."""
        self.group.check()
        st = int(self.group.status.item()) | int(self.status.item())
        if st & N.STATUS_NONFINITE:
            self.group.status.zero_()
            self.status.zero_()
            raise NumericalError("training aborted: the aggregated gradient contains non-finite values")

    def state_bytes(self) -> int:
        """Bytes of this rank's per-worker training state (theta, moments,
        bf16 copy, gradient replica)."""
        extra = list(self.second.values()) if self.second is not None else []
        return sum(t.numel() * t.element_size() for w in self.local
                   for t in (self.theta[w], self.velocity[w], self.theta_bf16[w], self.grads[w])) + \
            sum(t.numel() * t.element_size() for t in extra)

    def _widthwise_step(self, w: int, x, y, cache: bool) -> torch.Tensor:
        """One width-wise worker's fwd/bwd: compact subnetwork out of the
        worker's sync-space copy, its gradient into the worker's replica."""
        if self.autocast:
            return self._compact_step_bf16(w, x, y, cache, src=self.theta_bf16[w])
        sub = self.subs[w]
        leaf = self.transfers[w].to_compact(self.theta[w]).requires_grad_(True)
        loss = self.loss_fn(self.model.arch.forward_compact(sub.views(leaf), x, sub), y)
        (g,) = torch.autograd.grad(loss, leaf)
        self.transfers[w].from_compact(g.float(), self.group.replicas[w])
        return loss.detach()

    def _step_eager(self, batches: dict, cache: bool = True) -> torch.Tensor:
        if self.compact_storage:
            return self._step_compact_storage(batches, cache)
        topo = self.model.topology
        losses = []
        for w in self.local:
            x, y = batches[w]
            if self.compact:
                losses.append(self._widthwise_step(w, x, y, cache))
                continue
            src = (self.theta_bf16[w] if self.autocast else self.theta[w]).detach()
            params = {}
            for k, v in param_views(topo, src).items():
                if self.autocast and v.dim() == 4:  # channels-last conv weights (cuDNN NHWC)
                    v = v.contiguous(memory_format=torch.channels_last)
                params[k] = v.requires_grad_(True)
            with torch.autocast("cuda", dtype=torch.bfloat16, enabled=self.autocast, cache_enabled=cache):
                loss = self.loss_fn(self.model.arch.forward(params, x, self.views[w]), y)
            names = self._live[w]
            gs = torch.autograd.grad(loss, [params[k] for k in names])
            self._store_grads(w, names, gs)
            losses.append(loss.detach())
        self.group.launch()  # peer-mapped owner sync: replicas[w] <- mean on w's elements
        for w in self.local:  # width-wise: replicas in the sync layout, update per worker
            N.call("sdp_nesterov_update", N.DTYPE_F32, self.theta[w].numel(), ptr(self.theta[w]),
                   ptr(self.velocity[w]), ptr(self.group.replicas[w]), float(self.lr), float(self.momentum),
                   ptr(self.theta_bf16[w]), ptr(self.status), stream_ptr(self.device))
        return torch.stack(losses).mean()

    def theta_of(self, w: int) -> torch.Tensor:
        """Worker w's parameter copy in the reference's flat layout (compact
        storage: elements of tiles w does not store read 0)."""
        flat = self.theta[w]
        if self.compact_storage:
            d = self.model.topology.total
            flat = self.group.compact.scatter(w, self.theta[w], torch.zeros(d, device=self.device))
        return self.slayout.from_sync(flat) if self.slayout else flat

    def close(self) -> None:
        self.group.close()


def build_resnet18(dev, seed: int = 1) -> GlobalModel:
    arch = ResNet18Cifar()
    topo = arch.topology
    theta = torch.zeros(topo.total, device=dev)
    m = GlobalModel(arch=arch, topology=topo, theta=theta)
    from .models import kaiming_fan_out_init
    m.theta = kaiming_fan_out_init(m, None, seed)
    fc = topo.index["fc.w"]
    m.theta[fc.offset:fc.offset + fc.size] = 0.0  # zero-init classifier: initial loss ln(10)
    return m


def worker_memory(model: GlobalModel, assignment, worker: int | None, batch: int,
                  dev, make_batch=None, loss_fn=None, return_grad: bool = False) -> dict:
    """Peak device memory of ONE worker's training state and step, as a GPU
    holding one worker would see it (paper: params, grads, optimizer state and
    activations all scale with the subnetwork).  worker=None: the full model
    (a full-replica DP worker).  Parameters/grad/momentum are allocated for
    the worker's active elements only (compact storage), the forward/backward
    runs on the subnetwork."""
    from .models import SubnetLayout
    topo = model.topology
    if worker is None:  # full replica = the P = N assignment's worker 0
        assignment = masking.build_assignment(topo, "block", 1, 1, seed=0)
        worker = 0
    sub = SubnetLayout(assignment, worker)
    view = assignment.worker_view(worker)
    if make_batch is None:
        x = torch.randn(batch, 3, 32, 32, device=dev)
        y = torch.randint(0, 10, (batch,), device=dev)
    else:
        x, y = make_batch()
    loss_fn = loss_fn or (lambda logits, yy: F.cross_entropy(logits.float(), yy))
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()
    base = torch.cuda.memory_allocated(dev)
    torch.cuda.reset_peak_memory_stats(dev)
    # compact fp32 master + fp32 gradient (what the sync reads) + momentum + bf16
    # training copy.  The step mirrors SubnetTrainer's: every worker runs on
    # the bf16 copy under autocast (no weight-cast cache, as in the graphed
    # step).  Every
    # parameter is a leaf view whose gradient is written into its slot of the
    # fp32 flat gradient the moment autograd finishes it and then freed
    # (post-accumulate hook): no second gradient-sized buffer and no
    # all-parameter gradient set alive at once.
    master = sub.gather(model.theta)
    grad = torch.zeros_like(master)
    momentum = torch.zeros_like(master)
    shadow = master.to(torch.bfloat16)
    gviews = sub.views(grad)
    weights = sub.views(shadow)
    leaves = {}
    for name, v in weights.items():
        if v.numel() == 0:
            leaves[name] = v
            continue
        t = v.detach().requires_grad_(True)

        def _to_flat(param, slot=gviews[name]):
            slot.copy_(param.grad)
            param.grad = None

        t.register_post_accumulate_grad_hook(_to_flat)
        leaves[name] = t
    with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
        if assignment.strategy == "neuron":
            logits = model.arch.forward_compact(leaves, x, sub)
        else:
            logits = model.arch.forward(leaves, x, view)
        loss = loss_fn(logits, y)
    del logits
    loss.backward()
    torch.cuda.synchronize(dev)
    peak = torch.cuda.max_memory_allocated(dev) - base
    active = sub.compact_total
    out = {"active_params": int(active), "peak_bytes": int(peak), "state_bytes": int(active * (4 * 3 + 2))}
    if return_grad:
        out["grad"] = grad
    del master, grad, momentum, shadow, loss, leaves
    return out


def build_block_assignment(topo, n=8, p=4, seed=1):
    return masking.build_assignment(topo, "block", n, p, seed)
