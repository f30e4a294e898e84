"""Extraction / write-back behind the reference's model API (models.py:147-382).

    masked_forward(model, worker, xs, ys, block_mode="skip", record=True,
                   layout="full") -> (loss, tape, params)
    flat_gradient(model, tape, loss, params) -> flat [d] gradient

layout="full" is the reference's semantics: the worker's parameters are
theta * mask over the full tensors (models.py:355), extracted by libsdp's
`sdp_masked_extract`; dropped blocks are skipped ("skip") or scaled by zero
("multiply"), inactive channels leave the active-channel GroupNorm as exact
zeros (ops.py:140-204).

layout="compact" runs the worker's structurally smaller subnetwork: the live
rows/columns of every weight are gathered into one contiguous compact buffer
(`sdp_gather_slices`), the forward/backward runs dense cuDNN/cuBLAS on the
compact tensors with ragged per-group GroupNorm statistics, and
flat_gradient scatters the compact gradient back into the flat [d] layout with
zeros elsewhere (`sdp_scatter_slices`).  Both layouts give the same loss and
gradient; the forward/backward math itself is torch (dense
GEMMs, not the optimisation target).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F

from . import _native as N
from ._device import device, ptr, sdp_dtype, slice_dtype, stream_ptr
from .errors import ConfigError, InputError, UsageError
from .topology import GlobalModel, fast_divisor
from . import zoo


# ---------------------------------------------------------------------------
# group norm over active channels (ops.py:140-204)
# ---------------------------------------------------------------------------

def _group_norm_by_membership(x: torch.Tensor, member: torch.Tensor, gamma: torch.Tensor,
                              beta: torch.Tensor, eps: float) -> torch.Tensor:
    """x [B, C, H, W]; member [C, G] 0/1: statistics of group g over its member
    channels only.  Non-member channels produce 0."""
    b, c, h, w = x.shape
    m = member.to(x.dtype)
    count = m.sum(dim=0) * (h * w)                                  # [G]
    s = x.sum(dim=(2, 3)) @ m                                       # [B, G]
    mean = s / count
    xc = x - (mean @ m.t())[:, :, None, None]
    var = (xc * xc).sum(dim=(2, 3)) @ m / count
    inv = 1.0 / torch.sqrt(var + eps)
    xhat = xc * (inv @ m.t())[:, :, None, None]
    live = (m.sum(dim=1) > 0)[None, :, None, None]
    return torch.where(live, xhat * gamma[None, :, None, None] + beta[None, :, None, None],
                       torch.zeros((), dtype=x.dtype, device=x.device))


def active_group_norm(x, groups: int, gamma, beta, active: torch.Tensor, eps: float = 1e-5):
    c = x.shape[1]
    if c % groups:
        raise ConfigError(f"group_norm: {groups} groups do not divide {c} channels")
    gsize = c // groups
    member = F.one_hot(torch.arange(c, device=x.device) // gsize, groups) * active.to(torch.long)[:, None]
    if bool((member.sum(dim=0) == 0).any()):
        raise ConfigError("group_norm: a group has no active channels")
    return _group_norm_by_membership(x, member, gamma, beta, eps)


_STARTS: dict = {}


def _group_starts(starts: tuple[int, ...], dev) -> torch.Tensor:
    key = (starts, dev)
    if key not in _STARTS:
        _STARTS[key] = torch.tensor(starts, dtype=torch.int32, device=dev)
    return _STARTS[key]


class _GroupNormCL(torch.autograd.Function):
    """libsdp k_gn_fwd / k_gn_bwd: GroupNorm (+ReLU) on channels-last bf16
    activations over contiguous, possibly ragged channel groups; fp32
    statistics; dgamma / dbeta in the affine dtype, deterministic (per-CTA
    partial rows + an ordered fold, no atomics)."""

    @staticmethod
    def forward(ctx, x, gamma, beta, starts, eps, relu):
        b, c, h, w = x.shape
        x = x.contiguous(memory_format=torch.channels_last)
        sd = _group_starts(starts, x.device)
        groups = len(starts) - 1
        max_cg = max(starts[k + 1] - starts[k] for k in range(groups))
        if beta.dtype != gamma.dtype:
            beta = beta.to(gamma.dtype)
        gamma, beta = gamma.contiguous(), beta.contiguous()
        # SDP_GN_RELU | SDP_GN_GROUPS_ALIGNED8 | SDP_GN_AFFINE_BF16
        flags = ((1 if relu else 0) | (2 if all(v % 8 == 0 for v in starts) else 0)
                 | (4 if gamma.dtype == torch.bfloat16 else 0))
        if gamma.dtype not in (torch.float32, torch.bfloat16):
            gamma, beta = gamma.float(), beta.float()
            flags &= ~4
        y = torch.empty_like(x, memory_format=torch.channels_last)
        mean = torch.empty(b * groups, dtype=torch.float32, device=x.device)
        rstd = torch.empty_like(mean)
        N.call("sdp_group_norm_fwd", ptr(x), b, h * w, c, ptr(sd), groups, max_cg, ptr(gamma), ptr(beta),
               C.c_float(eps), flags, ptr(y), ptr(mean), ptr(rstd), stream_ptr(x.device))
        ctx.save_for_backward(x, y, gamma, mean, rstd)
        ctx.meta = (starts, flags, max_cg)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, y, gamma, mean, rstd = ctx.saved_tensors
        starts, flags, max_cg = ctx.meta
        b, c, h, w = x.shape
        dy = dy.contiguous(memory_format=torch.channels_last)
        dx = torch.empty_like(x, memory_format=torch.channels_last)
        dgb = torch.empty(2 * c, dtype=gamma.dtype, device=x.device)  # dgamma | dbeta, written
        if b > 0:
            n = C.c_longlong(0)
            N.call("sdp_group_norm_bwd_scratch", b, h * w, c, max_cg, C.byref(n))
            # per call from the caching allocator: stream-ordered, so co-resident
            # workers on different streams never share partial rows
            scratch = torch.empty(n.value, dtype=torch.float32, device=x.device)
            N.call("sdp_group_norm_bwd", ptr(x), ptr(y), ptr(dy), b, h * w, c,
                   ptr(_group_starts(starts, x.device)), len(starts) - 1, max_cg, ptr(gamma), ptr(mean), ptr(rstd),
                   flags, ptr(dx), ptr(dgb[:c]), ptr(dgb[c:]), ptr(scratch), n, stream_ptr(x.device))
        else:
            dgb.zero_()
        return dx, dgb[:c], dgb[c:], None, None, None


def _channels_last_bf16(x) -> bool:
    return (x.is_cuda and x.dtype == torch.bfloat16 and x.dim() == 4 and torch.is_autocast_enabled("cuda")
            and x.is_contiguous(memory_format=torch.channels_last))


def group_norm(x, groups: int, gamma, beta, eps: float = 1e-5, relu: bool = False,
               starts: tuple[int, ...] | None = None):
    """GroupNorm (+ReLU).  Channels-last bf16 activations under autocast (the
    training path) run libsdp's kernels over contiguous channel groups
    (`starts`: ragged group boundaries, default equal groups); otherwise
    F.group_norm, where bf16 activations under autocast stay bf16 in and out
    (fp32 statistics inside) instead of autocast's fp32 upcast."""
    if _channels_last_bf16(x):
        if starts is None:
            c = x.shape[1]
            starts = tuple(range(0, c + 1, c // groups))
        return _GroupNormCL.apply(x, gamma, beta, starts, eps, relu)
    if x.dtype == torch.bfloat16 and torch.is_autocast_enabled("cuda"):
        with torch.autocast("cuda", enabled=False):
            out = F.group_norm(x, groups, gamma.to(x.dtype), beta.to(x.dtype), eps)
    else:
        out = F.group_norm(x, groups, gamma, beta, eps)
    return F.relu(out) if relu else out


def ragged_group_norm(x, group_of: torch.Tensor, groups: int, gamma, beta, eps: float = 1e-5,
                      counts: tuple[int, ...] | None = None, relu: bool = False):
    """Compact channels, each tagged with its original norm group (F4: ragged).

    Compact channels keep ascending original order, so each group's live
    channels are contiguous: with the per-group `counts` known, equal counts
    (the grouped assignment's balanced case) are one fused F.group_norm and
    unequal ones are a few contiguous F.group_norm(., 1) calls."""
    if counts is not None:
        if _channels_last_bf16(x):  # one kernel over the ragged groups
            starts = [0]
            for c in counts:
                if c:
                    starts.append(starts[-1] + c)
            return group_norm(x, len(starts) - 1, gamma, beta, eps, relu=relu, starts=tuple(starts))
        elif len(set(counts)) == 1:
            out = group_norm(x, len(counts), gamma, beta, eps)
        else:
            outs, pos = [], 0
            for c in counts:
                if c:
                    outs.append(group_norm(x[:, pos:pos + c], 1, gamma[pos:pos + c], beta[pos:pos + c], eps))
                pos += c
            out = torch.cat(outs, dim=1)
        return F.relu(out) if relu else out
    member = F.one_hot(group_of.to(torch.long), groups)
    out = _group_norm_by_membership(x, member, gamma, beta, eps)
    return F.relu(out) if relu else out


# ---------------------------------------------------------------------------
# architectures (same constructor arguments as models.py:45-267)
# ---------------------------------------------------------------------------

class MiniResNet:
    def __init__(self, channels, blocks, classes, norm_groups=2, in_channels=3, image_hw=(8, 8)):
        if blocks < 1:
            raise ConfigError(f"mini resnet needs at least one block, got {blocks}")
        if channels % norm_groups:
            raise ConfigError(f"{norm_groups} norm groups do not divide {channels} channels")
        self.channels, self.blocks, self.classes = channels, blocks, classes
        self.norm_groups, self.in_channels, self.image_hw = norm_groups, in_channels, tuple(image_hw)

    def build_topology(self):
        return zoo.mini_resnet_topology(self.channels, self.blocks, self.classes, self.norm_groups,
                                        self.in_channels, self.image_hw)

    def forward(self, params, x, worker=None, block_mode="skip"):
        g = self.norm_groups
        ones = torch.ones(self.channels, dtype=torch.bool, device=x.device)
        # bf16 autocast training: channels-last activations and libsdp's
        # GroupNorm wherever every channel is live (block dropping); the
        # membership formulation otherwise (the f64 parity path)
        fast = x.is_cuda and torch.is_autocast_enabled("cuda")
        if fast:
            x = x.contiguous(memory_format=torch.channels_last)

        def gn(h, gamma, beta, active, relu):
            if fast and active is ones:
                return group_norm(h, g, gamma, beta, relu=relu)
            out = active_group_norm(h, g, gamma, beta, active)
            return F.relu(out) if relu else out

        h = F.conv2d(x, params["stem.w"], params["stem.b"], padding=1)
        h = gn(h, params["stem_gn.gamma"], params["stem_gn.beta"], ones, True)
        for i in range(self.blocks):
            live = True if worker is None else bool(worker.block_active[i])
            if not live and block_mode == "skip":
                continue
            a1 = _flags(worker, f"block{i}.conv1", ones)
            a2 = _flags(worker, f"block{i}.conv2", ones)
            hb = F.conv2d(h, params[f"block{i}.conv1.w"], params[f"block{i}.conv1.b"], padding=1)
            hb = gn(hb, params[f"block{i}.gn1.gamma"], params[f"block{i}.gn1.beta"], a1, True)
            hb = F.conv2d(hb, params[f"block{i}.conv2.w"], params[f"block{i}.conv2.b"], padding=1)
            hb = gn(hb, params[f"block{i}.gn2.gamma"], params[f"block{i}.gn2.beta"], a2, False)
            if not live:
                hb = hb * 0.0
            h = h + hb
        return F.linear(h.mean(dim=(2, 3)), params["head.w"], params["head.b"])

    def forward_compact(self, cp, x, sub):
        """Compact subnetwork: cp holds only live rows/columns (SubnetLayout)."""
        g = self.norm_groups
        gsize = self.channels // g
        ones = torch.ones(self.channels, dtype=torch.bool, device=x.device)
        h = F.conv2d(x, cp["stem.w"], cp["stem.b"], padding=1)
        h = F.relu(active_group_norm(h, g, cp["stem_gn.gamma"], cp["stem_gn.beta"], ones))
        for i in range(self.blocks):
            if not sub.present(f"block{i}.conv1.w"):
                continue  # dropped block: never executed (models.py:161-163)
            a1 = sub.channels(f"block{i}.conv1", self.channels)
            a2 = sub.channels(f"block{i}.conv2", self.channels)
            hb = F.conv2d(h, cp[f"block{i}.conv1.w"], cp[f"block{i}.conv1.b"], padding=1)
            hb = F.relu(ragged_group_norm(hb, a1 // gsize, g, cp[f"block{i}.gn1.gamma"], cp[f"block{i}.gn1.beta"]))
            hb = F.conv2d(hb, cp[f"block{i}.conv2.w"], cp[f"block{i}.conv2.b"], padding=1)
            hb = ragged_group_norm(hb, a2 // gsize, g, cp[f"block{i}.gn2.gamma"], cp[f"block{i}.gn2.beta"])
            h = h.index_add(1, a2, hb)
        return F.linear(h.mean(dim=(2, 3)), cp["head.w"], cp["head.b"])


class ResidualMLP:
    def __init__(self, width, blocks, classes, in_dim=16):
        if blocks < 1:
            raise ConfigError(f"residual mlp needs at least one block, got {blocks}")
        self.width, self.blocks, self.classes, self.in_dim = width, blocks, classes, in_dim

    def build_topology(self):
        return zoo.residual_mlp_topology(self.width, self.blocks, self.classes, self.in_dim)

    def forward(self, params, x, worker=None, block_mode="skip"):
        h = F.relu(F.linear(x, params["stem.w"], params["stem.b"]))
        for i in range(self.blocks):
            live = True if worker is None else bool(worker.block_active[i])
            if not live and block_mode == "skip":
                continue
            hb = F.relu(F.linear(h, params[f"block{i}.lin1.w"], params[f"block{i}.lin1.b"]))
            hb = F.linear(hb, params[f"block{i}.lin2.w"], params[f"block{i}.lin2.b"])
            if not live:
                hb = hb * 0.0
            h = h + hb
        return F.linear(h, params["head.w"], params["head.b"])

    def forward_compact(self, cp, x, sub):
        h = F.relu(F.linear(x, cp["stem.w"], cp["stem.b"]))
        for i in range(self.blocks):
            if not sub.present(f"block{i}.lin1.w"):
                continue
            hb = F.relu(F.linear(h, cp[f"block{i}.lin1.w"], cp[f"block{i}.lin1.b"]))
            h = h + F.linear(hb, cp[f"block{i}.lin2.w"], cp[f"block{i}.lin2.b"])
        return F.linear(h, cp["head.w"], cp["head.b"])


def _flags(worker, layer_id, ones):
    if worker is None or layer_id not in worker.channel_active:
        return ones
    flags = np.array(worker.channel_active[layer_id], dtype=bool)
    if flags.all():  # every channel live (block strategy): the shared all-ones mask
        return ones
    return torch.as_tensor(flags, device=ones.device)


def _make_global(arch, theta: torch.Tensor | None, dtype, dev) -> GlobalModel:
    topo = arch.build_topology()
    if theta is None:
        theta = torch.zeros(topo.total, dtype=dtype, device=dev)
    return GlobalModel(arch=arch, topology=topo, theta=theta)


def build_mini_resnet(channels, blocks, classes, norm_groups=2, in_channels=3, image_hw=(8, 8),
                      seed=0, dtype=torch.float32, device_=None, theta=None) -> GlobalModel:
    m = _make_global(MiniResNet(channels, blocks, classes, norm_groups, in_channels, image_hw),
                     theta, dtype, device(device_))
    if theta is None:
        m.theta = kaiming_fan_out_init(m, None, seed)
    return m


def build_residual_mlp(width, blocks, classes, in_dim=16, seed=0, dtype=torch.float32,
                       device_=None, theta=None) -> GlobalModel:
    m = _make_global(ResidualMLP(width, blocks, classes, in_dim), theta, dtype, device(device_))
    if theta is None:
        m.theta = kaiming_fan_out_init(m, None, seed)
    return m


def kaiming_fan_out_init(model: GlobalModel, assignment, seed: int) -> torch.Tensor:
    """masked_kaiming_init's rule (models.py:270-298): N(0, 2/fan_out_active) for
    weights, gamma = 1, bias/beta = 0.  Drawn with torch's device generator, so
    the values (not the distribution) differ from the reference's numpy draw."""
    t = model.theta
    gen = torch.Generator(device=t.device)
    gen.manual_seed(int(seed))
    theta = torch.zeros_like(t)
    for spec in model.topology.params:
        sl = slice(spec.offset, spec.offset + spec.size)
        if spec.kind == "conv_w":
            fan_out = spec.shape[0] * spec.shape[2] * spec.shape[3]
        elif spec.kind == "linear_w":
            fan_out = spec.shape[0]
        elif spec.kind in ("gamma", "norm_w"):
            theta[sl] = 1.0
            continue
        else:
            continue
        frac = 1.0 if assignment is None else assignment.output_fraction(spec.layer_id)
        std = math.sqrt(2.0 / max(1, round(fan_out * frac)))
        theta[sl] = torch.randn(spec.size, generator=gen, device=t.device, dtype=t.dtype) * std
    return theta


# ---------------------------------------------------------------------------
# compact subnetwork layout (gather / scatter descriptor tables)
# ---------------------------------------------------------------------------

SLICE_DTYPE = np.dtype([("full_offset", "<i8"), ("compact_offset", "<i8"), ("rows", "<i4"),
                        ("cols", "<i4"), ("inner", "<i4"), ("crows", "<i4"), ("ccols", "<i4"),
                        ("row_map", "<i4"), ("col_map", "<i4"), ("inner_mul", "<u4"),
                        ("inner_shr", "<u4"), ("rowlen_mul", "<u4"), ("rowlen_shr", "<u4"),
                        ("col_tab", "<i4")])
TASK_DTYPE = np.dtype([("desc", "<i4"), ("row_begin", "<i4"), ("row_end", "<i4"),
                       ("elem_begin", "<i4"), ("elem_end", "<i4"), ("seg", "<i4"), ("pad_", "<i4", 2)])
TASK_ELEMS = 4096   # elements per gather/scatter task (one worker per launch)
BATCH_TASK_ELEMS = 8192  # ... with all workers in one launch (tools/task_size_probe.py: C3 scatter
                         # 0.57 -> 0.61 of HBM, C4 gather 0.95 -> 1.03; one worker prefers 4096)
TILE_ELEMS = 2048   # max row elements a tiled task walks (256 threads x 8)
TILED_MIN = 256     # walked rows at least this long are tiled (sdp_slices.cu)


def slice_tasks(descs: np.ndarray, compact: bool, per_task: int = TASK_ELEMS) -> np.ndarray:
    """Split every tensor into work units of ~per_task elements (compact rows
    for gather, full rows for scatter): rows of >= TILED_MIN elements are cut
    into balanced, warp-aligned column chunks of <= TILE_ELEMS, and a task
    takes that chunk of several rows (the kernel resolves the chunk's column
    offsets once per task); shorter rows are grouped whole."""
    out = []
    for i, d in enumerate(descs):
        rows = int(d["crows"] if compact else d["rows"])
        row_len = int((d["ccols"] if compact else d["cols"]) * d["inner"])
        if rows == 0 or row_len == 0:
            continue
        if row_len >= TILED_MIN:
            n_chunks = -(-row_len // TILE_ELEMS)
            chunk = min(TILE_ELEMS, -(-(-(-row_len // n_chunks)) // 32) * 32)
            k = max(1, per_task // chunk)
            for e in range(0, row_len, chunk):
                for r in range(0, rows, k):
                    out.append((i, r, min(rows, r + k), e, min(row_len, e + chunk), 0, (0, 0)))
        else:
            k = max(1, per_task // row_len)
            for r in range(0, rows, k):
                out.append((i, r, min(rows, r + k), 0, row_len, 0, (0, 0)))
    return np.array(out, dtype=TASK_DTYPE)


def add_col_tables(descs: np.ndarray, maps: np.ndarray, inverse: bool) -> np.ndarray:
    """Append each column-mapped descriptor's expanded column table to `maps`
    and point `col_tab` at it (sdp.h): one int32 per element of the walked row
    -- gather: the element's offset in the full row, fwd[col_map + t // inner]
    * inner + t % inner over ccols * inner; inverse (scatter): its offset in
    the compact row or -1, over cols * inner.  Identical tables are shared."""
    parts, pos, seen = [maps.astype(np.int32)], len(maps), {}
    tabs = np.full(len(descs), -1, dtype=np.int32)
    for i, d in enumerate(descs):
        cm = int(d["col_map"])
        if cm < 0:
            continue
        inner = int(d["inner"])
        n_cols = int(d["cols"] if inverse else d["ccols"])
        key = (cm, inner, n_cols)
        if key not in seen:
            cmap = maps[cm:cm + n_cols].astype(np.int64)
            tab = (cmap[:, None] * inner + np.arange(inner)[None, :])
            if inverse:
                tab[cmap < 0] = -1
            seen[key] = pos
            parts.append(tab.reshape(-1).astype(np.int32))
            pos += tab.size
        tabs[i] = seen[key]
    descs["col_tab"] = tabs
    return np.concatenate(parts)


class SliceBatch:
    """Several workers' slice tables concatenated so ONE sdp_*_slices_multi
    launch moves all of them (task `seg` = the part's position): the
    co-resident trainer's N gathers / scatters per step become one launch
    each, large enough to be bandwidth- rather than launch-latency-bound.

    parts: [(descs, tasks, maps, compact_rows)] host tables
    (SubnetLayout.host_gather / host_scatter, layout.WorkerTransfer.host) --
    descriptor map offsets and task descriptor indices are rebased onto the
    concatenation; the tasks are re-cut at `per_task` elements (a batch
    launch has work to spare: larger tasks amortise the per-task column
    tables)."""

    def __init__(self, parts, dev, per_task: int = BATCH_TASK_ELEMS):
        from ._device import upload_struct
        if not 1 <= len(parts) <= N.MAX_WORKERS:
            raise ConfigError(f"a slice batch holds 1..{N.MAX_WORKERS} parts, got {len(parts)}")
        ds, ts, ms = [], [], []
        nd = nm = 0
        for k, (descs, tasks, maps, compact_rows) in enumerate(parts):
            if per_task:
                tasks = slice_tasks(descs, compact=compact_rows, per_task=per_task)
            d = descs.copy()
            for f in ("row_map", "col_map", "col_tab"):
                d[f] = np.where(d[f] >= 0, d[f] + nm, d[f])
            t = tasks.copy()
            t["desc"] += nd
            t["seg"] = k
            ds.append(d)
            ts.append(t)
            ms.append(maps)
            nd += len(descs)
            nm += len(maps)
        descs = np.concatenate(ds)
        tasks = np.concatenate(ts)
        # interleave the parts' tasks (round-robin) so every wave of the
        # persistent CTAs streams several workers' tensors at once
        order = np.argsort(np.concatenate([np.arange(len(t)) for t in ts]), kind="stable")
        tasks = tasks[order]
        self.n_parts = len(parts)
        self.d_descs = upload_struct(descs, dev)
        self.d_tasks = upload_struct(tasks, dev)
        self.n_tasks = len(tasks)
        self.maps = torch.from_numpy(np.concatenate(ms).astype(np.int32)).to(dev)
        self.device = dev

    def _segs(self, fulls, compacts) -> N.SliceSegs:
        if len(fulls) != self.n_parts or len(compacts) != self.n_parts:
            raise UsageError(f"slice batch of {self.n_parts} parts got {len(fulls)} / {len(compacts)} buffers")
        sg = N.SliceSegs()
        sg.n = self.n_parts
        for k, (f, c) in enumerate(zip(fulls, compacts)):
            sg.full[k] = ptr(f)
            sg.compact[k] = ptr(c)
        return sg

    def gather(self, fulls, compacts, reverse: bool = False) -> None:
        """compacts[k][...] = fulls[k][...] for every part (REVERSE: the other way)."""
        dt = slice_dtype(fulls[0].dtype)
        sg = self._segs(fulls, compacts)
        N.call("sdp_gather_slices_multi", dt, ptr(self.d_descs), ptr(self.d_tasks), self.n_tasks, ptr(self.maps),
               C.byref(sg), N.GATHER_REVERSE if reverse else 0, stream_ptr(self.device))

    def scatter(self, compacts, fulls, accumulate: bool = False) -> None:
        """fulls[k] = scatter(compacts[k]) (zero fill) or += for every part."""
        sg = self._segs(fulls, compacts)
        flags = N.SCATTER_ACCUMULATE if accumulate else N.SCATTER_ZERO_FILL
        N.call("sdp_scatter_slices_multi", sdp_dtype(compacts[0].dtype), ptr(self.d_descs), ptr(self.d_tasks),
               self.n_tasks, ptr(self.maps), C.byref(sg), flags, stream_ptr(self.device))


class SubnetLayout:
    """One worker's compact subnetwork: for every parameter the live index set
    along each governed axis (own/consumer slices, masking.py:140-149) or, for
    block masking, presence of the whole tensor (masking.py:160-169)."""

    def __init__(self, assignment, worker: int):
        topo = assignment.topology
        self.topology = topo
        self.worker = worker
        dev = assignment.device
        view = assignment.worker_view(worker)
        self.view = view
        # live channel indices per layer (neuron) / live blocks (block)
        live_ch: dict[str, np.ndarray] = {}
        axes: dict[str, dict[int, str]] = {p.name: {} for p in topo.params}
        present = {p.name: True for p in topo.params}
        if assignment.strategy == "neuron":
            for layer in topo.channel_layers:
                if not layer.maskable:
                    continue
                live_ch[layer.layer_id] = np.nonzero(view.channel_active[layer.layer_id])[0]
                for pname, axis in tuple(layer.own_slices) + tuple(layer.consumer_slices):
                    if axis in axes[pname]:
                        raise ConfigError(f"{pname} axis {axis} governed twice")
                    axes[pname][axis] = layer.layer_id
        else:
            for b in topo.blocks:
                if b.maskable and not view.block_active[b.index]:
                    for pname in b.param_names:
                        present[pname] = False
        self.live_channels = {k: torch.as_tensor(v, dtype=torch.long, device=dev) for k, v in live_ch.items()}
        self.present_map = present
        # forward / inverse index maps, one pair per layer
        fwd, inv, fwd_off, inv_off = [], [], {}, {}
        for lid, idx in live_ch.items():
            layer = topo.channel_layer(lid)
            fwd_off[lid] = sum(len(a) for a in fwd)
            fwd.append(idx.astype(np.int32))
            m = np.full(layer.channels, -1, dtype=np.int32)
            m[idx] = np.arange(len(idx), dtype=np.int32)
            inv_off[lid] = sum(len(a) for a in inv)
            inv.append(m)
        descs = np.zeros(len(topo.params), dtype=SLICE_DTYPE)
        self.shapes: dict[str, tuple[int, ...]] = {}
        self.offsets: dict[str, int] = {}
        inv_rows: list[tuple[int, int]] = []   # (row_map, col_map) offsets into the inverse maps
        pos = 0
        for i, p in enumerate(topo.params):
            ax = axes[p.name]
            if any(a > 1 for a in ax):
                raise ConfigError(f"{p.name}: only axes 0 and 1 may be channel-governed")
            # canonical [rows, cols, inner]: a 1-D tensor is one row of `cols`;
            # an ungoverned axis 1 folds into `inner` (contiguous rows)
            if len(p.shape) == 1:
                rows, cols, inner = 1, p.shape[0], 1
                rlid, clid = None, ax.get(0)
            else:
                rows, cols = p.shape[0], p.shape[1]
                inner = int(np.prod(p.shape[2:])) if len(p.shape) > 2 else 1
                rlid, clid = ax.get(0), ax.get(1)
                if clid is None:
                    inner *= cols
                    cols = 1
            if rows * cols * inner >= 1 << 31:
                raise ConfigError(f"{p.name}: 2^31 or more elements exceed the slice kernels' "
                                  "32-bit in-tensor offsets")
            crows = len(live_ch[rlid]) if rlid else rows
            ccols = len(live_ch[clid]) if clid else cols
            if not present[p.name]:
                crows = 0
            cshape = list(p.shape)
            for axis, lid in ax.items():
                cshape[axis] = len(live_ch[lid])
            if not present[p.name]:
                cshape[0] = 0
            mul, shr = fast_divisor(inner)
            rl_mul, rl_shr = fast_divisor(max(1, ccols * inner))
            descs[i] = (p.offset, pos, rows, cols, inner, crows, ccols,
                        fwd_off[rlid] if rlid else -1, fwd_off[clid] if clid else -1, mul, shr,
                        rl_mul, rl_shr, 0)
            inv_rows.append((inv_off[rlid] if rlid else -1, inv_off[clid] if clid else -1))
            self.shapes[p.name] = tuple(cshape)
            self.offsets[p.name] = pos
            pos += crows * ccols * inner
        self.compact_total = pos
        descs_inv = descs.copy()
        descs_inv["row_map"] = [r for r, _ in inv_rows]
        descs_inv["col_map"] = [c for _, c in inv_rows]
        full_rl = [fast_divisor(max(1, int(d["cols"] * d["inner"]))) for d in descs]
        descs_inv["rowlen_mul"] = [m for m, _ in full_rl]
        descs_inv["rowlen_shr"] = [s for _, s in full_rl]
        from ._device import upload_struct
        fw = np.concatenate(fwd) if fwd else np.zeros(1, np.int32)
        iv = np.concatenate(inv) if inv else np.zeros(1, np.int32)
        fw = add_col_tables(descs, fw, inverse=False)
        iv = add_col_tables(descs_inv, iv, inverse=True)
        self.descs = descs
        self.d_fwd = upload_struct(descs, dev)
        self.d_inv = upload_struct(descs_inv, dev)
        g_tasks = slice_tasks(descs, compact=True)
        s_tasks = slice_tasks(descs, compact=False)
        # host copies: SliceBatch concatenates several workers' tables
        # (descriptors, tasks, maps, whether tasks walk compact rows)
        self.host_gather = (descs, g_tasks, fw.astype(np.int32), True)
        self.host_scatter = (descs_inv, s_tasks, iv.astype(np.int32), False)
        self.t_gather, self.n_gather = upload_struct(g_tasks, dev), len(g_tasks)
        self.t_scatter, self.n_scatter = upload_struct(s_tasks, dev), len(s_tasks)
        self.fwd_maps = torch.from_numpy(fw.astype(np.int32)).to(dev)
        self.inv_maps = torch.from_numpy(iv.astype(np.int32)).to(dev)

    def present(self, name: str) -> bool:
        return self.present_map[name] and int(np.prod(self.shapes[name])) > 0

    def group_counts(self, layer_id: str, channels: int, groups: int) -> tuple[int, ...]:
        """Live channels per original norm group (ragged)."""
        key = (layer_id, channels, groups)
        if not hasattr(self, "_gcounts"):
            self._gcounts = {}
        if key not in self._gcounts:
            t = self.live_channels.get(layer_id)
            gsize = channels // groups
            if t is None:
                self._gcounts[key] = (gsize,) * groups
            else:
                idx = t.cpu().numpy()
                self._gcounts[key] = tuple(int(v) for v in np.bincount(idx // gsize, minlength=groups))
        return self._gcounts[key]

    def channels(self, layer_id: str, c: int) -> torch.Tensor:
        t = self.live_channels.get(layer_id)
        if t is None:
            return torch.arange(c, device=self.fwd_maps.device)
        return t

    def views(self, compact: torch.Tensor) -> dict:
        """Per-parameter views of the compact buffer: one split (backward = one
        concatenation, not a [compact] zero-fill + accumulate per parameter)."""
        sizes = [int(np.prod(self.shapes[p.name])) for p in self.topology.params]
        flat = compact if compact.numel() == sum(sizes) else compact[:sum(sizes)]
        parts = flat.split(sizes)
        return {p.name: t.view(self.shapes[p.name]) for p, t in zip(self.topology.params, parts)}

    # -- kernels --------------------------------------------------------------
    def gather(self, theta: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Full theta -> compact buffer (sdp_gather_slices)."""
        if out is None:
            out = torch.empty(max(1, self.compact_total), dtype=theta.dtype, device=theta.device)
        N.call("sdp_gather_slices", slice_dtype(theta.dtype), ptr(self.d_fwd), ptr(self.t_gather),
               self.n_gather, ptr(self.fwd_maps), ptr(theta), ptr(out), 0, stream_ptr(theta.device))
        return out

    def scatter(self, compact: torch.Tensor, full: torch.Tensor | None = None,
                accumulate: bool = False) -> torch.Tensor:
        """Compact gradient -> flat [d] (zero elsewhere), or += into `full`."""
        d = self.topology.total
        if full is None:
            full = torch.empty(d, dtype=compact.dtype, device=compact.device)
            accumulate = False
        flags = N.SCATTER_ACCUMULATE if accumulate else N.SCATTER_ZERO_FILL
        N.call("sdp_scatter_slices", sdp_dtype(compact.dtype), ptr(self.d_inv), ptr(self.t_scatter),
               self.n_scatter, ptr(self.inv_maps), ptr(compact), ptr(full), flags,
               stream_ptr(compact.device))
        return full


# ---------------------------------------------------------------------------
# reference-facing entry points
# ---------------------------------------------------------------------------

@dataclass
class Tape:
    """What flat_gradient needs from masked_forward (the reference's tape role)."""
    leaf: torch.Tensor
    layout: SubnetLayout | None


def _extract(theta: torch.Tensor, worker) -> torch.Tensor:
    """theta * mask (models.py:355) via sdp_masked_extract on the worker's byte mask."""
    out = torch.empty_like(theta)
    mask = worker.param_mask_bool.view(torch.uint8)
    N.call("sdp_masked_extract", sdp_dtype(theta.dtype), ptr(theta), ptr(mask), 1, theta.numel(), 0,
           ptr(out), stream_ptr(theta.device))
    return out


def masked_forward(model: GlobalModel, worker, xs, ys, block_mode: str = "skip",
                   record: bool = True, layout: str = "full", subnet: SubnetLayout | None = None):
    """One loss evaluation on the worker's subnetwork (models.py:333-366)."""
    topo = model.topology
    xs = torch.as_tensor(xs, device=model.theta.device)
    if tuple(xs.shape[1:]) != tuple(topo.input_shape):
        raise InputError(f"batch shape {tuple(xs.shape[1:])} does not match model input {topo.input_shape}")
    if block_mode not in ("skip", "multiply"):
        raise ConfigError(f"unknown block_mode {block_mode!r}")
    ys = torch.as_tensor(ys, device=model.theta.device, dtype=torch.long)
    xs = xs.to(model.theta.dtype)
    if layout == "compact":
        if subnet is None:
            raise ConfigError("layout='compact' needs the worker's SubnetLayout")
        leaf = subnet.gather(model.theta).requires_grad_(record)
        cp = subnet.views(leaf)
        logits = model.arch.forward_compact(cp, xs, subnet)
        loss = F.cross_entropy(logits, ys)
        return loss, Tape(leaf, subnet), cp
    if layout != "full":
        raise ConfigError(f"unknown layout {layout!r}")
    theta = model.theta if worker is None else _extract(model.theta, worker)
    leaf = theta.detach().requires_grad_(record)
    params = {p.name: leaf[p.offset:p.offset + p.size].view(p.shape) for p in topo.params}
    logits = model.arch.forward(params, xs, worker, block_mode)
    loss = F.cross_entropy(logits, ys)
    return loss, Tape(leaf, None), params


def aggregate_compact(compact_grads, layouts, assignment) -> torch.Tensor:
    """engine.aggregate over compact per-worker gradients: each worker's compact
    gradient is scatter-ACCUMULATED into one [d] buffer in ascending worker id
    (exactly the reference's num += m_i * g_i order, engine.py:71-73), then
    divided by the divisor (engine.py:74) -- no [d] gradient per worker."""
    d = assignment.topology.total
    dt = compact_grads[0].dtype
    acc = torch.zeros(d, dtype=dt, device=assignment.device)
    for g, lay in sorted(zip(compact_grads, layouts), key=lambda x: x[1].worker):
        lay.scatter(g, acc, accumulate=True)
    out = torch.empty_like(acc)
    N.call("sdp_divide", sdp_dtype(dt), ptr(acc), ptr(assignment.divisor), d, ptr(out),
           stream_ptr(assignment.device))
    return out


def flat_gradient(model: GlobalModel, tape: Tape, loss, params) -> torch.Tensor:
    """Backward pass assembled into a vector aligned with the flat theta
    (models.py:369-382): entries of dropped / dead parameters are exactly 0."""
    (g,) = torch.autograd.grad(loss, tape.leaf, allow_unused=True)
    if g is None:
        g = torch.zeros_like(tape.leaf)
    if tape.layout is None:
        return g
    return tape.layout.scatter(g.contiguous())
