"""Window-class-major sync layout (SURVEY.md §7 hard part 4).

In the reference's flat layout a width-wise (neuron) assignment changes owner
set every 1-9 elements: a conv weight's element (o, i, k) is owned by
window(o) ∩ window(i).  The sync then has to read a per-element owner mask
and its owner writes cover partial 32-B sectors, which L2 turns into DRAM
read-modify-writes (ncu: 1.6x the algorithmic reads, 0.40 of the HBM peak).

The sync layout permutes every tensor so that rows are grouped by their row
owner set and columns by their column owner set, and stores each
(row class, column class) block contiguously.  A block has ONE owner set
(row bits & column bits & block bits), so the sync sees long uniform runs:
tiles carry their owner set, no mask is read, every write covers whole
sectors.  The permutation is a set of canonical slice descriptors (one per
block) run by libsdp's gather kernel: `to_sync` gathers, `from_sync` is the
reverse gather; a worker's compact tensors map to the blocks it owns with
the same kernel (`WorkerTransfer`), so width-wise training never touches the
reference layout at all.  For the block strategy the layout is the identity.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from ._device import ptr, slice_dtype, stream_ptr, upload_struct
from .errors import ConfigError
from .topology import fast_divisor


def _canonical(shape):
    """[rows, cols, inner] of a tensor, with the axis-0 rule on rows and the
    axis-1 rule on cols (a 1-D tensor is one row of cols)."""
    if len(shape) == 1:
        return 1, int(shape[0]), 1, (None, 0)
    inner = int(np.prod(shape[2:])) if len(shape) > 2 else 1
    return int(shape[0]), int(shape[1]), inner, (0, 1)


def _classes(bits: np.ndarray):
    """Group indices by owner bits: [(bits, ascending indices)] ordered by bits."""
    out = []
    for b in np.unique(bits):
        out.append((int(b), np.nonzero(bits == b)[0].astype(np.int32)))
    return out


class _DescBuilder:
    def __init__(self):
        from .models import SLICE_DTYPE
        self.rows, self.maps, self.map_len = [], [], 0
        self.dtype = SLICE_DTYPE

    def map_offset(self, idx: np.ndarray | None) -> int:
        if idx is None:
            return -1
        off = self.map_len
        self.maps.append(idx.astype(np.int32))
        self.map_len += len(idx)
        return off

    def add(self, full_off, comp_off, rows, cols, inner, rmap, cmap):
        if rows * cols * inner >= 1 << 31:
            raise ConfigError("a tensor of 2^31 or more elements exceeds the slice kernels' "
                              "32-bit in-tensor offsets")
        crows = len(rmap) if rmap is not None else rows
        ccols = len(cmap) if cmap is not None else cols
        mul, shr = fast_divisor(inner)
        rl_mul, rl_shr = fast_divisor(max(1, ccols * inner))
        self.rows.append((full_off, comp_off, rows, cols, inner, crows, ccols, self.map_offset(rmap),
                          self.map_offset(cmap), mul, shr, rl_mul, rl_shr, -1))
        return crows * ccols * inner

    def upload(self, dev):
        from .models import add_col_tables, slice_tasks
        descs = np.array(self.rows, dtype=self.dtype)
        tasks = slice_tasks(descs, compact=True)
        maps = np.concatenate(self.maps) if self.maps else np.zeros(1, np.int32)
        maps = add_col_tables(descs, maps, inverse=False)
        self.host = (descs, tasks, maps.astype(np.int32), True)  # for models.SliceBatch
        return (upload_struct(descs, dev), upload_struct(tasks, dev), len(tasks),
                torch.from_numpy(maps.astype(np.int32)).to(dev))


def _gather(dtype_code, d_desc, d_tasks, n_tasks, maps, full, compact, reverse, dev):
    N.call("sdp_gather_slices", dtype_code, ptr(d_desc), ptr(d_tasks), n_tasks, ptr(maps), ptr(full),
           ptr(compact), N.GATHER_REVERSE if reverse else 0, stream_ptr(dev))


class SyncLayout:
    """Window-class-major permutation of one assignment's flat vector."""

    def __init__(self, assignment):
        if assignment._unit_bits is None or assignment._tables is None:
            raise ConfigError("the sync layout needs an assignment built from unit ownership "
                              "(build_assignment / load_assignment)")
        if assignment.mask_bytes != 1:
            raise ConfigError("the sync layout currently supports N <= 8 workers")
        self.assignment = assignment
        topo = assignment.topology
        dev = assignment.device
        table = assignment._tables.table
        ub = assignment._unit_bits.cpu().numpy().view(np.uint64)
        full = np.uint64((1 << assignment.n_workers) - 1)
        axes: dict[str, dict[int, str]] = {p.name: {} for p in topo.params}
        pbits = {p.name: full for p in topo.params}
        if assignment.strategy == "neuron":
            for layer in topo.channel_layers:
                if layer.layer_id in table.layer_base:
                    for pname, axis in tuple(layer.own_slices) + tuple(layer.consumer_slices):
                        axes[pname][axis] = layer.layer_id
        else:
            for b in topo.blocks:
                if b.block_id in table.block_unit:
                    for pname in b.param_names:
                        pbits[pname] = pbits[pname] & ub[table.block_unit[b.block_id]]
        self.blocks: dict[str, list] = {}   # param -> [(sync_off, row_idx, col_idx, bits)]
        self.shapes: dict[str, tuple] = {}
        self.axis_layers: dict[str, tuple] = {}  # param -> (row layer, col layer) or None
        builder = _DescBuilder()
        pos = 0
        for p in topo.params:
            rows, cols, inner, (rax, cax) = _canonical(p.shape)
            ax = axes[p.name]
            if any(a > 1 for a in ax):
                raise ConfigError(f"{p.name}: only axes 0 and 1 may be channel-governed")
            if len(p.shape) == 1:
                rbits = np.full(1, full, np.uint64)
                cbits = ub[table.layer_base[ax[0]] + np.arange(cols)] if 0 in ax else np.full(cols, full, np.uint64)
            else:
                rbits = ub[table.layer_base[ax[0]] + np.arange(rows)] if 0 in ax else np.full(rows, full, np.uint64)
                cbits = ub[table.layer_base[ax[1]] + np.arange(cols)] if 1 in ax else np.full(cols, full, np.uint64)
            self.shapes[p.name] = (rows, cols, inner)
            self.axis_layers[p.name] = (None, ax.get(0)) if len(p.shape) == 1 else (ax.get(0), ax.get(1))
            blocks = []
            rcl, ccl = _classes(rbits), _classes(cbits)
            ident_r = len(rcl) == 1
            ident_c = len(ccl) == 1
            for rb, ridx in rcl:
                for cb, cidx in ccl:
                    bits = np.uint64(rb) & np.uint64(cb) & pbits[p.name]
                    n = builder.add(p.offset, pos, rows, cols, inner,
                                    None if ident_r else ridx, None if ident_c else cidx)
                    blocks.append((pos, ridx, cidx, int(bits)))
                    pos += n
            self.blocks[p.name] = blocks
        assert pos == topo.total
        self.d_desc, self.d_tasks, self.n_tasks, self.maps = builder.upload(dev)
        # owner mask in sync space -> tile plan with (mostly) uniform tiles
        self.owner_mask = torch.empty_like(assignment.owner_mask)
        _gather(N.DTYPE_U8, self.d_desc, self.d_tasks, self.n_tasks, self.maps, assignment.owner_mask,
                self.owner_mask, False, dev)
        self._plans = {}

    def plan(self, **kw):
        from .engine import SyncPlan
        key = tuple(sorted(kw.items()))
        if key not in self._plans:
            self._plans[key] = SyncPlan(self.assignment, owner_mask=self.owner_mask, **kw)
        return self._plans[key]

    def to_sync(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        out = torch.empty_like(x) if out is None else out
        _gather(slice_dtype(x.dtype), self.d_desc, self.d_tasks, self.n_tasks, self.maps, x, out, False, x.device)
        return out

    def from_sync(self, s: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        out = torch.empty_like(s) if out is None else out
        _gather(slice_dtype(s.dtype), self.d_desc, self.d_tasks, self.n_tasks, self.maps, out, s, True, s.device)
        return out


class WorkerTransfer:
    """Worker w's compact tensors (models.SubnetLayout) <-> the sync-layout
    blocks w owns: `to_compact(theta_sync)` extracts the worker's parameters,
    `from_compact(g, grad_sync)` writes its gradient into its replica in sync
    space.  Entries of blocks w does not own are never touched (and never read
    by the sync kernel)."""

    def __init__(self, layout: SyncLayout, sub, compact=None):
        """compact: a storage.CompactLayout of the sync-space plan -- the
        worker's sync-space buffers (theta, bf16 copy, gradient replica) then
        hold only the tiles it owns, and every sync block is addressed at its
        slot-mapped offset (a block the worker owns spans stored tiles only,
        in consecutive slots)."""
        a = layout.assignment
        w = sub.worker
        topo = a.topology
        builder = _DescBuilder()
        for p in topo.params:
            if not sub.present_map.get(p.name, True) or int(np.prod(sub.shapes[p.name])) == 0:
                continue
            rows, cols, inner = layout.shapes[p.name]
            rl, cl = layout.axis_layers[p.name]
            live_r = sub.live_channels[rl].cpu().numpy() if rl else np.arange(rows)
            live_c = sub.live_channels[cl].cpu().numpy() if cl else np.arange(cols)
            crows, ccols = len(live_r), len(live_c)
            for off, ridx, cidx, bits in layout.blocks[p.name]:
                if not (bits >> w) & 1:
                    continue
                rpos = np.searchsorted(live_r, ridx).astype(np.int32)
                cpos = np.searchsorted(live_c, cidx).astype(np.int32)
                # "full" = the worker's compact tensor [crows, ccols, inner] (same memory
                # order as SubnetLayout's), "compact" = the contiguous sync block
                size = len(ridx) * len(cidx) * inner
                if compact is not None and size:
                    c0 = compact.compact_offset(w, off)
                    if compact.compact_offset(w, off + size - 1) != c0 + size - 1:
                        raise ConfigError(f"{p.name}: sync block at {off} is not contiguous in worker {w}'s "
                                          "owned-tile storage")
                    off = c0
                builder.add(sub.offsets[p.name], off, crows, ccols, inner,
                            None if len(rpos) == crows else rpos, None if len(cpos) == ccols else cpos)
        self.d_desc, self.d_tasks, self.n_tasks, self.maps = builder.upload(a.device)
        self.host = builder.host
        self.compact_total = sub.compact_total

    def to_compact(self, theta_sync: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        out = torch.empty(max(1, self.compact_total), dtype=theta_sync.dtype, device=theta_sync.device) \
            if out is None else out
        _gather(slice_dtype(theta_sync.dtype), self.d_desc, self.d_tasks, self.n_tasks, self.maps, out,
                theta_sync, True, theta_sync.device)
        return out

    def from_compact(self, g: torch.Tensor, grad_sync: torch.Tensor) -> torch.Tensor:
        _gather(slice_dtype(g.dtype), self.d_desc, self.d_tasks, self.n_tasks, self.maps, g, grad_sync, False,
                g.device)
        return grad_sync

