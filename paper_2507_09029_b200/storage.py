"""Compact owned-block storage (SURVEY.md §7 hard part 7, §8(b) per-owner offsets).

The paper's memory claim -- each worker's parameters, gradients and optimizer
state shrink by 1 - P/N (the reference's analytic accounting,
diagnostics.py:113-140) -- needs storage that holds only what a worker owns.
The unit of storage here is the owner-sync tile (engine.SyncPlan: `tile`
consecutive elements of the reference's flat layout): worker w stores exactly
the tiles whose owner union contains w, back to back in tile order.  Tile t of
worker w sits at element `slot[w, t] * tile` of w's compact buffer; the slot
table (int32 [N, n_tiles], -1 = not stored) is the per-owner offset table that
k_owner_sync reads for every owner of every tile (sdp_sync_args.slots), so the
same kernel syncs compact replicas, local or peer-mapped.

Block strategy: every parameter of a live block (and every always-active one)
lies in tiles the worker stores, in consecutive slots, so each live parameter
is ONE contiguous range of the compact buffer (`param_offset`); parameters of
dropped blocks have no storage at all.  Tiles straddling a block boundary are
stored whole (at most one tile of slack per boundary).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .errors import UsageError

UPDATE_DTYPE = np.dtype([("state", "<u4"), ("slot", "<u4"), ("len", "<u4"), ("pad", "<u4")])


def dispatch_order(tiles: np.ndarray, order: str = "mixed_first") -> np.ndarray:
    """Permutation of a rank's tiles into launch order (CTA b runs positions
    b, b + grid, ...): lane-per-element mixed tiles first (engine.SyncPlan)."""
    if order == "index":
        return np.arange(len(tiles))
    uni = (tiles["len_flags"] & N.TILE_UNIFORM) != 0
    if order == "mixed_first":
        key = uni.astype(np.int64)
    elif order == "cost":  # heaviest first: owners read, x5 for lane-per-element tiles
        pc = np.bitwise_count(tiles["owner_bits"]).astype(np.int64)
        key = -(pc * np.where(uni, 1, 5))
    else:
        raise ValueError(f"unknown tile order {order!r}")
    return np.argsort(key, kind="stable")


def leader_cta(all_tiles: np.ndarray, leaders: np.ndarray, world: int, grid: int,
               order: str = "mixed_first") -> np.ndarray:
    """For every tile: the CTA index that reduces it on its leader rank (each
    rank runs its led tiles in dispatch order, CTA b taking positions
    b, b + grid, ...; every rank launches the same grid)."""
    cta = np.empty(len(all_tiles), dtype=np.int64)
    for r in range(world):
        idx = np.nonzero(leaders == r)[0]
        ordered = idx[dispatch_order(all_tiles[idx], order)]
        cta[ordered] = np.arange(len(ordered)) % grid
    return cta


class CompactLayout:
    """Owned-tile storage of every worker of one sync plan."""

    def __init__(self, plan):
        tiles = plan.all_tiles
        self.plan = plan
        self.tile = int(plan.tile)
        self.n_tiles = len(tiles)
        self.total = int(plan.assignment.topology.total)
        self.n_workers = int(plan.assignment.n_workers)
        self.tile_len = (tiles["len_flags"] & N.TILE_LEN_MASK).astype(np.int64)
        bits = tiles["owner_bits"].astype(np.uint64)
        self.stored = [np.nonzero((bits >> np.uint64(w)) & np.uint64(1))[0] for w in range(self.n_workers)]
        slots = np.full((self.n_workers, max(1, self.n_tiles)), -1, dtype=np.int32)
        for w, st in enumerate(self.stored):
            slots[w, st] = np.arange(len(st), dtype=np.int32)
        self.slots_host = slots
        self.slots = torch.from_numpy(slots.reshape(-1).copy()).to(plan.assignment.device)

    @property
    def slot_stride(self) -> int:
        return self.slots_host.shape[1]

    def length(self, w: int) -> int:
        """Elements of worker w's compact buffer (>= one tile, so every buffer
        has a valid 16-byte aligned base)."""
        return max(1, len(self.stored[w])) * self.tile

    def stored_elements(self, w: int) -> int:
        """Flat elements covered by worker w's stored tiles."""
        return int(self.tile_len[self.stored[w]].sum())

    def compact_offset(self, w: int, flat: int) -> int:
        t = flat // self.tile
        sl = int(self.slots_host[w, t])
        if sl < 0:
            raise UsageError(f"worker {w} does not store element {flat} (tile {t})")
        return sl * self.tile + flat % self.tile

    def param_offset(self, w: int, spec) -> int:
        """Compact offset of parameter `spec` (ParamSpec) in worker w's buffer;
        the parameter must lie in tiles w stores, in consecutive slots."""
        if spec.size == 0:
            return 0
        t0, t1 = spec.offset // self.tile, (spec.offset + spec.size - 1) // self.tile
        sl = self.slots_host[w, t0:t1 + 1]
        if sl[0] < 0 or np.any(np.diff(sl) != 1):
            raise UsageError(f"parameter {spec.name} is not stored contiguously by worker {w}")
        return int(sl[0]) * self.tile + spec.offset % self.tile

    def views(self, w: int, buf: torch.Tensor, specs) -> dict:
        """{name: view of buf} for the given ParamSpecs of worker w."""
        out = {}
        for p in specs:
            o = self.param_offset(w, p)
            out[p.name] = buf[o:o + p.size].view(p.shape)
        return out

    def _index(self, w: int, dev) -> torch.Tensor:
        key = (w, str(dev))
        if not hasattr(self, "_idx"):
            self._idx = {}
        if key not in self._idx:
            self._idx[key] = torch.from_numpy(self.stored[w].astype(np.int64)).to(dev)
        return self._idx[key]

    def gather(self, w: int, flat: torch.Tensor) -> torch.Tensor:
        """Worker w's compact buffer of a flat [d] vector (tiles beyond d zero)."""
        pad = self.n_tiles * self.tile - flat.numel()
        full = torch.nn.functional.pad(flat, (0, pad)) if pad else flat
        out = torch.zeros(self.length(w), dtype=flat.dtype, device=flat.device)
        if len(self.stored[w]):
            n = len(self.stored[w]) * self.tile
            out[:n] = full.view(self.n_tiles, self.tile).index_select(0, self._index(w, flat.device)).reshape(-1)
        return out

    def scatter(self, w: int, compact: torch.Tensor, flat: torch.Tensor) -> torch.Tensor:
        """Write worker w's stored tiles back into a flat [d] vector (in place)."""
        if not len(self.stored[w]):
            return flat
        pad = self.n_tiles * self.tile - flat.numel()
        full = torch.nn.functional.pad(flat, (0, pad)) if pad else flat.clone()
        n = len(self.stored[w]) * self.tile
        full.view(self.n_tiles, self.tile).index_copy_(0, self._index(w, flat.device),
                                                        compact[:n].view(-1, self.tile))
        flat.copy_(full[:flat.numel()])
        return flat

    def update_table(self, local_workers, cta_of_tile: np.ndarray, grid: int):
        """CTA-major sdp_update_desc table of the local-update phase: CTA b gets
        (state, slot, len) for every stored tile of every local worker whose
        leader ran in CTA b.  Returns (table uint8 device tensor, per_cta)."""
        per = [[] for _ in range(grid)]
        for si, w in enumerate(local_workers):
            for sl, t in enumerate(self.stored[w]):
                per[int(cta_of_tile[t])].append((si, sl, int(self.tile_len[t])))
        per_cta = max(1, max(len(x) for x in per))
        table = np.zeros(grid * per_cta, dtype=UPDATE_DTYPE)
        for b, lst in enumerate(per):
            for k, (si, sl, ln) in enumerate(lst):
                table[b * per_cta + k] = (si, sl, ln, 0)
        from ._device import upload_struct
        return upload_struct(table, self.plan.assignment.device), per_cta


def worker_states(entries, dev) -> torch.Tensor:
    """Device array of sdp_worker_state: entries = [(theta, velocity,
    second_moment|None, theta_bf16|None, grad)] tensors."""
    arr = (N.WorkerState * max(1, len(entries)))()
    for i, (th, v, m2, tb, g) in enumerate(entries):
        arr[i] = N.WorkerState(th.data_ptr(), v.data_ptr(), None if m2 is None else m2.data_ptr(),
                               None if tb is None else tb.data_ptr(), g.data_ptr())
    raw = np.frombuffer(bytes(arr), dtype=np.uint8)
    from ._device import upload_struct
    return upload_struct(raw, dev)
