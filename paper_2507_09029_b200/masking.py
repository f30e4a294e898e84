"""Mask construction on the GPU, behind the reference's masking API
(`/root/reference/pkg/src/subnetdp/masking.py`).

Same names, arguments, return shapes and exceptions as the reference; the
difference is where the arrays live.  `param_masks`, `coverage`, `divisor`,
`governors` are CUDA tensors built by libsdp's k_assign + k_build_masks, and
every MaskAssignment also carries the compact per-element owner bitmask
(`owner_mask`, one byte per element for N <= 8) that the sync kernel reads.

Reference map:
  StructuralUnit ............. masking.py:35-53
  slot_windows ............... masking.py:56-66
  assign_units ............... masking.py:69-85     (device: sdp_assign_units)
  assign_grouped_units ....... masking.py:88-117    (device: sdp_assign_units)
  induce_channel_param_mask .. masking.py:120-150   (device: sdp_build_masks)
  induce_block_param_mask .... masking.py:153-170   (device: sdp_build_masks)
  WorkerMaskView ............. masking.py:173-185
  MaskAssignment ............. masking.py:188-269   (worker_view: sdp_worker_mask)
  build_assignment ........... masking.py:305-359
  validate ................... masking.py:384-444
  JSON I/O ................... masking.py:447-503
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _native as N
from ._device import MASK_TORCH_DTYPE, device, mask_bytes_for, ptr, read_only, stream_ptr, upload_struct
from .errors import ConfigError, TopologyError, UsageError, ValidationError
from .topology import ModelTopology, UnitTable, unit_table

KIND_CHANNEL = "channel"
KIND_BLOCK = "block"
STRATEGIES = ("neuron", "block")


@dataclass(frozen=True, order=True)
class StructuralUnit:
    kind: str
    ref: str
    index: int = -1

    def key(self) -> str:
        if self.kind == KIND_BLOCK:
            return f"block:{self.ref}"
        return f"channel:{self.ref}:{self.index}"

    @staticmethod
    def from_key(key: str) -> "StructuralUnit":
        parts = key.split(":")
        if len(parts) == 2 and parts[0] == KIND_BLOCK:
            return StructuralUnit(KIND_BLOCK, parts[1])
        if len(parts) == 3 and parts[0] == KIND_CHANNEL:
            return StructuralUnit(KIND_CHANNEL, parts[1], int(parts[2]))
        raise ConfigError(f"unparseable unit key {key!r}")


def _check_replication(n_workers: int, replication: int) -> None:
    if not 1 <= replication <= n_workers:
        raise ConfigError(
            f"replication must satisfy 1 <= P <= N, got P={replication}, N={n_workers}")
    if n_workers > N.MAX_WORKERS:
        raise ConfigError(f"at most {N.MAX_WORKERS} workers are supported, got {n_workers}")


def slot_windows(num_units: int, n_workers: int, replication: int) -> list[tuple[int, ...]]:
    """Cyclic window of slot j: {(j*P + t) mod N}, ascending (masking.py:56-66)."""
    if not 1 <= replication <= n_workers:
        raise ConfigError(
            f"replication must satisfy 1 <= P <= N, got P={replication}, N={n_workers}")
    out = []
    for j in range(num_units):
        start = (j * replication) % n_workers
        out.append(tuple(sorted((start + t) % n_workers for t in range(replication))))
    return out


def _bits_to_workers(bits: int, n_workers: int) -> tuple[int, ...]:
    return tuple(w for w in range(n_workers) if (bits >> w) & 1)


def _device_assign(groups: list[tuple[int, int]], n_units: int, n_workers: int,
                   replication: int, seed: int, dev: torch.device) -> torch.Tensor:
    """Run k_assign: uint64 owner bits per unit (stored as int64)."""
    garr = np.array(groups, dtype=np.int32).reshape(-1, 2)
    g_dev = upload_struct(garr, dev)
    unit_bits = torch.empty(max(n_units, 1), dtype=torch.int64, device=dev)
    max_group = int(garr[:, 1].max())
    scratch = torch.empty(8 * max(n_units, 1) + 1, dtype=torch.int32, device=dev)
    words, nw = N.seed_words(seed)
    N.call("sdp_assign_units", words, nw, ptr(g_dev), len(groups), max_group, n_units,
           n_workers, replication, ptr(unit_bits), ptr(scratch), stream_ptr(dev))
    return unit_bits[:n_units]


def assign_units(units: list[StructuralUnit], n_workers: int, replication: int, seed: int,
                 device_=None) -> dict[StructuralUnit, tuple[int, ...]]:
    """Each unit on exactly P workers, balanced and seeded (masking.py:69-85)."""
    if not units:
        raise ConfigError("assign_units requires a non-empty unit list")
    _check_replication(n_workers, replication)
    bits = _device_assign([(0, len(units))], len(units), n_workers, replication, seed,
                          device(device_)).cpu().numpy().view(np.uint64)
    return {u: _bits_to_workers(int(bits[i]), n_workers) for i, u in enumerate(units)}


def assign_grouped_units(unit_groups: list[list[StructuralUnit]], n_workers: int,
                         replication: int, seed: int,
                         device_=None) -> dict[StructuralUnit, tuple[int, ...]]:
    """Group-balanced assignment with one generator and a running slot counter
    (masking.py:88-117)."""
    if not unit_groups or any(not g for g in unit_groups):
        raise ConfigError("assign_grouped_units requires non-empty groups")
    _check_replication(n_workers, replication)
    groups, flat, pos = [], [], 0
    for g in unit_groups:
        groups.append((pos, len(g)))
        flat.extend(g)
        pos += len(g)
    bits = _device_assign(groups, pos, n_workers, replication, seed,
                          device(device_)).cpu().numpy().view(np.uint64)
    out: dict[StructuralUnit, tuple[int, ...]] = {}
    for i, u in enumerate(flat):
        out[u] = _bits_to_workers(int(bits[i]), n_workers)
    return out


# ---------------------------------------------------------------------------
# device mask tables
# ---------------------------------------------------------------------------

class _DeviceTables:
    """Topology lowered to device descriptors for one strategy (cached)."""

    def __init__(self, topology: ModelTopology, strategy: str, dev: torch.device):
        self.table: UnitTable = unit_table(topology, strategy)
        self.params = upload_struct(self.table.params, dev)
        self.rules = upload_struct(self.table.rules, dev)
        self.n_params = len(self.table.params)
        self.n_rules = len(self.table.rules)


def _expand(topology: ModelTopology, tables: _DeviceTables, unit_bits: torch.Tensor,
            n_workers: int, dev: torch.device, *, want_param_masks: bool = False,
            want_stats: bool = True, want_owner: bool = True, want_counts: bool | None = None):
    """Run k_build_masks; returns dict of device tensors.  want_stats: the
    [d] coverage / divisor / governors tables (25 B per parameter);
    want_counts (default: with the stats): per-worker active counts."""
    d = topology.total
    mb = mask_bytes_for(n_workers)
    out = {}
    if want_owner:
        out["owner_mask"] = torch.empty(d, dtype=MASK_TORCH_DTYPE[mb], device=dev)
    if want_param_masks:
        out["param_masks"] = torch.empty((n_workers, d), dtype=torch.bool, device=dev)
    if want_stats:
        out["coverage"] = torch.empty(d, dtype=torch.int64, device=dev)
        out["divisor"] = torch.empty(d, dtype=torch.float64, device=dev)
        out["governors"] = torch.empty(d, dtype=torch.int64, device=dev)
    if want_stats if want_counts is None else want_counts:
        out["active_counts"] = torch.zeros(n_workers, dtype=torch.int64, device=dev)
    ub = unit_bits if unit_bits.numel() else torch.zeros(1, dtype=torch.int64, device=dev)
    N.call("sdp_build_masks", ptr(tables.params), tables.n_params, ptr(tables.rules),
           tables.n_rules, ptr(ub), n_workers, d, ptr(out.get("owner_mask")), mb,
           ptr(out.get("param_masks")), ptr(out.get("coverage")), ptr(out.get("divisor")),
           ptr(out.get("governors")), ptr(out.get("active_counts")), stream_ptr(dev))
    return out


def _unit_bits_from_active(table: UnitTable, topology: ModelTopology, active: dict,
                           n_workers: int) -> np.ndarray:
    """Unit owner bits from explicit per-layer / per-block activity flags."""
    bits = np.full(table.n_units, (1 << n_workers) - 1 if n_workers < 64 else -1, dtype=np.int64)
    weights = (np.uint64(1) << np.arange(n_workers, dtype=np.uint64))
    for key, flags in active.items():
        f = np.asarray(flags, dtype=bool)
        packed = (f.astype(np.uint64) * weights[:, None]).sum(axis=0, dtype=np.uint64)
        if table.strategy == "neuron":
            base = table.layer_base[key]
            bits[base:base + f.shape[1]] = packed.view(np.int64)
        else:
            bits[table.block_unit[key]] = packed.view(np.int64)[0]
    return bits


def induce_channel_param_mask(topology: ModelTopology, channel_active: dict,
                              device_=None) -> torch.Tensor:
    """[N, C] channel flags per layer -> [N, d] bool device mask (masking.py:120-150)."""
    known = {layer.layer_id for layer in topology.channel_layers}
    for layer_id in channel_active:
        if layer_id not in known:
            raise TopologyError(f"channel mask refers to undeclared layer {layer_id!r}")
    n_workers = next(iter(channel_active.values())).shape[0] if channel_active else 1
    dev = device(device_)
    # every declared layer named in channel_active governs its slices, maskable or not
    layers = [layer for layer in topology.channel_layers if layer.layer_id in channel_active]
    for layer in layers:
        if np.asarray(channel_active[layer.layer_id]).shape[1] != layer.channels:
            raise TopologyError(
                f"mask for {layer.layer_id} has {np.asarray(channel_active[layer.layer_id]).shape[1]} "
                f"channels, layer has {layer.channels}")
    sub = _SubsetTopology(topology, {lay.layer_id for lay in layers})
    tables = _DeviceTables(sub, "neuron", dev)
    flags = {lid: channel_active[lid] for lid in tables.table.layer_base}
    ub = torch.from_numpy(_unit_bits_from_active(tables.table, topology, flags, n_workers)).to(dev)
    return _expand(topology, tables, ub, n_workers, dev, want_param_masks=True,
                   want_stats=False)["param_masks"]


def induce_block_param_mask(topology: ModelTopology, block_active, device_=None) -> torch.Tensor:
    """[N, K] block flags -> [N, d] bool device mask (masking.py:153-170)."""
    ba = np.asarray(block_active, dtype=bool)
    n_workers, n_blocks = ba.shape
    if n_blocks != len(topology.blocks):
        raise TopologyError(
            f"block mask covers {n_blocks} blocks, topology declares {len(topology.blocks)}")
    for block in topology.blocks:
        if (~ba[:, block.index]).any() and not (block.maskable and block.has_skip):
            raise ConfigError(
                f"block {block.block_id} has no skip connection and cannot be masked")
    dev = device(device_)
    sub = _SubsetTopology(topology, None, blocks_any=True)
    tables = _DeviceTables(sub, "block", dev)
    flags = {b.block_id: ba[:, b.index][:, None] for b in topology.blocks if b.block_id in tables.table.block_unit}
    ub = torch.from_numpy(_unit_bits_from_active(tables.table, topology, flags, n_workers)).to(dev)
    return _expand(topology, tables, ub, n_workers, dev, want_param_masks=True,
                   want_stats=False)["param_masks"]


class _SubsetTopology:
    """View of a topology where a chosen set of channel layers (or every block)
    counts as maskable -- the induce_* functions expand exactly the flags they
    are given, maskable or not (masking.py:132-149, 161-169)."""

    def __init__(self, topo: ModelTopology, layer_ids, blocks_any: bool = False):
        from dataclasses import replace
        self.params = topo.params
        self.index = topo.index
        self.total = topo.total
        self.channel_layers = tuple(
            replace(lay, maskable=(layer_ids is not None and lay.layer_id in layer_ids))
            for lay in topo.channel_layers)
        self.blocks = tuple(replace(b, maskable=True) for b in topo.blocks) if blocks_any else topo.blocks


# ---------------------------------------------------------------------------
# MaskAssignment
# ---------------------------------------------------------------------------

class WorkerMaskView:
    """Everything one worker needs to run a masked forward pass (masking.py:173-185).

    worker_id, channel_active (layer id -> read-only numpy bool [C]) and
    block_active (read-only numpy bool [num_blocks]) are built at once; the
    per-parameter masks param_mask (float64 [d], 0.0 / 1.0) and
    param_mask_bool (bool [d]) are device tensors expanded by libsdp's
    sdp_worker_mask on first access (9 B per parameter that a trainer, which
    only needs the block / channel flags, never allocates)."""

    __slots__ = ("worker_id", "channel_active", "block_active", "_owner_mask", "_mask_bytes", "_pm", "_pmb")

    def __init__(self, worker_id, channel_active, block_active, *, owner_mask=None, mask_bytes=1,
                 param_mask=None, param_mask_bool=None):
        self.worker_id = worker_id
        self.channel_active = channel_active
        self.block_active = block_active
        self._owner_mask, self._mask_bytes = owner_mask, mask_bytes
        self._pm, self._pmb = param_mask, param_mask_bool

    def _expand(self) -> None:
        d = self._owner_mask.numel()
        dev = self._owner_mask.device
        mf = torch.empty(d, dtype=torch.float64, device=dev)
        mu = torch.empty(d, dtype=torch.uint8, device=dev)
        N.call("sdp_worker_mask", ptr(self._owner_mask), self._mask_bytes, d, self.worker_id, ptr(mf),
               ptr(mu), stream_ptr(dev))
        self._pm, self._pmb = read_only(mf), read_only(mu.view(torch.bool))

    @property
    def param_mask(self) -> torch.Tensor:
        if self._pm is None:
            self._expand()
        return self._pm

    @property
    def param_mask_bool(self) -> torch.Tensor:
        if self._pmb is None:
            self._expand()
        return self._pmb

    @property
    def active_params(self) -> int:
        return int(self.param_mask_bool.sum().item())


class MaskAssignment:
    """Unit-to-worker assignment plus induced masks, resident on the GPU
    (masking.py:188-269)."""

    def __init__(self, n_workers, replication, strategy, seed, topology, unit_workers,
                 param_masks, governors, *, _tables=None, _owner_mask=None, _coverage=None,
                 _divisor=None, _active_counts=None, _unit_bits=None, _device=None):
        self.n_workers = int(n_workers)
        self.replication = int(replication)
        self.strategy = strategy
        self.seed = int(seed)
        self.topology = topology
        self._unit_workers = unit_workers
        self._unit_bits = _unit_bits
        self._tables = _tables
        if _owner_mask is None:
            # explicit [N, d] masks (tests, hand-built assignments): pack on device
            pm = torch.as_tensor(np.asarray(param_masks) if not torch.is_tensor(param_masks) else param_masks)
            dev = device(pm.device if pm.is_cuda else _device)
            pm = pm.to(dev, dtype=torch.bool)
            mb = mask_bytes_for(self.n_workers)
            packed = torch.zeros(pm.shape[1], dtype=torch.int64, device=dev)
            for w in range(self.n_workers):
                packed |= pm[w].to(torch.int64) << w
            self.owner_mask = packed.to(MASK_TORCH_DTYPE[mb]) if mb < 8 else packed
            self._param_masks = pm
            self._coverage = pm.sum(dim=0, dtype=torch.int64)
            self._divisor = self._coverage.clamp(min=1).to(torch.float64)
            self._governors = torch.as_tensor(np.asarray(governors) if not torch.is_tensor(governors)
                                              else governors).to(dev, dtype=torch.int64)
            self._active_counts = pm.sum(dim=1, dtype=torch.int64)
        else:
            # built on the device: only the 1-byte-per-parameter owner mask and
            # the per-worker counts exist up front; the 25 B/parameter coverage /
            # divisor / governors tables are expanded on first use (a training
            # rank never needs them -- they were 3 GB per GPT-2 rank)
            self.owner_mask = _owner_mask
            self._param_masks = param_masks
            self._coverage = _coverage
            self._divisor = _divisor
            self._governors = governors
            self._active_counts = _active_counts
        # the reference freezes these (masking.py:206-207): read-only views
        self.owner_mask = read_only(self.owner_mask)
        self.mask_bytes = mask_bytes_for(self.n_workers)
        self._uncovered = None
        self._plans: dict = {}

    # -- reference attributes ------------------------------------------------
    @property
    def device(self) -> torch.device:
        return self.owner_mask.device

    def _stats(self) -> None:
        if self._coverage is None or self._divisor is None or self._governors is None:
            out = _expand(self.topology, self._tables, self._unit_bits, self.n_workers, self.device,
                          want_owner=False, want_stats=True, want_counts=False)
            self._coverage, self._divisor, self._governors = out["coverage"], out["divisor"], out["governors"]

    @property
    def coverage(self) -> torch.Tensor:
        """int64 [d] owner count per parameter (masking.py:203)."""
        self._stats()
        return read_only(self._coverage)

    @property
    def divisor(self) -> torch.Tensor:
        """float64 [d] max(coverage, 1) (masking.py:204)."""
        self._stats()
        return read_only(self._divisor)

    @property
    def governors(self) -> torch.Tensor:
        """int64 [d] number of units governing each parameter (masking.py:288-302)."""
        self._stats()
        return read_only(self._governors)

    @property
    def unit_workers(self) -> dict[StructuralUnit, tuple[int, ...]]:
        if self._unit_workers is None:
            bits = self._unit_bits.cpu().numpy().view(np.uint64)
            keys = self._tables.table.keys
            groups = self._tables.table.groups
            uw = {}
            for first, size in groups:
                for u in range(first, first + size):
                    uw[StructuralUnit.from_key(keys[u])] = _bits_to_workers(int(bits[u]), self.n_workers)
            self._unit_workers = uw
        return self._unit_workers

    @property
    def param_masks(self) -> torch.Tensor:
        """[N, d] bool (reference layout); materialised on first use."""
        if self._param_masks is None:
            self._param_masks = _expand(self.topology, self._tables, self._unit_bits, self.n_workers,
                                        self.device, want_param_masks=True,
                                        want_stats=False)["param_masks"]
        return read_only(self._param_masks)

    @property
    def always_active(self) -> torch.Tensor:
        return self.governors == 0

    @property
    def dp_equivalent(self) -> bool:
        return self.replication == self.n_workers

    @property
    def uncovered_params(self) -> int:
        if self._uncovered is None:
            self._uncovered = int((self.owner_mask == 0).sum().item())
        return self._uncovered

    def owned_total(self) -> int:
        """sum_j |O_j| -- replica elements one sync reads (cached; the per-worker
        held counts sum to it, masking.py:442)."""
        if getattr(self, "_owned_total", None) is None:
            self._owned_total = int(self._active_counts.sum().item())
        return self._owned_total

    def host_divisor(self) -> np.ndarray:
        """Read-only numpy copy of `divisor` (cached; the reference's type)."""
        if getattr(self, "_host_divisor", None) is None:
            hd = self.divisor.cpu().numpy()
            hd.setflags(write=False)
            self._host_divisor = hd
        return self._host_divisor

    def active_param_counts(self) -> list[int]:
        return [int(x) for x in self._active_counts.cpu().tolist()]

    def worker_view(self, worker_id: int) -> WorkerMaskView:
        if not 0 <= worker_id < self.n_workers:
            raise ConfigError(f"worker id {worker_id} outside [0, {self.n_workers})")
        channel_active = {layer.layer_id: np.ones(layer.channels, dtype=bool)
                          for layer in self.topology.channel_layers}
        block_active = np.ones(len(self.topology.blocks), dtype=bool)
        block_index = {b.block_id: b.index for b in self.topology.blocks}
        for unit, workers in self.unit_workers.items():
            if unit.kind == KIND_CHANNEL:
                channel_active[unit.ref][unit.index] = worker_id in workers
            else:
                block_active[block_index[unit.ref]] = worker_id in workers
        for arr in channel_active.values():
            arr.setflags(write=False)
        block_active.setflags(write=False)
        return WorkerMaskView(worker_id, channel_active, block_active, owner_mask=self.owner_mask,
                              mask_bytes=self.mask_bytes)

    def worker_views(self) -> list[WorkerMaskView]:
        return [self.worker_view(i) for i in range(self.n_workers)]

    def unit_counts(self) -> list[int]:
        counts = [0] * self.n_workers
        for workers in self.unit_workers.values():
            for i in workers:
                counts[i] += 1
        return counts

    def output_fraction(self, layer_id: str) -> float:
        if self.strategy != "neuron":
            return 1.0
        layer = self.topology.channel_layer(layer_id)
        if not layer.maskable:
            return 1.0
        active = np.zeros(self.n_workers)
        for unit, workers in self.unit_workers.items():
            if unit.kind == KIND_CHANNEL and unit.ref == layer_id:
                for i in workers:
                    active[i] += 1
        return float(active.mean() / layer.channels)

    # -- B200 additions ------------------------------------------------------
    def sync_plan(self, **kw):
        """Tile plan of the owner-subset sync for this assignment (cached)."""
        from .engine import SyncPlan
        key = tuple(sorted(kw.items()))
        if key not in self._plans:
            self._plans[key] = SyncPlan(self, **kw)
        return self._plans[key]


def _reference_module(name: str):
    """subnetdp.<name> of the reference package, when the caller has it."""
    import importlib
    try:
        return importlib.import_module(f"subnetdp.{name}")
    except ImportError as exc:
        raise UsageError("the reference package `subnetdp` is not importable here") from exc


def is_reference_assignment(obj) -> bool:
    """A reference MaskAssignment (numpy arrays, masking.py:188-207)."""
    return not isinstance(obj, MaskAssignment) and hasattr(obj, "param_masks") \
        and isinstance(getattr(obj, "param_masks"), np.ndarray)


_FROM_REF: dict = {}


def from_reference(ref, device_=None) -> MaskAssignment:
    """A reference MaskAssignment as a device one: its [N, d] masks packed into
    the per-element owner bitmask on the GPU, governors and unit_workers kept.
    Cached per reference object (the reference freezes its arrays,
    masking.py:206-207, so the cache can never go stale)."""
    import weakref
    key = id(ref)
    hit = _FROM_REF.get(key)
    if hit is not None and hit[0]() is ref:
        return hit[1]
    uw = {StructuralUnit.from_key(u.key()): tuple(w) for u, w in ref.unit_workers.items()}
    ours = MaskAssignment(ref.n_workers, ref.replication, ref.strategy, ref.seed, ref.topology, uw,
                          np.asarray(ref.param_masks), np.asarray(ref.governors), _device=device(device_))
    try:
        wr = weakref.ref(ref, lambda _, k=key: _FROM_REF.pop(k, None))
    except TypeError:  # not weak-referenceable: no caching
        return ours
    _FROM_REF[key] = (wr, ours)
    return ours


def reference_topology(topology):
    """`topology` declared through the reference's own types (field-for-field
    equal dataclasses, reference topology.py:16-84)."""
    T = _reference_module("topology")
    if isinstance(topology, T.ModelTopology):
        return topology
    return T.ModelTopology(
        params=tuple(T.ParamSpec(p.name, tuple(p.shape), p.offset, p.size, p.kind, p.layer_id)
                     for p in topology.params),
        channel_layers=tuple(T.ChannelLayerSpec(c.layer_id, c.channels, c.norm_groups, c.maskable,
                                                tuple(c.own_slices), tuple(c.consumer_slices))
                             for c in topology.channel_layers),
        blocks=tuple(T.BlockSpec(b.block_id, b.index, tuple(b.param_names), b.has_skip, b.maskable,
                                 b.activation_per_sample) for b in topology.blocks),
        base_activation_per_sample=topology.base_activation_per_sample,
        input_shape=tuple(topology.input_shape),
        default_alignment_layer=topology.default_alignment_layer)


def to_reference(assignment: MaskAssignment, topology=None):
    """The GPU-built assignment as the reference's own MaskAssignment (numpy,
    frozen by its constructor, masking.py:188-207), for callers that hand it to
    the reference's loop (validate, masked_kaiming_init, worker_view,
    save_assignment; engine.py:167-185).  `topology`: the caller's reference
    topology object (default: this assignment's, converted)."""
    M = _reference_module("masking")
    topo = reference_topology(assignment.topology if topology is None else topology)
    uw = {M.StructuralUnit.from_key(u.key()): tuple(w) for u, w in assignment.unit_workers.items()}
    return M.MaskAssignment(
        n_workers=assignment.n_workers, replication=assignment.replication, strategy=assignment.strategy,
        seed=assignment.seed, topology=topo, unit_workers=uw,
        param_masks=assignment.param_masks.cpu().numpy(), governors=assignment.governors.cpu().numpy())


def build_assignment(topology: ModelTopology, strategy: str, n_workers: int, replication: int,
                     seed: int, device_=None) -> MaskAssignment:
    """Construct the full per-worker mask set on the GPU (masking.py:305-359)."""
    if strategy not in STRATEGIES:
        raise ConfigError(f"strategy must be one of {STRATEGIES}, got {strategy!r}")
    _check_replication(n_workers, replication)
    dev = device(device_)
    tables = _DeviceTables(topology, strategy, dev)
    t = tables.table
    if not t.groups:
        if strategy == "neuron":
            raise ConfigError("model declares no maskable channels for neuron masking")
        raise ConfigError("model declares no maskable blocks for block masking")
    if strategy == "block":
        for b in topology.blocks:
            if b.maskable and not b.has_skip and replication < n_workers:
                raise ConfigError(f"block {b.block_id} has no skip connection and cannot be masked")
    if any(size == 0 for _, size in t.groups):
        raise ConfigError("assign_grouped_units requires non-empty groups")
    unit_bits = _device_assign(t.groups, t.n_units, n_workers, replication, seed, dev)
    out = _expand(topology, tables, unit_bits, n_workers, dev, want_stats=False, want_counts=True)
    return MaskAssignment(
        n_workers, replication, strategy, seed, topology, None, None, None,
        _tables=tables, _owner_mask=out["owner_mask"], _active_counts=out["active_counts"],
        _unit_bits=unit_bits)


@dataclass
class MaskValidationReport:
    n_workers: int
    replication: int
    strategy: str
    dp_equivalent: bool
    unit_counts: list[int]
    active_param_counts: list[int]
    uncovered_params: int

    def to_dict(self) -> dict:
        return dict(self.__dict__)


def validate(assignment: MaskAssignment) -> MaskValidationReport:
    """Every assignment invariant (masking.py:384-444); reductions run on device."""
    errors: list[str] = []
    n, p = assignment.n_workers, assignment.replication
    topo = assignment.topology
    for unit, workers in assignment.unit_workers.items():
        if len(set(workers)) != p:
            errors.append(f"unit {unit.key()} is held by {len(set(workers))} workers, expected {p}")
        if any(not 0 <= w < n for w in workers):
            errors.append(f"unit {unit.key()} names a worker outside [0, {n})")
    cov, gov = assignment.coverage, assignment.governors
    always, single = gov == 0, gov == 1
    if bool(always.any()) and not bool((cov[always] == n).all()):
        errors.append("an always-active parameter is missing from some worker mask")
    if bool(single.any()) and not bool((cov[single] == p).all()):
        bad = int((cov[single] != p).sum().item())
        errors.append(f"{bad} unit-governed parameters have coverage != {p}")
    if bool((cov[gov < 2] == 0).any()):
        errors.append("a parameter governed by at most one unit has zero coverage")
    counts = assignment.unit_counts()
    if counts and max(counts) - min(counts) > 1:
        errors.append(f"per-worker unit loads are unbalanced: {counts}")
    if assignment.strategy == "neuron":
        views = [assignment.worker_view(i) for i in range(n)]
        for layer in topo.channel_layers:
            gsize = layer.channels // layer.norm_groups
            for view in views:
                act = view.channel_active[layer.layer_id]
                for g in range(layer.norm_groups):
                    if not act[g * gsize:(g + 1) * gsize].any():
                        errors.append(f"layer {layer.layer_id} group {g} has no active channel "
                                      f"on worker {view.worker_id}")
    else:
        maskable = [b.index for b in topo.blocks if b.maskable]
        if maskable:
            for i in range(n):
                view = assignment.worker_view(i)
                if not view.block_active[maskable].any():
                    errors.append(f"worker {view.worker_id} holds no active block")
    if errors:
        raise ValidationError("; ".join(errors))
    return MaskValidationReport(n, p, assignment.strategy, assignment.dp_equivalent, counts,
                                assignment.active_param_counts(), assignment.uncovered_params)


def assignment_to_dict(assignment: MaskAssignment) -> dict:
    return {
        "version": 1,
        "n_workers": assignment.n_workers,
        "replication": assignment.replication,
        "strategy": assignment.strategy,
        "seed": assignment.seed,
        "units": {u.key(): list(w) for u, w in assignment.unit_workers.items()},
    }


def save_assignment(assignment: MaskAssignment, path) -> None:
    Path(path).write_text(json.dumps(assignment_to_dict(assignment), indent=2, sort_keys=True))


def assignment_from_dict(doc: dict, topology: ModelTopology, device_=None) -> MaskAssignment:
    """masks.json -> device tables: unit bits from the document, then k_build_masks
    (masking.py:462-499)."""
    strategy = doc["strategy"]
    if strategy not in STRATEGIES:
        raise ConfigError(f"strategy must be one of {STRATEGIES}, got {strategy!r}")
    n_workers = int(doc["n_workers"])
    dev = device(device_)
    tables = _DeviceTables(topology, strategy, dev)
    t = tables.table
    full = (1 << n_workers) - 1
    bits = np.array([full] * t.n_units, dtype=np.uint64)
    unit_workers = {}
    for key, workers in doc["units"].items():
        unit = StructuralUnit.from_key(key)
        ws = tuple(sorted(int(w) for w in workers))
        if strategy == "neuron":
            if unit.ref not in t.layer_base:
                raise TopologyError(f"unit {key} refers to a non-maskable or unknown layer")
            channels = topology.channel_layer(unit.ref).channels
            idx = unit.index
            # numpy indexing semantics of the reference (masking.py:479):
            # negative indices wrap, anything outside [-C, C) is an IndexError
            if not -channels <= idx < channels:
                raise IndexError(f"unit {key}: index {idx} is out of bounds for layer "
                                 f"{unit.ref} with {channels} channels")
            uid = t.layer_base[unit.ref] + idx % channels
        else:
            if unit.ref not in t.block_unit:
                raise TopologyError(f"unit {key} refers to an unknown block")
            uid = t.block_unit[unit.ref]
        b = 0
        for w in ws:
            if 0 <= w < n_workers:  # the reference only deactivates workers in range(n)
                b |= 1 << w
        bits[uid] = b
        unit_workers[unit] = ws
    ub = torch.from_numpy(bits.view(np.int64)).to(dev)
    out = _expand(topology, tables, ub, n_workers, dev, want_stats=False, want_counts=True)
    return MaskAssignment(
        n_workers, int(doc["replication"]), strategy, int(doc.get("seed", 0)), topology,
        unit_workers, None, None, _tables=tables, _owner_mask=out["owner_mask"],
        _active_counts=out["active_counts"], _unit_bits=ub)


def load_assignment(path, topology: ModelTopology, device_=None) -> MaskAssignment:
    return assignment_from_dict(json.loads(Path(path).read_text()), topology, device_)
