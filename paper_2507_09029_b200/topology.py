"""Topology descriptors: the same types the reference's masking consumes
(topology.py:16-97), plus their lowering into libsdp's descriptor tables.

`ParamSpec` / `ChannelLayerSpec` / `BlockSpec` / `ModelTopology` /
`GlobalModel` keep the reference's field names and invariants (contiguous
in-order tiling of the flat vector, topology.py:66-74), so a reference
topology object can be passed to this package unchanged.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError, TopologyError


@dataclass(frozen=True)
class ParamSpec:
    name: str
    shape: tuple[int, ...]
    offset: int
    size: int
    kind: str      # conv_w | linear_w | bias | gamma | beta | embed | norm_w | norm_b
    layer_id: str  # channel layer that owns the output units


@dataclass(frozen=True)
class ChannelLayerSpec:
    """A layer whose output channels are structural units.

    own_slices: (param, axis) entries indexed by this layer's channel mask;
    consumer_slices: downstream (param, axis) entries that die with a channel.
    """

    layer_id: str
    channels: int
    norm_groups: int
    maskable: bool
    own_slices: tuple[tuple[str, int], ...]
    consumer_slices: tuple[tuple[str, int], ...]


@dataclass(frozen=True)
class BlockSpec:
    block_id: str
    index: int
    param_names: tuple[str, ...]
    has_skip: bool
    maskable: bool
    activation_per_sample: int


@dataclass
class ModelTopology:
    params: tuple[ParamSpec, ...]
    channel_layers: tuple[ChannelLayerSpec, ...]
    blocks: tuple[BlockSpec, ...]
    base_activation_per_sample: int
    input_shape: tuple[int, ...]
    default_alignment_layer: str
    index: dict[str, ParamSpec] = field(init=False)
    total: int = field(init=False)

    def __post_init__(self):
        self.index = {p.name: p for p in self.params}
        self.total = int(sum(p.size for p in self.params))
        pos = 0
        for p in self.params:
            if p.offset != pos:
                raise ValueError(
                    f"parameter specs must tile the flat vector in order; {p.name} starts at "
                    f"{p.offset}, expected {pos}")
            pos += p.size

    def slice_of(self, name: str) -> slice:
        p = self.index[name]
        return slice(p.offset, p.offset + p.size)

    def channel_layer(self, layer_id: str) -> ChannelLayerSpec:
        for layer in self.channel_layers:
            if layer.layer_id == layer_id:
                return layer
        raise KeyError(layer_id)


@dataclass
class GlobalModel:
    """Architecture + topology + the flat parameter vector (a device tensor)."""

    arch: object
    topology: ModelTopology
    theta: object

    def param_view(self, name: str):
        p = self.topology.index[name]
        return self.theta[p.offset:p.offset + p.size].reshape(p.shape)


class TopologyBuilder:
    """Appends ParamSpecs contiguously (the flat layout every table indexes)."""

    def __init__(self):
        self.specs: list[ParamSpec] = []
        self.offset = 0

    def add(self, name: str, shape: tuple[int, ...], kind: str, layer_id: str) -> None:
        n = int(math.prod(shape))
        self.specs.append(ParamSpec(name, tuple(int(s) for s in shape), self.offset, n, kind, layer_id))
        self.offset += n


# ---------------------------------------------------------------------------
# lowering to libsdp descriptor tables
# ---------------------------------------------------------------------------

@dataclass
class UnitTable:
    """Structural units of one strategy, numbered densely.

    neuron: the channels of every maskable channel layer, layer-major
            (masking.py:272-285 orders the assignment groups the same way);
    block:  the maskable blocks in topology order (masking.py:335-339).
    """

    strategy: str
    keys: list[str]                       # StructuralUnit.key() per unit id
    layer_base: dict[str, int]            # neuron: first unit id of each layer
    block_unit: dict[str, int]            # block: unit id of each block
    groups: list[tuple[int, int]]         # (first_unit, size) drawn in order
    params: np.ndarray                    # structured array of ParamDesc fields
    rules: np.ndarray                     # structured array of RuleDesc fields

    @property
    def n_units(self) -> int:
        return len(self.keys)


PARAM_DTYPE = np.dtype([("offset", "<i8"), ("size", "<i8"), ("rule_begin", "<i4"), ("rule_count", "<i4")])
RULE_DTYPE = np.dtype([("inner", "<i4"), ("dim", "<i4"), ("unit_base", "<i4"),
                       ("inner_mul", "<u4"), ("inner_shr", "<u4"), ("dim_mul", "<u4"),
                       ("dim_shr", "<u4"), ("pad_", "<i4")])


def fast_divisor(d: int) -> tuple[int, int]:
    """(mul, shr) with n // d == umulhi(n, mul) >> shr for 0 <= n < 2**31
    (mul = 0 encodes d == 1)."""
    if d == 1:
        return 0, 0
    p = 31 + (d - 1).bit_length()
    return ((1 << p) + d - 1) // d, p - 32


def unit_table(topology: ModelTopology, strategy: str) -> UnitTable:
    """Lower a topology into the per-parameter rule lists k_build_masks reads.

    Every (layer, param, axis) own/consumer entry (masking.py:140-149) and every
    maskable block's parameter (masking.py:167-169) becomes one rule; the rule
    count of a parameter is exactly its governor count (masking.py:288-302).
    """
    keys: list[str] = []
    layer_base: dict[str, int] = {}
    block_unit: dict[str, int] = {}
    groups: list[tuple[int, int]] = []
    per_param: dict[str, list[tuple[int, int, int]]] = {p.name: [] for p in topology.params}
    if strategy == "neuron":
        for layer in topology.channel_layers:
            if not layer.maskable:
                continue
            base = len(keys)
            layer_base[layer.layer_id] = base
            keys.extend(f"channel:{layer.layer_id}:{c}" for c in range(layer.channels))
            gsize = layer.channels // layer.norm_groups
            groups.extend((base + g * gsize, gsize) for g in range(layer.norm_groups))
            for pname, axis in tuple(layer.own_slices) + tuple(layer.consumer_slices):
                spec = topology.index.get(pname)
                if spec is None:
                    raise TopologyError(
                        f"layer {layer.layer_id} references unknown parameter {pname!r}")
                if not 0 <= axis < len(spec.shape):
                    raise TopologyError(f"axis {axis} out of range for {pname} {spec.shape}")
                if spec.shape[axis] != layer.channels:
                    raise TopologyError(
                        f"{pname} axis {axis} has {spec.shape[axis]} entries, layer "
                        f"{layer.layer_id} has {layer.channels} channels")
                inner = int(math.prod(spec.shape[axis + 1:]))
                per_param[pname].append((inner, int(spec.shape[axis]), base))
    elif strategy == "block":
        for block in topology.blocks:
            if not block.maskable:
                continue
            uid = len(keys)
            block_unit[block.block_id] = uid
            keys.append(f"block:{block.block_id}")
            for pname in block.param_names:
                if pname not in per_param:
                    raise TopologyError(f"block {block.block_id} names unknown parameter {pname!r}")
                per_param[pname].append((1, 1, uid))
        if keys:
            groups = [(0, len(keys))]
    else:
        raise ConfigError(f"strategy must be one of ('neuron', 'block'), got {strategy!r}")

    params = np.zeros(len(topology.params), dtype=PARAM_DTYPE)
    rules_list: list[tuple[int, int, int, int]] = []
    for i, p in enumerate(topology.params):
        rs = per_param[p.name]
        if p.size >= 2**31:
            raise TopologyError(f"parameter {p.name} exceeds 2^31 elements")
        params[i] = (p.offset, p.size, len(rules_list), len(rs))
        rules_list.extend((inner, dim, base, *fast_divisor(inner), *fast_divisor(dim), 0)
                          for inner, dim, base in rs)
    rules = np.array(rules_list if rules_list else [(1, 1, 0, 0, 0, 0, 0, 0)], dtype=RULE_DTYPE)
    return UnitTable(strategy, keys, layer_base, block_unit, groups, params, rules)
