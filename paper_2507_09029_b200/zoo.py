"""Topology declarations for the benchmark configurations (BASELINE.json).

  mini_resnet_topology / residual_mlp_topology
      the reference's desk-scale models, declared parameter-for-parameter as
      models.py:67-145 and :190-246 declare them (config C1 and the parity
      tests use these).
  resnet18_cifar_topology
      ResNet-18, CIFAR stem (3x3 conv, no max-pool), GroupNorm(2) affine
      params; the 3 downsampling BasicBlocks are not maskable,
      the other 5 are (configs C2/C3).  d = 11,173,962.
  gpt2_small_topology
      GPT-2 small (124M, tied head): 12 pre-LN blocks, each maskable with its
      residual skip; the MLP hidden units are the width-wise channel units
      (config C4).  d = 124,439,808.
  sweep_topology
      config C5: 1% always-active prefix + 64 equal maskable blocks.
"""

from __future__ import annotations

from .errors import ConfigError
from .topology import BlockSpec, ChannelLayerSpec, ModelTopology, TopologyBuilder


def mini_resnet_topology(channels: int, blocks: int, classes: int, norm_groups: int = 2,
                         in_channels: int = 3, image_hw=(8, 8)) -> ModelTopology:
    if blocks < 1:
        raise ConfigError(f"mini resnet needs at least one block, got {blocks}")
    if channels % norm_groups:
        raise ConfigError(f"{norm_groups} norm groups do not divide {channels} channels")
    c, k, m = channels, blocks, classes
    h, w = image_hw
    tb = TopologyBuilder()
    tb.add("stem.w", (c, in_channels, 3, 3), "conv_w", "stem")
    for nm, kind in (("stem.b", "bias"), ("stem_gn.gamma", "gamma"), ("stem_gn.beta", "beta")):
        tb.add(nm, (c,), kind, "stem")
    layers = [ChannelLayerSpec("stem", c, norm_groups, False,
                               (("stem.w", 0), ("stem.b", 0), ("stem_gn.gamma", 0), ("stem_gn.beta", 0)), ())]
    blocks_ = []
    for i in range(k):
        names = []
        for conv, gn in (("conv1", "gn1"), ("conv2", "gn2")):
            lid = f"block{i}.{conv}"
            tb.add(f"{lid}.w", (c, c, 3, 3), "conv_w", lid)
            tb.add(f"{lid}.b", (c,), "bias", lid)
            tb.add(f"block{i}.{gn}.gamma", (c,), "gamma", lid)
            tb.add(f"block{i}.{gn}.beta", (c,), "beta", lid)
            names += [f"{lid}.w", f"{lid}.b", f"block{i}.{gn}.gamma", f"block{i}.{gn}.beta"]
            own = ((f"{lid}.w", 0), (f"{lid}.b", 0), (f"block{i}.{gn}.gamma", 0), (f"block{i}.{gn}.beta", 0))
            consumer = ((f"block{i}.conv2.w", 1),) if conv == "conv1" else ()
            layers.append(ChannelLayerSpec(lid, c, norm_groups, True, own, consumer))
        blocks_.append(BlockSpec(f"block{i}", i, tuple(names), True, True, 6 * c * h * w))
    tb.add("head.w", (m, c), "linear_w", "head")
    tb.add("head.b", (m,), "bias", "head")
    layers.append(ChannelLayerSpec("head", m, 1, False, (("head.w", 0), ("head.b", 0)), ()))
    return ModelTopology(tuple(tb.specs), tuple(layers), tuple(blocks_), 3 * c * h * w + c + m,
                         (in_channels, h, w), f"block{k // 2}.conv2.w")


def residual_mlp_topology(width: int, blocks: int, classes: int, in_dim: int = 16) -> ModelTopology:
    if blocks < 1:
        raise ConfigError(f"residual mlp needs at least one block, got {blocks}")
    w, k, m = width, blocks, classes
    tb = TopologyBuilder()
    tb.add("stem.w", (w, in_dim), "linear_w", "stem")
    tb.add("stem.b", (w,), "bias", "stem")
    layers = [ChannelLayerSpec("stem", w, 1, False, (("stem.w", 0), ("stem.b", 0)), ())]
    blocks_ = []
    for i in range(k):
        for lin in ("lin1", "lin2"):
            tb.add(f"block{i}.{lin}.w", (w, w), "linear_w", f"block{i}.{lin}")
            tb.add(f"block{i}.{lin}.b", (w,), "bias", f"block{i}.{lin}")
        # only the hidden units are structural (no norm after lin2)
        layers.append(ChannelLayerSpec(f"block{i}.lin1", w, 1, True,
                                       ((f"block{i}.lin1.w", 0), (f"block{i}.lin1.b", 0)),
                                       ((f"block{i}.lin2.w", 1),)))
        layers.append(ChannelLayerSpec(f"block{i}.lin2", w, 1, False,
                                       ((f"block{i}.lin2.w", 0), (f"block{i}.lin2.b", 0)), ()))
        blocks_.append(BlockSpec(f"block{i}", i, (f"block{i}.lin1.w", f"block{i}.lin1.b",
                                                  f"block{i}.lin2.w", f"block{i}.lin2.b"),
                                 True, True, 4 * w))
    tb.add("head.w", (m, w), "linear_w", "head")
    tb.add("head.b", (m,), "bias", "head")
    layers.append(ChannelLayerSpec("head", m, 1, False, (("head.w", 0), ("head.b", 0)), ()))
    return ModelTopology(tuple(tb.specs), tuple(layers), tuple(blocks_), 2 * w + m, (in_dim,),
                         f"block{k // 2}.lin1.w")


def resnet18_cifar_topology(classes: int = 10, norm_groups: int = 2, image_hw=(32, 32)) -> ModelTopology:
    h, w = image_hw
    tb = TopologyBuilder()
    tb.add("conv1.w", (64, 3, 3, 3), "conv_w", "stem")
    tb.add("gn1.gamma", (64,), "gamma", "stem")
    tb.add("gn1.beta", (64,), "beta", "stem")
    layers = [ChannelLayerSpec("stem", 64, norm_groups, False,
                               (("conv1.w", 0), ("gn1.gamma", 0), ("gn1.beta", 0)), ())]
    blocks_ = []
    cin, bi, hw = 64, 0, h * w
    for stage, planes in enumerate((64, 128, 256, 512), start=1):
        for j in range(2):
            stride = 2 if (stage > 1 and j == 0) else 1
            if stride == 2:
                hw //= 4
            p = f"layer{stage}.{j}"
            names = []
            tb.add(f"{p}.conv1.w", (planes, cin, 3, 3), "conv_w", f"{p}.conv1")
            tb.add(f"{p}.gn1.gamma", (planes,), "gamma", f"{p}.conv1")
            tb.add(f"{p}.gn1.beta", (planes,), "beta", f"{p}.conv1")
            tb.add(f"{p}.conv2.w", (planes, planes, 3, 3), "conv_w", f"{p}.conv2")
            tb.add(f"{p}.gn2.gamma", (planes,), "gamma", f"{p}.conv2")
            tb.add(f"{p}.gn2.beta", (planes,), "beta", f"{p}.conv2")
            names += [f"{p}.conv1.w", f"{p}.gn1.gamma", f"{p}.gn1.beta",
                      f"{p}.conv2.w", f"{p}.gn2.gamma", f"{p}.gn2.beta"]
            down = stride != 1 or cin != planes
            if down:
                tb.add(f"{p}.down.w", (planes, cin, 1, 1), "conv_w", f"{p}.down")
                tb.add(f"{p}.down_gn.gamma", (planes,), "gamma", f"{p}.down")
                tb.add(f"{p}.down_gn.beta", (planes,), "beta", f"{p}.down")
                names += [f"{p}.down.w", f"{p}.down_gn.gamma", f"{p}.down_gn.beta"]
                layers.append(ChannelLayerSpec(f"{p}.down", planes, norm_groups, False,
                                               ((f"{p}.down.w", 0), (f"{p}.down_gn.gamma", 0),
                                                (f"{p}.down_gn.beta", 0)), ()))
            layers.append(ChannelLayerSpec(f"{p}.conv1", planes, norm_groups, True,
                                           ((f"{p}.conv1.w", 0), (f"{p}.gn1.gamma", 0), (f"{p}.gn1.beta", 0)),
                                           ((f"{p}.conv2.w", 1),)))
            layers.append(ChannelLayerSpec(f"{p}.conv2", planes, norm_groups, True,
                                           ((f"{p}.conv2.w", 0), (f"{p}.gn2.gamma", 0), (f"{p}.gn2.beta", 0)),
                                           ()))
            # a downsampling block changes the residual shape: never dropped
            blocks_.append(BlockSpec(p, bi, tuple(names), not down, not down, 6 * planes * hw))
            bi += 1
            cin = planes
    tb.add("fc.w", (classes, 512), "linear_w", "head")
    tb.add("fc.b", (classes,), "bias", "head")
    layers.append(ChannelLayerSpec("head", classes, 1, False, (("fc.w", 0), ("fc.b", 0)), ()))
    return ModelTopology(tuple(tb.specs), tuple(layers), tuple(blocks_), 3 * 64 * h * w + 512 + classes,
                         (3, h, w), "layer3.1.conv2.w")


def gpt2_small_topology(vocab: int = 50257, n_ctx: int = 1024, d_model: int = 768,
                        n_layer: int = 12, seq_len: int = 1024) -> ModelTopology:
    e = d_model
    tb = TopologyBuilder()
    tb.add("wte", (vocab, e), "embed", "embed")
    tb.add("wpe", (n_ctx, e), "embed", "embed")
    layers = []
    blocks_ = []
    for i in range(n_layer):
        p = f"h{i}"
        spec = [
            (f"{p}.ln_1.w", (e,), "norm_w"), (f"{p}.ln_1.b", (e,), "norm_b"),
            (f"{p}.attn.c_attn.w", (e, 3 * e), "linear_w"), (f"{p}.attn.c_attn.b", (3 * e,), "bias"),
            (f"{p}.attn.c_proj.w", (e, e), "linear_w"), (f"{p}.attn.c_proj.b", (e,), "bias"),
            (f"{p}.ln_2.w", (e,), "norm_w"), (f"{p}.ln_2.b", (e,), "norm_b"),
            (f"{p}.mlp.c_fc.w", (e, 4 * e), "linear_w"), (f"{p}.mlp.c_fc.b", (4 * e,), "bias"),
            (f"{p}.mlp.c_proj.w", (4 * e, e), "linear_w"), (f"{p}.mlp.c_proj.b", (e,), "bias"),
        ]
        for name, shape, kind in spec:
            tb.add(name, shape, kind, f"{p}.mlp" if ".mlp.c_fc" in name else p)
        # Conv1D weights are [in, out]: hidden unit u is column u of c_fc, row u of c_proj
        layers.append(ChannelLayerSpec(f"{p}.mlp", 4 * e, 1, True,
                                       ((f"{p}.mlp.c_fc.w", 1), (f"{p}.mlp.c_fc.b", 0)),
                                       ((f"{p}.mlp.c_proj.w", 0),)))
        blocks_.append(BlockSpec(p, i, tuple(n for n, _, _ in spec), True, True, 16 * e * seq_len))
    tb.add("ln_f.w", (e,), "norm_w", "head")
    tb.add("ln_f.b", (e,), "norm_b", "head")
    return ModelTopology(tuple(tb.specs), tuple(layers), tuple(blocks_), 4 * e * seq_len, (seq_len,),
                         "h6.mlp.c_fc.w")


def sweep_topology(total: int, n_blocks: int = 64, always_frac: float = 0.01) -> ModelTopology:
    """Config C5: an always-active prefix of ~1% of d, then n_blocks equal blocks."""
    a = max(16, int(round(total * always_frac)) // 16 * 16)
    per = (total - a) // n_blocks
    tb = TopologyBuilder()
    tb.add("always", (a,), "bias", "always")
    blocks_ = []
    for b in range(n_blocks):
        size = per if b < n_blocks - 1 else total - a - per * (n_blocks - 1)
        tb.add(f"block{b}.w", (size,), "linear_w", f"block{b}")
        blocks_.append(BlockSpec(f"block{b}", b, (f"block{b}.w",), True, True, 0))
    return ModelTopology(tuple(tb.specs), (), tuple(blocks_), 0, (1,), "block0.w")
