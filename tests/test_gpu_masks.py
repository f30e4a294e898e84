"""GPU mask builder (k_assign + k_build_masks) vs the reference's golden masks
and the pinned oracle: bit-exact for every array field."""

import ctypes as C

import numpy as np
import pytest
import torch

import _golden as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _m():
    from paper_2507_09029_b200 import masking
    return masking


def test_device_permutation_matches_numpy(cuda):
    from paper_2507_09029_b200 import _native as N
    p = G.permutations()
    off = 0
    for seed, n in zip(G.seeds(), p["n"]):
        n = int(n)
        out = torch.full((max(n, 1),), -1, dtype=torch.int32, device=cuda)
        words, nw = N.seed_words(seed)
        N.call("sdp_permutation", words, nw, None, 0, n, C.c_void_p(out.data_ptr()), None)
        assert np.array_equal(out[:n].cpu().numpy(), p["values"][off:off + n]), (seed, n)
        off += n
    # sequential draws from one generator
    sizes = [int(x) for x in p["seq_sizes"]]
    off = 0
    for k, n in enumerate(sizes):
        skip = torch.tensor(sizes[:k] or [0], dtype=torch.int32, device=cuda)
        out = torch.empty(n, dtype=torch.int32, device=cuda)
        words, nw = N.seed_words(int(p["seq_seed"][0]))
        N.call("sdp_permutation", words, nw, C.c_void_p(skip.data_ptr()), k, n,
               C.c_void_p(out.data_ptr()), None)
        assert np.array_equal(out.cpu().numpy(), p["seq_values"][off:off + n])
        off += n


@pytest.mark.parametrize("case", G.cases(), ids=lambda c: f"{c['model']}-{c['strategy']}-N{c['n']}P{c['p']}s{c['seed']}")
def test_build_assignment_bitexact_vs_reference(cuda, case):
    masking = _m()
    topo = G.topology(case["model"])
    a = masking.build_assignment(topo, case["strategy"], case["n"], case["p"], case["seed"])
    want = G.case_masks(case)
    assert np.array_equal(a.param_masks.cpu().numpy(), want)
    arr = G.arrays()
    assert np.array_equal(a.governors.cpu().numpy(), arr[f"c{case['id']}_governors"].astype(np.int64))
    cov = arr[f"c{case['id']}_coverage"].astype(np.int64)
    assert np.array_equal(a.coverage.cpu().numpy(), cov)
    assert np.array_equal(a.divisor.cpu().numpy(), np.maximum(cov, 1).astype(np.float64))
    assert {u.key(): list(w) for u, w in a.unit_workers.items()} == case["unit_workers"]
    assert a.active_param_counts() == case["active_param_counts"]
    assert a.uncovered_params == case["uncovered_params"]
    rep = masking.validate(a)
    assert rep.unit_counts == case["unit_counts"]
    # owner bitmask == packed reference masks
    om = a.owner_mask.cpu().numpy().astype(np.uint64) & np.uint64((1 << case["n"]) - 1)
    packed = (want.astype(np.uint64) << np.arange(case["n"], dtype=np.uint64)[:, None]).sum(0)
    assert np.array_equal(om, packed)


def test_worker_view_matches_mask_rows(cuda):
    masking = _m()
    case = G.cases()[1]
    topo = G.topology(case["model"])
    a = masking.build_assignment(topo, case["strategy"], case["n"], case["p"], case["seed"])
    want = G.case_masks(case)
    for w in range(case["n"]):
        v = a.worker_view(w)
        assert np.array_equal(v.param_mask_bool.cpu().numpy(), want[w])
        assert np.array_equal(v.param_mask.cpu().numpy(), want[w].astype(np.float64))
        assert v.active_params == int(want[w].sum())
        assert not v.block_active.flags.writeable
    v1, v2 = a.worker_view(2), a.worker_view(2)
    assert torch.equal(v1.param_mask_bool, v2.param_mask_bool)
    from paper_2507_09029_b200.errors import ConfigError
    with pytest.raises(ConfigError):
        a.worker_view(case["n"])


def test_randomized_coverage_invariants(cuda):
    """test_masking.py:271-287 on the device builder: 100 random (N, P, blocks, seed)."""
    masking = _m()
    from paper_2507_09029_b200 import zoo
    rng = np.random.default_rng(99)
    for _ in range(100):
        n = int(rng.integers(2, 17))
        p = int(rng.integers(1, n + 1))
        blocks = int(rng.integers(max(2, n), 64))
        width = int(rng.integers(2, 7))
        seed = int(rng.integers(1 << 31))
        topo = zoo.residual_mlp_topology(width=width, blocks=blocks, classes=3, in_dim=4)
        a = masking.build_assignment(topo, "block", n, p, seed)
        cov = a.coverage.cpu().numpy()
        gov = a.governors.cpu().numpy()
        assert np.all(cov[gov >= 1] == p) and np.all(cov[gov == 0] == n)
        o = O.build_assignment(topo, "block", n, p, seed)
        assert np.array_equal(a.param_masks.cpu().numpy(), o.param_masks)


def test_randomized_grouped_assignment_matches_oracle(cuda):
    """assign_grouped_units (masking.py:88-117): one generator across groups."""
    masking = _m()
    rng = np.random.default_rng(7)
    for _ in range(30):
        n = int(rng.integers(2, 9))
        p = int(rng.integers(1, n + 1))
        sizes = [int(rng.integers(n, 40)) for _ in range(int(rng.integers(1, 5)))]
        groups = [[masking.StructuralUnit("channel", f"layer{g}", i) for i in range(s)]
                  for g, s in enumerate(sizes)]
        seed = int(rng.integers(1 << 31))
        got = masking.assign_grouped_units(groups, n, p, seed)
        bits = O.assign_grouped(sizes, n, p, seed)
        flat = [u for g in groups for u in g]
        for u, b in zip(flat, bits):
            assert got[u] == tuple(w for w in range(n) if b >> w & 1)
        for g in groups:
            loads = np.zeros(n, int)
            for u in g:
                loads[list(got[u])] += 1
            assert loads.max() - loads.min() <= 1


def test_assign_units_errors_and_windows(cuda):
    masking = _m()
    from paper_2507_09029_b200.errors import ConfigError
    us = [masking.StructuralUnit("block", f"u{i}") for i in range(8)]
    assert all(w == tuple(range(8)) for w in masking.assign_units(us, 8, 8, seed=0).values())
    assert masking.slot_windows(8, 8, 4)[0] == (0, 1, 2, 3)
    with pytest.raises(ConfigError):
        masking.assign_units(us[:4], 4, 5, seed=0)
    with pytest.raises(ConfigError):
        masking.assign_units([], 4, 2, seed=0)
    a1 = masking.assign_units([masking.StructuralUnit("block", f"u{i}") for i in range(17)], 6, 2, seed=42)
    a2 = masking.assign_units([masking.StructuralUnit("block", f"u{i}") for i in range(17)], 6, 2, seed=43)
    assert a1 != a2


def test_channel_induction_hand_expansion(cuda):
    """test_masking.py:124-139: dropping channel 0 of block0.conv1."""
    masking = _m()
    from paper_2507_09029_b200 import zoo
    topo = zoo.mini_resnet_topology(4, 2, 3, 2, 2, (4, 4))
    ca = {"block0.conv1": np.ones((1, 4), dtype=bool)}
    ca["block0.conv1"][0, 0] = False
    masks = masking.induce_channel_param_mask(topo, ca).cpu().numpy()
    dead = np.zeros(topo.total, dtype=bool)
    w1 = topo.index["block0.conv1.w"]
    dead[w1.offset:w1.offset + w1.size].reshape(w1.shape)[0] = True
    for name in ("block0.conv1.b", "block0.gn1.gamma", "block0.gn1.beta"):
        dead[topo.index[name].offset] = True
    w2 = topo.index["block0.conv2.w"]
    dead[w2.offset:w2.offset + w2.size].reshape(w2.shape)[:, 0] = True
    assert np.array_equal(~masks[0], dead)
    from paper_2507_09029_b200.errors import TopologyError
    with pytest.raises(TopologyError, match="undeclared"):
        masking.induce_channel_param_mask(topo, {"nope": np.ones((2, 4), dtype=bool)})


def test_channel_induction_random_flags_vs_oracle_loops(cuda):
    masking = _m()
    from paper_2507_09029_b200 import zoo
    topo = zoo.mini_resnet_topology(4, 2, 3, 2, 2, (4, 4))
    rng = np.random.default_rng(11)
    ca = {}
    for layer in topo.channel_layers:
        if layer.maskable:
            f = rng.random((3, layer.channels)) > 0.4
            f[:, 0] = True
            ca[layer.layer_id] = f
    got = masking.induce_channel_param_mask(topo, ca).cpu().numpy()
    want = np.ones((3, topo.total), dtype=bool)
    for w in range(3):
        for layer in topo.channel_layers:
            if layer.layer_id not in ca:
                continue
            for pname, axis in tuple(layer.own_slices) + tuple(layer.consumer_slices):
                spec = topo.index[pname]
                for coord in np.ndindex(spec.shape):
                    if not ca[layer.layer_id][w, coord[axis]]:
                        want[w, spec.offset + np.ravel_multi_index(coord, spec.shape)] = False
    assert np.array_equal(got, want)


def test_block_induction_and_errors(cuda):
    masking = _m()
    from paper_2507_09029_b200 import zoo
    from paper_2507_09029_b200.errors import ConfigError, ValidationError
    topo = zoo.residual_mlp_topology(6, 8, 3, 4)
    active = np.ones((1, 8), dtype=bool)
    active[0, [2, 5]] = False
    masks = masking.induce_block_param_mask(topo, active).cpu().numpy()
    assert masks[0].sum() == topo.total - 2 * 2 * (36 + 6)
    assert masking.induce_block_param_mask(topo, np.ones((4, 8), bool)).all()
    a = masking.build_assignment(topo, "block", 2, 1, seed=0)
    act = np.zeros((2, 8), dtype=bool)
    act[1] = True
    broken = masking.MaskAssignment(2, 1, "block", 0, topo, {u: (1,) for u in a.unit_workers},
                                    masking.induce_block_param_mask(topo, act), a.governors)
    with pytest.raises(ValidationError, match="no active block"):
        masking.validate(broken)


def test_json_round_trip(cuda, tmp_path):
    masking = _m()
    from paper_2507_09029_b200 import zoo
    topo = zoo.mini_resnet_topology(8, 3, 4, 2, 2, (4, 4))
    for strategy in ("neuron", "block"):
        a = masking.build_assignment(topo, strategy, 8, 5, seed=21)
        path = tmp_path / f"{strategy}.json"
        masking.save_assignment(a, path)
        b = masking.load_assignment(path, topo)
        assert b.unit_workers == a.unit_workers
        assert torch.equal(b.param_masks, a.param_masks)
        assert torch.equal(b.owner_mask, a.owner_mask)


def test_large_topologies_match_oracle(cuda):
    """ResNet-18 (C2 block, C3 neuron) and GPT-2 small (C4) on the device."""
    masking = _m()
    from paper_2507_09029_b200 import zoo
    for topo, strategy in ((zoo.resnet18_cifar_topology(), "block"),
                           (zoo.resnet18_cifar_topology(), "neuron")):
        a = masking.build_assignment(topo, strategy, 8, 4, seed=1)
        o = O.build_assignment(topo, strategy, 8, 4, 1)
        assert np.array_equal(a.owner_mask.cpu().numpy().astype(np.uint64), o.owner_bits)
        assert np.array_equal(a.coverage.cpu().numpy(), o.coverage)
        assert np.array_equal(a.governors.cpu().numpy(), o.governors)
        masking.validate(a)
    g = zoo.gpt2_small_topology()
    a = masking.build_assignment(g, "block", 8, 4, seed=1)
    cov = a.coverage.cpu().numpy()
    assert cov.size == 124_439_808
    assert int((cov == 4).sum()) == 12 * 7_087_872 and int((cov == 8).sum()) == 39_385_344


@pytest.mark.parametrize("sizes", [[20000], [5000, 7000, 3000, 9000, 1, 2]],
                         ids=["scratch-group", "multi-refill"])
def test_device_assign_long_streams(cuda, sizes):
    """k_assign over groups that outrun one refill of the parallel PCG64 stream
    (8192 words) and a group too large for shared memory: the unit owner bits
    equal numpy's default_rng permutations (masking.py:107-116) drawn in order."""
    masking = _m()
    groups, pos = [], 0
    for s in sizes:
        groups.append((pos, s))
        pos += s
    got = masking._device_assign(groups, pos, 8, 3, 7, cuda).cpu().numpy().view(np.uint64)
    rng = np.random.default_rng(7)
    want, slot = np.zeros(pos, dtype=np.uint64), 0
    for first, s in groups:
        for k, u in enumerate(rng.permutation(s)):
            want[first + int(u)] = O.window_bits(slot + k, 8, 3)
        slot += s
    assert np.array_equal(got, want)
