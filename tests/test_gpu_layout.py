"""Window-class-major sync layout (layout.py): exact permutation, uniform
tiles, and a sync in the permuted space that is bit-identical to the sync in
the reference layout."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _assign(topo, strategy, n=8, p=4):
    from paper_2507_09029_b200 import masking
    return masking.build_assignment(topo, strategy, n, p, seed=1)


def _topos():
    from paper_2507_09029_b200 import zoo
    return [("mini", zoo.mini_resnet_topology(26, 8, 10, 2, 3, (32, 32))),
            ("mlp", zoo.residual_mlp_topology(32, 4, 3, 16)),
            ("r18", zoo.resnet18_cifar_topology())]


@pytest.mark.parametrize("strategy", ["neuron", "block"])
def test_round_trip_and_block_owner_sets(cuda, strategy):
    from paper_2507_09029_b200.layout import SyncLayout
    for name, topo in _topos():
        a = _assign(topo, strategy)
        lay = SyncLayout(a)
        for dt in (torch.float32, torch.float64):
            x = torch.randn(topo.total, device=cuda, dtype=dt)
            s = lay.to_sync(x)
            assert torch.equal(lay.from_sync(s), x), name
            if strategy == "block":
                assert torch.equal(s, x)  # identity for whole-tensor ownership
        # every block has one owner set; the permuted mask is the permuted bits
        om = lay.owner_mask.cpu().numpy()
        for pname, blocks in lay.blocks.items():
            for off, ridx, cidx, bits in blocks:
                rows, cols, inner = lay.shapes[pname]
                n = len(ridx) * len(cidx) * inner
                assert np.all(om[off:off + n] == bits), (name, pname)
        ref = a.owner_mask.cpu().numpy()
        assert np.array_equal(np.sort(om), np.sort(ref))


def test_neuron_tiles_become_uniform(cuda):
    from paper_2507_09029_b200 import zoo
    from paper_2507_09029_b200.layout import SyncLayout
    a = _assign(zoo.resnet18_cifar_topology(), "neuron")
    ref_plan = a.sync_plan()
    plan = SyncLayout(a).plan()
    assert plan.n_uniform / plan.n_tiles > 0.95 > ref_plan.n_uniform / ref_plan.n_tiles


@pytest.mark.parametrize("name_idx", [0, 1, 2])
def test_sync_in_sync_space_is_bitidentical(cuda, name_idx):
    from paper_2507_09029_b200 import engine
    from paper_2507_09029_b200.layout import SyncLayout
    name, topo = _topos()[name_idx]
    a = _assign(topo, "neuron")
    lay = SyncLayout(a)
    pm = a.param_masks
    reps = [torch.randn(topo.total, device=cuda) * pm[w] for w in range(8)]
    out_ref = torch.empty(topo.total, device=cuda)
    engine.owner_sync(reps, a, out=out_ref, writeback=False)
    sreps = [lay.to_sync(r) for r in reps]
    out_s = torch.empty(topo.total, device=cuda)
    shadows = [torch.zeros(topo.total, dtype=torch.bfloat16, device=cuda) for _ in range(8)]
    engine.owner_sync(sreps, a, out=out_s, plan=lay.plan(), shadows_bf16=shadows)
    assert torch.equal(lay.from_sync(out_s).view(torch.int32), out_ref.view(torch.int32))
    masks = pm.cpu().numpy()
    want = O.aggregate_f32_ordered([r.cpu().numpy() for r in reps], masks)
    for w in range(8):  # write-back landed on exactly the owned entries
        back = lay.from_sync(sreps[w]).cpu().numpy()
        assert np.array_equal(back[masks[w]].view(np.uint32), want[masks[w]].view(np.uint32))


def test_worker_transfer_matches_subnet_gather_scatter(cuda):
    from paper_2507_09029_b200 import models, zoo
    from paper_2507_09029_b200.layout import SyncLayout, WorkerTransfer
    topo = zoo.resnet18_cifar_topology()
    a = _assign(topo, "neuron")
    lay = SyncLayout(a)
    theta = torch.randn(topo.total, device=cuda)
    ts = lay.to_sync(theta)
    for w in (0, 3, 7):
        sub = models.SubnetLayout(a, w)
        tr = WorkerTransfer(lay, sub)
        assert torch.equal(tr.to_compact(ts), sub.gather(theta))
        g = torch.randn(sub.compact_total, device=cuda)
        gs = torch.zeros(topo.total, device=cuda)
        tr.from_compact(g, gs)
        assert torch.equal(lay.from_sync(gs), sub.scatter(g))


def test_trainer_in_sync_layout_equals_reference_layout(cuda):
    from paper_2507_09029_b200 import masking, train
    torch.manual_seed(0)
    gen = torch.Generator(device=cuda)
    gen.manual_seed(0)
    batches = [(torch.randn(4, 3, 32, 32, generator=gen, device=cuda),
                torch.randint(0, 10, (4,), generator=gen, device=cuda)) for _ in range(8)]
    thetas = []
    # cuDNN's default weight-gradient algorithms are not run-to-run deterministic
    old = (torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark)
    torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark = True, False
    try:
        for sync_layout in (False, True):
            model = train.build_resnet18(cuda, seed=3)
            a = masking.build_assignment(model.topology, "neuron", 8, 4, seed=1)
            tr = train.SubnetTrainer(model, a, lr=0.05, autocast=False, sync_layout=sync_layout)
            tr.step(batches)
            tr.step(batches)
            thetas.append(tr.theta())
    finally:
        torch.backends.cudnn.deterministic, torch.backends.cudnn.benchmark = old
    assert torch.equal(thetas[0].view(torch.int32), thetas[1].view(torch.int32))
