"""Compact owned-block storage (storage.CompactLayout, sdp_sync_args.slots) and
the fused local-update phase (SDP_SYNC_LOCAL_UPDATE).

* the sync over compact replicas (each worker stores only the tiles it owns,
  found through the per-owner slot table) is bit-identical to the flat sync,
  and the write-back lands on every owner's compact copy;
* the local-update phase applies optim.SgdNesterov (optim.py:78-84) to every
  worker's compact theta / velocity / bf16 copy, bit-identical to the oracle's
  Nesterov on the flat mean, over two steps;
* train.PeerTrainer on compact storage (one process, all workers local) trains
  bit-identically to the co-resident SubnetTrainer's canonical theta on every
  worker's owned elements, with one libsdp launch per step for sync + update.
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _flat_reps(a, seed, dev):
    gen = torch.Generator(device=dev)
    pm = a.param_masks
    out = []
    for w in range(a.n_workers):
        gen.manual_seed(seed + w)
        out.append(torch.randn(a.topology.total, generator=gen, device=dev) * pm[w])
    return out


CASES = [("mini", "block", 4, 2), ("mini", "neuron", 8, 3), ("r18", "block", 8, 4), ("sweep", "block", 8, 2)]


def _topo(name):
    from paper_2507_09029_b200 import zoo
    if name == "mini":
        return zoo.mini_resnet_topology(26, 8, 10, 2, 3, (32, 32))
    if name == "r18":
        return zoo.resnet18_cifar_topology()
    return zoo.sweep_topology(3 << 20)


@pytest.mark.parametrize("name,strategy,n,p", CASES)
def test_compact_sync_equals_flat(cuda, name, strategy, n, p):
    from paper_2507_09029_b200 import engine, masking
    from paper_2507_09029_b200.storage import CompactLayout
    a = masking.build_assignment(_topo(name), strategy, n, p, seed=7)
    plan = a.sync_plan()
    lay = CompactLayout(plan)
    flat = _flat_reps(a, 3, cuda)
    comp = [lay.gather(w, flat[w]) for w in range(n)]
    shadows = [torch.zeros(lay.length(w), dtype=torch.bfloat16, device=cuda) for w in range(n)]
    d = a.topology.total
    out_c = torch.empty(d, device=cuda)
    engine.owner_sync(comp, a, out=out_c, writeback=True, shadows_bf16=shadows, plan=plan, compact=lay)
    out_f = torch.empty(d, device=cuda)
    engine.owner_sync(flat, a, out=out_f, writeback=True, plan=plan)
    assert torch.equal(out_c.view(torch.int32), out_f.view(torch.int32))
    want = O.aggregate_f32_ordered([r.cpu().numpy() for r in _flat_reps(a, 3, cuda)], a.param_masks.cpu().numpy())
    assert np.array_equal(out_c.cpu().numpy().view(np.uint32), want.view(np.uint32))
    pm = a.param_masks
    for w in range(n):
        back = lay.scatter(w, comp[w], torch.zeros(d, device=cuda))
        assert torch.equal(back[pm[w]].view(torch.int32), out_f[pm[w]].view(torch.int32)), w
        sh = lay.scatter(w, shadows[w].float(), torch.zeros(d, device=cuda))
        assert torch.equal(sh[pm[w]], out_f[pm[w]].bfloat16().float()), w
    # storage really is smaller than N full replicas below P = N
    assert sum(lay.length(w) for w in range(n)) < n * d or p == n


@pytest.mark.parametrize("name,strategy,n,p", CASES[:3])
def test_local_update_phase_is_reference_nesterov(cuda, name, strategy, n, p):
    from paper_2507_09029_b200 import engine, masking
    from paper_2507_09029_b200.storage import CompactLayout, worker_states
    a = masking.build_assignment(_topo(name), strategy, n, p, seed=7)
    plan = a.sync_plan()
    lay = CompactLayout(plan)
    d = a.topology.total
    gen = torch.Generator(device=cuda)
    gen.manual_seed(11)
    theta = torch.randn(d, generator=gen, device=cuda)
    th = [lay.gather(w, theta) for w in range(n)]
    ve = [torch.zeros_like(t) for t in th]
    tb = [t.bfloat16() for t in th]
    reps = [torch.zeros(lay.length(w), device=cuda) for w in range(n)]
    states = worker_states([(th[w], ve[w], None, tb[w], reps[w]) for w in range(n)], cuda)
    table, per = lay.update_table(list(range(n)), plan.leader_cta(), plan.grid)
    status = torch.zeros(1, dtype=torch.int32, device=cuda)
    pm = a.param_masks.cpu().numpy()
    th_ref, v_ref = theta.cpu().numpy(), np.zeros(d, dtype=np.float32)
    for step in range(2):
        flat = _flat_reps(a, 100 + step, cuda)
        for w in range(n):
            reps[w].copy_(lay.gather(w, flat[w]))
        engine.owner_sync(reps, a, writeback=True, plan=plan, compact=lay, status=status, check_finite=True,
                          nesterov={"lr": 0.05, "momentum": 0.9},
                          local_update={"states": states, "updates": table, "per_cta": per})
        gbar = O.aggregate_f32_ordered([f.cpu().numpy() for f in flat], pm)
        th_ref, v_ref = O.nesterov_update(th_ref, v_ref, gbar, 0.05, 0.9)
        for w in range(n):
            got = lay.scatter(w, th[w], torch.zeros(d, device=cuda)).cpu().numpy()
            assert np.array_equal(got[pm[w]].view(np.uint32), th_ref[pm[w]].view(np.uint32)), (step, w)
            gb = lay.scatter(w, tb[w].float(), torch.zeros(d, device=cuda)).cpu().numpy()
            assert np.array_equal(gb[pm[w]].view(np.uint32),
                                  torch.from_numpy(th_ref).bfloat16().float().numpy()[pm[w]].view(np.uint32))
    assert int(status.item()) == 0
    # a non-finite mean sets the status word
    reps[0].fill_(float("nan"))
    engine.owner_sync(reps, a, writeback=True, plan=plan, compact=lay, status=status, check_finite=True,
                      nesterov={"lr": 0.05, "momentum": 0.9},
                      local_update={"states": states, "updates": table, "per_cta": per})
    assert int(status.item()) & 0x2


@pytest.mark.parametrize("arch,strategy,autocast,opt", [
    ("resnet18", "block", False, "sgd-nesterov"), ("mini", "block", False, "sgd-nesterov"),
    ("resnet18", "neuron", False, "sgd-nesterov"), ("mini", "neuron", False, "sgd-nesterov"),
    ("resnet18", "neuron", True, "sgd-nesterov"), ("resnet18", "block", True, "sgd-nesterov"),
    ("resnet18", "block", False, "adam"), ("resnet18", "neuron", True, "adam")])
def test_peer_trainer_compact_storage_matches_coresident(cuda, arch, strategy, autocast, opt):
    """PeerTrainer at world 1 (every worker local, owned-tile storage, one
    sync+Nesterov launch per step) == SubnetTrainer's canonical theta on every
    worker's owned elements, bit for bit (deterministic cuDNN; fp32 and bf16
    autocast), for block workers and for width-wise workers (sync-layout
    blocks addressed through the slot table)."""
    from paper_2507_09029_b200 import masking, models, train
    prev = torch.backends.cudnn.deterministic
    torch.backends.cudnn.deterministic = True
    try:
        def model():
            if arch == "resnet18":
                return train.build_resnet18(cuda, seed=5)
            return models.build_mini_resnet(26, 8, 10, 2, 3, (32, 32), seed=1, device_=cuda)
        n, p = (8, 4) if arch == "resnet18" else (4, 2)
        gen = torch.Generator(device=cuda)
        gen.manual_seed(4)
        steps = [[(torch.randn(4, 3, 32, 32, generator=gen, device=cuda),
                   torch.randint(0, 10, (4,), generator=gen, device=cuda)) for _ in range(n)] for _ in range(3)]
        m1 = model()
        a = masking.build_assignment(m1.topology, strategy, n, p, seed=1)
        lr = 0.05 if opt == "sgd-nesterov" else 0.002
        ref = train.SubnetTrainer(m1, a, lr=lr, autocast=autocast, sync_layout=strategy == "neuron", optimizer=opt)
        for b in steps:
            ref.step(b)
        canon = ref.theta().cpu().numpy()
        m2 = model()
        tr = train.PeerTrainer(m2, a, 0, 1, cuda, lambda o: [o], lr=lr, autocast=autocast, optimizer=opt)
        assert tr.compact_storage
        for b in steps:
            tr.step({w: b[w] for w in range(n)})
        tr.check()
        pm = a.param_masks.cpu().numpy()
        d = m2.topology.total
        for w in range(n):
            got = tr.theta_of(w).cpu().numpy()
            assert np.array_equal(got[pm[w]].view(np.uint32), canon[pm[w]].view(np.uint32)), w
        # compact: every worker stores fewer elements than the flat vector
        if p < n:
            assert max(tr.theta[w].numel() for w in range(n)) < d
        tr.close()
    finally:
        torch.backends.cudnn.deterministic = prev
