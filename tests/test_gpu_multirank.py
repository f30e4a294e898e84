"""The cross-rank kernel path on ONE GPU: two ranks' k_owner_sync launches on
two concurrent streams, each reducing the tiles it leads, meeting at the
per-CTA release/acquire flag barriers (the NVLink path with local pointers)."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _setup(cuda, strategy, n, p, world, grid):
    from paper_2507_09029_b200 import comm, engine, masking, zoo
    topo = zoo.mini_resnet_topology(26, 8, 10, 2, 3, (32, 32))
    a = masking.build_assignment(topo, strategy, n, p, seed=1)
    d = topo.total
    gen = torch.Generator(device=cuda)
    reps, shs = [], []
    for w in range(n):
        gen.manual_seed(50 + w)
        reps.append(torch.randn(d, generator=gen, device=cuda) * a.param_masks[w])
        shs.append(torch.zeros(d, dtype=torch.bfloat16, device=cuda))
    pads = [torch.zeros(grid * comm.PAD_WORDS_PER_CTA, dtype=torch.int32, device=cuda) for _ in range(world)]
    status = [torch.zeros(1, dtype=torch.int32, device=cuda) for _ in range(world)]
    plans = [engine.SyncPlan(a, world=world, rank=r, resident=True, force_grid=grid) for r in range(world)]
    args = [comm.bind_rank_args(plans[r], 0, [t.data_ptr() for t in reps], [t.data_ptr() for t in shs],
                                [t.data_ptr() for t in pads], status[r].data_ptr(), 2_000_000_000)
            for r in range(world)]
    return a, reps, shs, args, status, plans


def _launch_all(args, epoch):
    import ctypes as C
    from paper_2507_09029_b200 import _native as N
    streams = [torch.cuda.Stream() for _ in args]
    torch.cuda.synchronize()
    for a, s in zip(args, streams):
        a.epoch = epoch
        N.check(N.lib().sdp_owner_sync(C.byref(a), C.c_void_p(s.cuda_stream)))
    torch.cuda.synchronize()


@pytest.mark.parametrize("strategy,n,p,world", [("block", 4, 2, 2), ("neuron", 8, 3, 2),
                                                ("block", 8, 4, 4), ("neuron", 8, 4, 8)])
def test_two_stream_ranks_match_single_launch(cuda, strategy, n, p, world):
    a, reps, shs, args, status, plans = _setup(cuda, strategy, n, p, world, grid=8)
    host = [r.cpu().numpy() for r in reps]
    masks = a.param_masks.cpu().numpy()
    # the ranks' tile sets partition the vector
    idx = sorted(i for pl in plans for i in pl.mine["tile_index"].tolist())
    assert idx == list(range(len(plans[0].all_tiles)))
    cur = [h.copy() for h in host]
    for epoch in (1, 2, 3):
        _launch_all(args, epoch)
        assert all(int(s.item()) == 0 for s in status), [int(s.item()) for s in status]
        # expected replicas after this epoch: the mean written into every owner
        want = O.aggregate_f32_ordered(cur, masks)
        prev = cur
        cur = [np.where(masks[w], want, prev[w]) for w in range(n)]
    for w in range(n):
        m = masks[w]
        got = reps[w].cpu().numpy()
        assert np.array_equal(got[m].view(np.uint32), want[m].view(np.uint32))
        assert np.array_equal(got[~m], host[w][~m])
        assert np.array_equal(shs[w].view(torch.int16).cpu().numpy().view(np.uint16)[m], O.bf16_rne(want)[m])


@pytest.mark.parametrize("strategy", ["block", "neuron"])
def test_plan_tiles_matches_oracle(cuda, strategy):
    from paper_2507_09029_b200 import masking, zoo
    topo = zoo.resnet18_cifar_topology()
    a = masking.build_assignment(topo, strategy, 8, 4, seed=1)
    o = O.build_assignment(topo, strategy, 8, 4, 1)
    plan = a.sync_plan()
    want = O.plan_tiles(o.owner_bits, plan.tile)
    assert np.array_equal(plan.all_tiles.view(np.uint8), want.view(np.uint8))


def test_missing_peer_times_out_instead_of_hanging(cuda):
    import ctypes as C
    from paper_2507_09029_b200 import _native as N
    a, reps, shs, args, status, plans = _setup(cuda, "block", 4, 2, 2, grid=4)
    args[0].timeout_cycles = 20_000_000  # ~10 ms
    args[0].epoch = 1
    N.check(N.lib().sdp_owner_sync(C.byref(args[0]), None))  # rank 1 never launches
    torch.cuda.synchronize()
    assert int(status[0].item()) & N.STATUS_BARRIER_TIMEOUT
