"""The real N > 1 path across PROCESSES on one GPU: the ranks export their
replicas + signal pads with CUDA IPC, exchange handles over gloo, open each
other's buffers and run k_owner_sync with the cross-rank flag barriers.

Without MPS the two processes' kernels are time-sliced rather than
co-scheduled, so the barrier waits span context switches; the spin timeout
(5 s) turns a stall into a reported failure instead of a hang."""

import os
import socket
import subprocess
import sys
import textwrap

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CHILD = textwrap.dedent(r"""
    import os, sys, numpy as np, torch, torch.distributed as dist
    sys.path.insert(0, os.environ["REPO"])
    from paper_2507_09029_b200 import comm, masking, zoo
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["RANK"]) % torch.cuda.device_count())  # own GPU when >= 2 are visible
    dist.init_process_group("gloo", rank=rank, world_size=world)
    def all_gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out
    topo = zoo.mini_resnet_topology(26, 8, 10, 2, 3, (32, 32))
    a = masking.build_assignment(topo, os.environ["STRATEGY"], 4, 2, seed=1)
    lay = None
    if os.environ.get("LAYOUT") == "sync":
        from paper_2507_09029_b200.layout import SyncLayout
        lay = SyncLayout(a)
    g = comm.PeerGroup(a, rank, world, torch.device("cuda", torch.cuda.current_device()), all_gather, max_grid=4,
                       timeout_cycles=10_000_000_000, owner_mask=None if lay is None else lay.owner_mask)
    gen = torch.Generator(device="cuda")
    for w, t in g.replicas.items():
        gen.manual_seed(50 + w)
        x = torch.randn(t.numel(), generator=gen, device="cuda") * a.param_masks[w]
        t.copy_(x if lay is None else lay.to_sync(x))
    torch.cuda.synchronize()
    dist.barrier()
    g.launch()
    torch.cuda.synchronize()
    dist.barrier()
    st = int(g.status.item())
    out = {w: (t if lay is None else lay.from_sync(t)).cpu().numpy() for w, t in g.replicas.items()}
    np.savez(os.path.join(os.environ["OUT"], f"rank{rank}.npz"), status=st, **{f"w{w}": v for w, v in out.items()})
    g.close()
    dist.destroy_process_group()
""")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("strategy,layout,world", [("block", "ref", 2), ("neuron", "ref", 2), ("neuron", "sync", 2),
                                                   ("block", "ref", 4), ("neuron", "sync", 4)])
def test_multi_process_ipc_owner_sync(cuda, tmp_path, strategy, layout, world):
    """world = 4 is one worker per rank (N = G = 4), the real deployment shape."""
    import torch
    from oracle import oracle as O
    from paper_2507_09029_b200 import masking, zoo
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = _port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), REPO=repo, OUT=str(tmp_path), STRATEGY=strategy,
                   LAYOUT=layout)
        procs.append(subprocess.Popen([sys.executable, "-c", CHILD], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=180)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("IPC ranks did not finish in 180 s")
    assert all(p.returncode == 0 for p in procs), "\n".join(outs)
    # expected: the oracle's ordered fp32 mean over the same seeded replicas
    topo = zoo.mini_resnet_topology(26, 8, 10, 2, 3, (32, 32))
    a = masking.build_assignment(topo, strategy, 4, 2, seed=1)
    gen = torch.Generator(device="cuda")
    host = []
    for w in range(4):
        gen.manual_seed(50 + w)
        host.append((torch.randn(topo.total, generator=gen, device="cuda") * a.param_masks[w]).cpu().numpy())
    masks = a.param_masks.cpu().numpy()
    want = O.aggregate_f32_ordered(host, masks)
    for r in range(world):
        z = np.load(tmp_path / f"rank{r}.npz")
        assert int(z["status"]) == 0, f"rank {r} status {int(z['status'])}"
        for w in [w for w in range(4) if w * world // 4 == r]:
            got = z[f"w{w}"]
            m = masks[w]
            assert np.array_equal(got[m].view(np.uint32), want[m].view(np.uint32))
            assert np.array_equal(got[~m], host[w][~m])


TRAIN_CHILD = textwrap.dedent(r"""
    import os, sys, numpy as np, torch, torch.distributed as dist
    sys.path.insert(0, os.environ["REPO"])
    from paper_2507_09029_b200 import masking, train
    torch.backends.cudnn.deterministic = True
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["RANK"]) % torch.cuda.device_count())  # own GPU when >= 2 are visible
    dist.init_process_group("gloo", rank=rank, world_size=world)
    def all_gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out
    dev = torch.device("cuda", torch.cuda.current_device())
    model = train.build_resnet18(dev, seed=5)
    a = masking.build_assignment(model.topology, os.environ["STRATEGY"], 4, 2, seed=1)
    opt = os.environ.get("OPT", "sgd-nesterov")
    tr = train.PeerTrainer(model, a, rank, world, dev, all_gather, lr=0.05 if opt == "sgd-nesterov" else 0.002,
                           autocast=os.environ["AUTOCAST"] == "1", timeout_cycles=10_000_000_000,
                           graphed=os.environ["GRAPHED"] == "1", optimizer=opt)
    for step in range(2):
        batches = {}
        for w in tr.local:
            gen = torch.Generator(device=dev)
            gen.manual_seed(100 * step + w)
            batches[w] = (torch.randn(4, 3, 32, 32, generator=gen, device=dev),
                          torch.randint(0, 10, (4,), generator=gen, device=dev))
        tr.step(batches)
        torch.cuda.synchronize()
        dist.barrier()
    tr.group.check()
    np.savez(os.path.join(os.environ["OUT"], f"rank{rank}.npz"),
             **{f"w{w}": tr.theta_of(w).cpu().numpy() for w in tr.local})
    tr.close()
    dist.destroy_process_group()
""")


@pytest.mark.parametrize("graphed,autocast,opt", [(False, False, "sgd-nesterov"), (True, False, "sgd-nesterov"),
                                                  (True, True, "sgd-nesterov"), (True, True, "adam")])
@pytest.mark.parametrize("strategy", ["block", "neuron"])
def test_peer_trainer_matches_coresident(cuda, tmp_path, strategy, graphed, autocast, opt):
    """train.PeerTrainer over 2 processes (CUDA-IPC replicas, cross-rank sync,
    local Nesterov) leaves every worker's copy of its parameters bit-identical
    to the co-resident trainer's canonical theta (deterministic cuDNN; fp32,
    and the bf16 autocast step with its fused gradient stores) -- also when
    each rank replays its step from a CUDA graph (device-resident barrier
    epochs)."""
    import torch
    from paper_2507_09029_b200 import masking, train
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = _port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), REPO=repo, OUT=str(tmp_path), STRATEGY=strategy,
                   GRAPHED=str(int(graphed)), AUTOCAST=str(int(autocast)), OPT=opt)
        procs.append(subprocess.Popen([sys.executable, "-c", TRAIN_CHILD], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=300)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("trainer ranks did not finish in 300 s")
    assert all(p.returncode == 0 for p in procs), "\n".join(outs)
    prev = torch.backends.cudnn.deterministic
    torch.backends.cudnn.deterministic = True
    try:
        model = train.build_resnet18(cuda, seed=5)
        a = masking.build_assignment(model.topology, strategy, 4, 2, seed=1)
        tr = train.SubnetTrainer(model, a, lr=0.05 if opt == "sgd-nesterov" else 0.002, autocast=autocast,
                                 sync_layout=strategy == "neuron", optimizer=opt)
        for step in range(2):
            batches = []
            for w in range(4):
                gen = torch.Generator(device=cuda)
                gen.manual_seed(100 * step + w)
                batches.append((torch.randn(4, 3, 32, 32, generator=gen, device=cuda),
                                torch.randint(0, 10, (4,), generator=gen, device=cuda)))
            tr.step(batches)
        canon = tr.theta().cpu().numpy()
    finally:
        torch.backends.cudnn.deterministic = prev
    masks = a.param_masks.cpu().numpy()
    for r in range(2):
        z = np.load(tmp_path / f"rank{r}.npz")
        for w in (0, 1) if r == 0 else (2, 3):
            got = z[f"w{w}"]
            # bit-identical in fp32 and under bf16 autocast (libsdp's GroupNorm
            # backward folds dgamma / dbeta in a fixed order: no atomics)
            assert np.array_equal(got[masks[w]].view(np.uint32), canon[masks[w]].view(np.uint32)), (r, w)


LOCAL_CHILD = textwrap.dedent(r"""
    import os, sys, numpy as np, torch, torch.distributed as dist
    sys.path.insert(0, os.environ["REPO"])
    from paper_2507_09029_b200 import comm, masking, zoo
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["RANK"]) % torch.cuda.device_count())  # own GPU when >= 2 are visible
    dist.init_process_group("gloo", rank=rank, world_size=world)
    topo = zoo.mini_resnet_topology(26, 8, 10, 2, 3, (32, 32))
    a = masking.build_assignment(topo, os.environ["STRATEGY"], 4, 2, seed=1)
    local = comm.rank_layout(4, world, rank).local_workers
    res = {}
    for step in range(2):  # the second call reuses the cached peer group
        grads = {}
        gen = torch.Generator(device="cuda")
        for w in local:
            gen.manual_seed(50 + 10 * step + w)
            grads[w] = torch.randn(topo.total, generator=gen, device="cuda") * a.param_masks[w]
        out = comm.aggregate_local(grads if len(local) > 1 else grads[local[0]], a, check=True)
        res.update({f"s{step}w{w}": t.cpu().numpy() for w, t in out.items()})
    np.savez(os.path.join(os.environ["OUT"], f"rank{rank}.npz"), **res)
    comm.close_local_groups()
    dist.destroy_process_group()
""")


@pytest.mark.parametrize("strategy,world", [("block", 2), ("neuron", 2), ("block", 4)])
def test_aggregate_local_matches_aggregate(cuda, tmp_path, strategy, world):
    """comm.aggregate_local (the per-rank form of engine.aggregate)
    over real processes: every rank gets gbar * mask_w for its local workers,
    bit-identical to the oracle's ordered fp32 mean; 0 off the mask."""
    import torch
    from oracle import oracle as O
    from paper_2507_09029_b200 import masking, zoo
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = _port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), REPO=repo, OUT=str(tmp_path), STRATEGY=strategy)
        procs.append(subprocess.Popen([sys.executable, "-c", LOCAL_CHILD], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=180)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("aggregate_local ranks did not finish in 180 s")
    assert all(p.returncode == 0 for p in procs), "\n".join(outs)
    topo = zoo.mini_resnet_topology(26, 8, 10, 2, 3, (32, 32))
    a = masking.build_assignment(topo, strategy, 4, 2, seed=1)
    masks = a.param_masks.cpu().numpy()
    for step in range(2):
        gen = torch.Generator(device="cuda")
        host = []
        for w in range(4):
            gen.manual_seed(50 + 10 * step + w)
            host.append((torch.randn(topo.total, generator=gen, device="cuda") * a.param_masks[w]).cpu().numpy())
        want = O.aggregate_f32_ordered(host, masks)
        for r in range(world):
            z = np.load(tmp_path / f"rank{r}.npz")
            for w in [w for w in range(4) if w * world // 4 == r]:
                got, m = z[f"s{step}w{w}"], masks[w]
                assert np.array_equal(got[m].view(np.uint32), want[m].view(np.uint32)), (step, r, w)
                assert not got[~m].any()
