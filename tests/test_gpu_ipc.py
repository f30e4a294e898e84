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
    torch.cuda.set_device(0)
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
    g = comm.PeerGroup(a, rank, world, torch.device("cuda", 0), all_gather, max_grid=4,
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
