"""Host logic of the N > 1 path on CPU: placement, tile leadership, CTA-major
tables, and the IPC-handle exchange over a real gloo process group (world 2)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2507_09029_b200 import comm, engine, zoo


def _tiles(topo, strategy, n, p, tile=4096):
    a = O.build_assignment(topo, strategy, n, p, 1)
    return O.plan_tiles(a.owner_bits, tile)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_contiguous_placement(world):
    lay = [comm.rank_layout(8, world, r) for r in range(world)]
    allw = sorted(w for l_ in lay for w in l_.local_workers)
    assert allw == list(range(8))
    assert all(len(l_.local_workers) == 8 // world for l_ in lay)
    assert lay[0].local_workers == list(range(8 // world))


@pytest.mark.parametrize("strategy", ["block", "neuron"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_tile_leaders_partition_and_locality(strategy, world):
    topo = zoo.resnet18_cifar_topology()
    tiles = _tiles(topo, strategy, 8, 4)
    gpu_of = engine.gpu_of_worker(8, world)
    lead = engine.tile_leaders(tiles, gpu_of, world)
    assert lead.min() >= 0 and lead.max() < world
    for t in range(len(tiles)):
        bits = int(tiles["owner_bits"][t])
        owners = {int(gpu_of[w]) for w in range(8) if bits >> w & 1}
        if owners:
            assert lead[t] in owners  # one of the reads is always local
    # leadership is spread across the owner GPUs of each window
    counts = np.bincount(lead, minlength=world)
    assert counts.min() > 0


def test_cta_major_table_covers_every_tile_once():
    tiles = _tiles(zoo.resnet18_cifar_topology(), "block", 8, 4)
    for grid in (1, 7, 148, len(tiles), len(tiles) + 5):
        tpc = max(1, -(-len(tiles) // grid))
        table = engine.cta_major(tiles, grid, tpc)
        live = table[(table["len_flags"] & 0xFFFFFF) > 0]
        assert sorted(live["tile_index"].tolist()) == list(range(len(tiles)))
        for b in range(min(grid, 5)):
            mine = table[b * tpc:(b + 1) * tpc]
            idx = mine[(mine["len_flags"] & 0xFFFFFF) > 0]["tile_index"]
            assert idx.tolist() == list(range(b, len(tiles), grid))[:tpc]


def test_plan_grid_residency():
    assert engine.plan_grid(10, 148, True) == 10
    assert engine.plan_grid(10_000, 148, True) == 148 * engine.CTAS_PER_SM
    assert engine.plan_grid(10_000, 148, False) == min(10_000, 148 * engine.CTAS_PER_SM * 8)
    assert engine.plan_grid(100_000, 148, False, traffic=2e9) == 100_000


def test_rank_layout_errors():
    from paper_2507_09029_b200.errors import ProtocolError
    with pytest.raises(ProtocolError):
        comm.rank_layout(4, 8, 0)
    with pytest.raises(ProtocolError):
        comm.rank_layout(16, 9, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def all_gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    try:
        lay = comm.rank_layout(8, world, rank)
        local = {f"rep{w}": (bytes([rank, w] * 32), 256 * w) for w in lay.local_workers}
        local["pad"] = (bytes([rank] * 64), 0)
        tables = comm.exchange_handles(local, all_gather)
        assert len(tables) == world
        for r, t in enumerate(tables):
            assert t["pad"] == (bytes([r] * 64), 0)
            for w in comm.rank_layout(8, world, r).local_workers:
                assert t[f"rep{w}"] == (bytes([r, w] * 32), 256 * w)
        # per-rank tile plans partition the tiles (same leaders everywhere)
        tiles = _tiles(zoo.resnet18_cifar_topology(), "block", 8, 4)
        lead = engine.tile_leaders(tiles, lay.gpu_of, world)
        mine = set(tiles[lead == rank]["tile_index"].tolist())
        everyone = all_gather(sorted(mine))
        flat = [t for m in everyone for t in m]
        assert sorted(flat) == list(range(len(tiles)))
        # a malformed handle is rejected
        with pytest.raises(Exception):
            comm.exchange_handles({"pad": (b"short", 0)}, all_gather)
        q.put((rank, "ok"))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_handle_exchange_and_partition():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_aggregate_local_requires_rank_or_process_group():
    """comm.aggregate_local raises the reference's ProtocolError (not a CUDA
    error) when it cannot tell which rank it runs on."""
    import torch.distributed as dist
    from paper_2507_09029_b200 import comm
    from paper_2507_09029_b200.errors import ProtocolError
    if dist.is_initialized():
        pytest.skip("a process group is already initialised in this process")
    with pytest.raises(ProtocolError):
        comm.aggregate_local({0: None}, object())
