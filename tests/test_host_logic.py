"""Host-side logic of the drop-in that needs no GPU: the pinned result pool's
lease rule (engine._PinnedResults) and masks.json index validation."""

import threading

import numpy as np
import pytest
import torch


class _Pool:
    def __new__(cls):
        from paper_2507_09029_b200 import engine

        class P(engine._PinnedResults):
            @staticmethod
            def _alloc(d, dt):
                return torch.empty(d, dtype=dt)  # pageable stand-in: the lease logic is the same
        return P()


def test_pool_never_hands_a_held_buffer_out_twice():
    pool = _Pool()
    a, _ = pool.get(16, torch.float32)
    b, _ = pool.get(16, torch.float32)
    assert not np.shares_memory(a, b)
    a2 = a[3:]  # a view of the caller's result keeps the buffer leased
    del a
    c, _ = pool.get(16, torch.float32)
    assert not np.shares_memory(c, a2) and not np.shares_memory(c, b)
    del a2, c
    d, _ = pool.get(16, torch.float32)  # a released buffer is reused
    assert any(np.shares_memory(d, e[0]) for e in pool.bufs[(16, torch.float32)])


def test_pool_concurrent_callers_get_distinct_buffers():
    pool = _Pool()
    got, barrier = [], threading.Barrier(8)

    def run():
        barrier.wait()
        arr, _ = pool.get(64, torch.float32)
        got.append(arr)

    ts = [threading.Thread(target=run) for _ in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i in range(len(got)):
        for j in range(i + 1, len(got)):
            assert not np.shares_memory(got[i], got[j])


def _fake_plan(owner_sets, tile_len, leaders):
    import types

    from paper_2507_09029_b200 import _native as N
    dt = np.dtype([("owner_bits", "<u8"), ("tile_index", "<u4"), ("len_flags", "<u4")])
    t = np.zeros(len(owner_sets), dtype=dt)
    for i, ws in enumerate(owner_sets):
        t[i] = (sum(1 << w for w in ws), i, tile_len | N.TILE_UNIFORM)
    return types.SimpleNamespace(all_tiles=t, leaders=np.asarray(leaders))


def test_busbw_and_link_bytes_accounting():
    """busbw bytes = sum over my elements of 2(k-1)/k * 4 B
    (k = owner GPUs); link bytes per direction = the leader's peer reads (4 B)
    and its writes of the mean (+2 B shadow) to every remote owner."""
    from paper_2507_09029_b200 import comm
    lay = comm.rank_layout(8, 8, 0)  # one worker per GPU
    plan = _fake_plan([(0, 1, 2, 3), (4, 5, 6, 7), tuple(range(8))], 1000, [0, 5, 1])
    # rank 0 owns tiles 0 (k=4) and 2 (k=8)
    assert comm.busbw_bytes(plan, lay) == int(2 * 3 / 4 * 1000 * 4 + 2 * 7 / 8 * 1000 * 4)
    lb = comm.link_bytes(plan, lay, shadows=True)
    # tile 0 led here: read 3 remote owners, write 3 x 6 B; tile 2 led by rank 1:
    # rank 1 reads my copy (my TX 4 B) and writes the mean + shadow into it (my RX 6 B)
    assert lb == {"rx": 3 * 1000 * 4 + 1000 * 6, "tx": 3 * 1000 * 6 + 1000 * 4}
    lay2 = comm.rank_layout(8, 2, 0)  # workers 0-3 on GPU 0: tile 0 is GPU-local
    plan2 = _fake_plan([(0, 1, 2, 3), (0, 4)], 1000, [0, 1])
    assert comm.busbw_bytes(plan2, lay2) == int(2 * 1 / 2 * 1000 * 4)
    assert comm.link_bytes(plan2, lay2, shadows=False) == {"rx": 1000 * 4, "tx": 1000 * 4}


def test_slice_batch_concatenation_rebases_tables():
    """models.SliceBatch (one launch for all workers): descriptor map offsets
    and col tables are rebased onto the concatenated map array, every task
    points at its part's descriptor and carries the part as its segment, and
    the parts' tasks are interleaved round-robin."""
    from paper_2507_09029_b200 import models
    from paper_2507_09029_b200.models import SLICE_DTYPE, TASK_DTYPE

    def part(n_desc, maps_len, map_base):
        d = np.zeros(n_desc, dtype=SLICE_DTYPE)
        d["rows"], d["cols"], d["inner"], d["crows"], d["ccols"] = 4, 300, 1, 2, 300
        d["row_map"] = [map_base, -1][:n_desc] + [-1] * max(0, n_desc - 2)
        d["col_map"] = -1
        d["col_tab"] = -1
        t = models.slice_tasks(d, compact=True, per_task=600)
        return d, t, np.arange(maps_len, dtype=np.int32), True

    parts = [part(2, 5, 1), part(1, 7, 3), part(2, 3, 0)]
    sb = models.SliceBatch(parts, torch.device("cpu"), per_task=600)
    descs = sb.d_descs.numpy().view(SLICE_DTYPE)[: 5]
    tasks = sb.d_tasks.numpy().view(TASK_DTYPE)[: sb.n_tasks]
    assert sb.maps.numel() == 5 + 7 + 3
    assert list(descs["row_map"]) == [1, -1, 5 + 3, 5 + 7 + 0, -1]
    assert sb.n_tasks == sum(len(p[1]) for p in parts)
    d_of_seg = {0: {0, 1}, 1: {2}, 2: {3, 4}}
    for t in tasks:
        assert int(t["desc"]) in d_of_seg[int(t["seg"])]
    # round-robin: the first len(parts) tasks come from different parts
    assert sorted(int(s) for s in tasks["seg"][:3]) == [0, 1, 2]
    with pytest.raises(Exception):
        models.SliceBatch([parts[0]] * 65, torch.device("cpu"))


def test_adam_bias_table_is_the_reference_arithmetic():
    """engine.adam_bias_rows: row t = (1 - beta1**t, 1 - beta2**t) computed as
    optim.py:107-108 does (Python float pow), ending at the first t where
    both are exactly 1.0 (the kernel clamps later steps there)."""
    from paper_2507_09029_b200 import engine, train
    tab = engine.adam_bias_rows(0.9, 0.999)
    for t in range(0, len(tab), 997):
        assert tab[t, 0] == 1 - 0.9 ** t and tab[t, 1] == 1 - 0.999 ** t
    assert (tab[-1] == 1.0).all() and not (tab[-2] == 1.0).all()
    assert 30000 < len(tab) < 60000
    with pytest.raises(Exception, match="unknown optimizer"):
        train._check_optimizer("lamb")
