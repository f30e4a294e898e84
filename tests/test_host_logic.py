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
