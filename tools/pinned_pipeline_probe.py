"""Pinned host inputs: the zero-copy sync (SM loads over PCIe) vs a chunked
copy-engine pipeline (owned ranges H2D per chunk, sync, D2H of the mean) at
C2 and C4.  Probe-only (gpurun)."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2507_09029_b200 import engine, masking, zoo  # noqa: E402

dev = torch.device("cuda", 0)


def tm(f, n):
    f()
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return float(np.mean(ts)) * 1e3, float(np.min(ts)) * 1e3


for tag, topo, reps in (("C2", zoo.resnet18_cifar_topology(), 20), ("C4", zoo.gpt2_small_topology(), 8)):
    a = masking.build_assignment(topo, "block", 8, 4, seed=1)
    d = topo.total
    pm = a.param_masks
    hosts = []
    for w in range(8):
        t = torch.empty(d, pin_memory=True)
        t.copy_(torch.randn(d, device=dev) * pm[w])
        hosts.append(t)
    del pm
    nbytes = a.sync_plan().owned_elems * 4
    ref = engine.aggregate([h.numpy() for h in hosts], a).gbar.copy()
    ms, mn = tm(lambda: engine.aggregate([h.numpy() for h in hosts], a), reps)
    print(json.dumps({"cfg": tag, "path": "zero-copy", "ms": round(ms, 2), "ms_min": round(mn, 2),
                      "GBps": round(nbytes / ms / 1e6, 1)}), flush=True)
    for mb in (32, 64, 128, 256):
        f = lambda: engine._host_staged(None, a, False, pinned=hosts, chunk_bytes=mb << 20)  # noqa: E731
        g = f().gbar
        assert np.array_equal(g.view(np.uint32), ref.view(np.uint32))
        ms, mn = tm(f, reps)
        print(json.dumps({"cfg": tag, "path": f"copy pipeline {mb} MB chunks", "ms": round(ms, 2),
                          "ms_min": round(mn, 2), "GBps": round(nbytes / ms / 1e6, 1)}), flush=True)
    del hosts
