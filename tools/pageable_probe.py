"""Tune the pageable host path of engine.aggregate at C4 (GPT-2, N=8, P=4):
host memcpy ceiling (pageable -> pinned, T threads) and aggregate() time per
staging chunk size / slot count / thread count.  Probe-only (gpurun)."""
import concurrent.futures
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2507_09029_b200 import engine, masking, zoo  # noqa: E402

dev = torch.device("cuda", 0)
topo = zoo.gpt2_small_topology()
d = topo.total
a = masking.build_assignment(topo, "block", 8, 4, seed=1)
pm = a.param_masks
grads = [(torch.randn(d, device=dev) * pm[w]).cpu().numpy() for w in range(8)]
del pm
owned = a.sync_plan().owned_elems * 4

# memcpy ceiling: 2 GB pageable -> pinned in 4 MB pieces on T threads
src = np.concatenate(grads[:4])[: 512 << 20]
dst = torch.empty(src.size, dtype=torch.float32, pin_memory=True).numpy()
for threads in (4, 8, 16, 32):
    pool = concurrent.futures.ThreadPoolExecutor(threads)
    piece = 1 << 20
    jobs = range(0, src.size, piece)
    list(pool.map(lambda i: np.copyto(dst[i:i + piece], src[i:i + piece]), jobs))
    t0 = time.perf_counter()
    list(pool.map(lambda i: np.copyto(dst[i:i + piece], src[i:i + piece]), jobs))
    dt = time.perf_counter() - t0
    print(json.dumps({"memcpy_threads": threads, "GBps": round(src.nbytes / dt / 1e9, 1)}), flush=True)
    pool.shutdown()

for threads in (8, 16, 32):
    engine._COPY_POOL = concurrent.futures.ThreadPoolExecutor(threads)
    for mb in (32, 64, 128, 256):
        for slots in (2, 3, 4):
            engine.STAGE_CHUNK_BYTES, engine.STAGE_SLOTS = mb << 20, slots
            engine._STAGING.clear()
            engine.aggregate(grads, a)
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                engine.aggregate(grads, a)
                ts.append(time.perf_counter() - t0)
            ms = sorted(ts)[1] * 1e3
            print(json.dumps({"threads": threads, "chunk_MB": mb, "slots": slots, "ms": round(ms, 1),
                              "GBps": round(owned / ms / 1e6, 1)}), flush=True)
