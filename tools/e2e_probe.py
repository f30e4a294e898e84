"""Break down the host-buffer aggregate (bench.py's e2e leg) on one B200.

    python tools/e2e_probe.py

Raw pinned H2D / D2H / bidirectional copy bandwidth, the owned-range H2D the
aggregate issues, and engine.aggregate at several pipeline depths.
"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2507_09029_b200 import engine, masking, zoo  # noqa: E402

dev = torch.device('cuda', 0)
topo = zoo.resnet18_cifar_topology()
d = topo.total
a = masking.build_assignment(topo, 'block', 8, 4, seed=1)
host = []
for w in range(8):
    t = torch.empty(d, pin_memory=True)
    t.normal_()
    host.append(t.numpy())
dst = [torch.empty(d, device=dev) for _ in range(8)]


def tm(f, n=10):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


big_h = torch.empty(64 << 20, pin_memory=True)
big_d = torch.empty(64 << 20, device=dev)
ms = tm(lambda: big_d.copy_(big_h, non_blocking=True))
print(f'H2D 256 MiB one copy: {ms:.3f} ms  {256 * 2**20 / ms / 1e6:.1f} GB/s')
ms = tm(lambda: big_h.copy_(big_d, non_blocking=True))
print(f'D2H 256 MiB one copy: {ms:.3f} ms  {256 * 2**20 / ms / 1e6:.1f} GB/s')
s2 = torch.cuda.Stream(dev)
big_h2 = torch.empty(64 << 20, pin_memory=True)
big_d2 = torch.empty(64 << 20, device=dev)


def bidir():
    big_d.copy_(big_h, non_blocking=True)
    with torch.cuda.stream(s2):
        big_h2.copy_(big_d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


ms = tm(bidir)
print(f'bidirectional 256+256 MiB: {ms:.3f} ms  {512 * 2**20 / ms / 1e6:.1f} GB/s total')
plan = a.sync_plan()
rng = [plan.worker_ranges(w) for w in range(8)]
owned = sum(ln for r in rng for _, ln in r) * 4
print('ranges per worker', [len(r) for r in rng], 'owned H2D bytes', owned)
ms = tm(lambda: [dst[w].copy_(torch.from_numpy(host[w]), non_blocking=True) for w in range(8)])
print(f'8 full H2D: {ms:.3f} ms  {8 * d * 4 / ms / 1e6:.1f} GB/s')
ms = tm(lambda: [dst[w][s:s + ln].copy_(torch.from_numpy(host[w])[s:s + ln], non_blocking=True)
                 for w in range(8) for s, ln in rng[w]])
print(f'owned-range H2D: {ms:.3f} ms  {owned / ms / 1e6:.1f} GB/s')
for mb in (16, 32, 64, 128):
    engine.STAGE_CHUNK_BYTES = mb << 20
    ms = tm(lambda: engine.aggregate([np.array(h) for h in host], a))
    print(f'pageable aggregate, {mb} MB chunks: {ms:.3f} ms  e2e {plan.owned_elems * 4 / ms / 1e6:.1f} GB/s')
engine.STAGE_CHUNK_BYTES = 64 << 20
t0 = time.perf_counter()
for _ in range(10):
    engine.aggregate(host, a)
print('host-side per call (incl. sync) ms', (time.perf_counter() - t0) / 10 * 1e3)

# zero-copy experiment: k_owner_sync reads the pinned host gradients over PCIe
# and writes the mean straight into pinned host memory (no staging copies)
import ctypes as C  # noqa: E402

from paper_2507_09029_b200 import _native as N  # noqa: E402

hp = [torch.from_numpy(h) for h in host]
print('inputs pinned:', all(t.is_pinned() for t in hp))
out_h = torch.empty(d, pin_memory=True)
for tl in (2048, 8192):
    zplan = a.sync_plan(tile=tl)
    args = zplan.args(N.DTYPE_F32)
    for w in range(8):
        args.replicas[w] = hp[w].data_ptr()
    args.out = out_h.data_ptr()
    args.flags = 0
    fn = N.lib().sdp_owner_sync

    def zc():
        rc = fn(C.byref(args), C.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert rc == 0, N.lib().sdp_last_error()
        torch.cuda.current_stream().synchronize()

    ms = tm(zc)
    ref = engine.aggregate(host, a).gbar
    print(f'zero-copy sync tile {tl} grid {zplan.grid}: {ms:.3f} ms  e2e {plan.owned_elems * 4 / ms / 1e6:.1f} GB/s',
          'bit-exact' if np.array_equal(out_h.numpy().view(np.uint32), ref.view(np.uint32)) else 'MISMATCH')

# hybrid: copy-engine H2D of the owned ranges in chunks, the sync of each chunk
# writing the mean straight into pinned host memory (no D2H stage)
s_in = torch.cuda.Stream(dev)
reps_d = [torch.empty(d, device=dev) for _ in range(8)]
full = a.sync_plan()
tile = full.tile
n_tiles = len(full.all_tiles)


def hybrid(k):
    bounds = [n_tiles * c // k for c in range(k + 1)]
    cur = torch.cuda.current_stream()
    s_in.wait_stream(cur)
    for c in range(k):
        lo_e, hi_e = bounds[c] * tile, min(d, bounds[c + 1] * tile)
        with torch.cuda.stream(s_in):
            for w in range(8):
                for st, ln in full.worker_ranges(w):
                    x0, x1 = max(st, lo_e), min(st + ln, hi_e)
                    if x0 < x1:
                        reps_d[w][x0:x1].copy_(hp[w][x0:x1], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(s_in)
        cur.wait_event(ev)
        plan = a.sync_plan(tile=tile, tile_lo=bounds[c], tile_hi=bounds[c + 1])
        engine.owner_sync(reps_d, a, out=out_h, writeback=False, plan=plan, zero_copy=True)
    cur.synchronize()


for k in (4, 8, 16, 32):
    ms = tm(lambda: hybrid(k))
    ref = engine.aggregate(host, a).gbar
    ok = np.array_equal(out_h.numpy().view(np.uint32), ref.view(np.uint32))
    print(f'hybrid copy-engine H2D + zero-copy output, {k} chunks: {ms:.3f} ms  e2e {plan.owned_elems * 4 / ms / 1e6:.1f} GB/s',
          'bit-exact' if ok else 'MISMATCH')

# where does the hybrid lose time?  (a) the same pipeline writing the mean to a
# DEVICE buffer (no PCIe writes), (b) pinned output; host issue time per call
out_d = torch.empty(d, device=dev)
plans = {}


def hybrid2(k, out):
    bounds = [n_tiles * c // k for c in range(k + 1)]
    cur = torch.cuda.current_stream()
    s_in.wait_stream(cur)
    for c in range(k):
        lo_e, hi_e = bounds[c] * tile, min(d, bounds[c + 1] * tile)
        with torch.cuda.stream(s_in):
            for w in range(8):
                for st, ln in full.worker_ranges(w):
                    x0, x1 = max(st, lo_e), min(st + ln, hi_e)
                    if x0 < x1:
                        reps_d[w][x0:x1].copy_(hp[w][x0:x1], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(s_in)
        cur.wait_event(ev)
        plan = a.sync_plan(tile=tile, tile_lo=bounds[c], tile_hi=bounds[c + 1])
        engine.owner_sync(reps_d, a, out=out, writeback=False, plan=plan, zero_copy=True)


for k in (4, 8):
    for name, o in (("device out", out_d), ("pinned out", out_h)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hybrid2(k, o)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        ms = tm(lambda: hybrid2(k, o))
        print(f'hybrid2 {k} chunks, {name}: {ms:.3f} ms (host issue {1e3 * (t1 - t0):.3f} ms of {1e3 * (t2 - t0):.3f})')
# copies only (same chunking), no kernels
for k in (1, 4, 8):
    def copies_only():
        bounds = [n_tiles * c // k for c in range(k + 1)]
        with torch.cuda.stream(s_in):
            for c in range(k):
                lo_e, hi_e = bounds[c] * tile, min(d, bounds[c + 1] * tile)
                for w in range(8):
                    for st, ln in full.worker_ranges(w):
                        x0, x1 = max(st, lo_e), min(st + ln, hi_e)
                        if x0 < x1:
                            reps_d[w][x0:x1].copy_(hp[w][x0:x1], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s_in)
    print(f'owned-range H2D in {k} chunks: {tm(copies_only):.3f} ms')
