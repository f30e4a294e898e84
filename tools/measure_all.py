"""Measure every libsdp kernel at the BASELINE configs on one B200 (gpurun).

    python tools/measure_all.py [--quick] > profiles/rN_measure.jsonl

One JSON line per (kernel, config): mean CUDA-event time per launch over
`reps` launches with a cold, clean L2 before each (256 MB write + 256 MB
read), the algorithmic bytes of one launch and the fraction of
MEASURED_PEAKS.json hbm_gbs they imply.  Also times the CPU reference port
(numpy f64 engine.aggregate, 1 thread) on the sweep points <= 64 MiB.
"""

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2507_09029_b200 import _native as N  # noqa: E402
from paper_2507_09029_b200 import engine, masking, models, zoo  # noqa: E402
from paper_2507_09029_b200._device import ptr, stream_ptr  # noqa: E402

PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
DEV = torch.device("cuda", 0)
FLUSH_W = None
FLUSH_R = None


def flush():
    FLUSH_W.zero_()
    FLUSH_R.sum()


def timed(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return float(np.mean(ts)), float(np.min(ts))


def emit(kernel, config, us, us_min, nbytes, **extra):
    gbs = nbytes / us / 1e3
    print(json.dumps({"kernel": kernel, "config": config, "us": round(us, 2), "us_min": round(us_min, 2),
                      "alg_bytes": int(nbytes), "GBps": round(gbs, 1), "frac_hbm": round(gbs / PEAK, 3),
                      **extra}), flush=True)


def sync_case(topo, tag, strategy, n, p, writeback=True, shadows=True, tile=None, reps=20,
              sync_layout=False, **plan_kw):
    a = masking.build_assignment(topo, strategy, n, p, seed=1)
    d = topo.total
    pm = a.param_masks
    gen = torch.Generator(device=DEV)
    reps_t = []
    for w in range(n):
        gen.manual_seed(1000 + w)
        reps_t.append(torch.randn(d, generator=gen, device=DEV) * pm[w])
    del pm
    sh = [torch.zeros(d, dtype=torch.bfloat16, device=DEV) for _ in range(n)] if shadows else None
    out = None if writeback else torch.empty(d, device=DEV)
    if sync_layout:
        from paper_2507_09029_b200.layout import SyncLayout
        lay = SyncLayout(a)
        reps_t = [lay.to_sync(r) for r in reps_t]
        plan = lay.plan(tile=tile, **plan_kw)
    else:
        plan = a.sync_plan(tile=tile, **plan_kw)
    prep = engine.PreparedSync(reps_t, a, writeback=writeback, shadows_bf16=sh, out=out, plan=plan)
    us, us_min = timed(prep.launch, reps=reps)
    own = plan.owned_elems
    mixed = plan.n_tiles - plan.n_uniform
    nbytes = own * 4 + (own * (4 + (2 if shadows else 0)) if writeback else d * 4) + mixed * plan.tile
    emit("k_owner_sync", tag, us, us_min, nbytes, strategy=strategy, n=n, p=p, d=d,
         mode="replica writeback" + (" + bf16" if shadows else "") if writeback else "aggregate (out)",
         tile=plan.tile, tiles=plan.n_tiles, mixed_tiles=mixed, grid=plan.grid,
         sync_GBps=round(own * 4 / us / 1e3, 1))
    return a, reps_t


def build_case(topo, tag, strategy, n, p, with_pm=False):
    dev = DEV
    tables = masking._DeviceTables(topo, strategy, dev)
    t = tables.table
    ub = masking._device_assign(t.groups, t.n_units, n, p, 1, dev)

    def go():
        masking._expand(topo, tables, ub, n, dev, want_param_masks=with_pm)

    us, us_min = timed(go, reps=10)
    d = topo.total
    nbytes = d * (1 + 8 + 8 + 8) + (n * d if with_pm else 0)
    emit("k_build_masks", tag, us, us_min, nbytes, strategy=strategy, n=n, p=p, d=d,
         outputs="owner_mask+coverage+divisor+governors" + ("+[N,d] bool" if with_pm else ""))

    def assign():
        masking._device_assign(t.groups, t.n_units, n, p, 1, dev)

    us, us_min = timed(assign, reps=5)
    emit("k_assign", tag, us, us_min, 0, strategy=strategy, units=t.n_units, groups=len(t.groups))


def slices_case(topo, tag, strategy, n, p):
    a = masking.build_assignment(topo, strategy, n, p, seed=1)
    theta = torch.randn(topo.total, device=DEV)
    sub = models.SubnetLayout(a, 0)
    comp = torch.empty(sub.compact_total, device=DEV)
    us, us_min = timed(lambda: sub.gather(theta, comp))
    emit("k_gather", tag, us, us_min, sub.compact_total * 8, compact=sub.compact_total, d=topo.total)
    full = torch.empty(topo.total, device=DEV)
    us, us_min = timed(lambda: sub.scatter(comp, full))
    emit("k_scatter(zero-fill)", tag, us, us_min, sub.compact_total * 4 + topo.total * 4,
         compact=sub.compact_total, d=topo.total)
    us, us_min = timed(lambda: sub.scatter(comp, full, accumulate=True))
    emit("k_scatter(accumulate)", tag, us, us_min, sub.compact_total * 12, compact=sub.compact_total,
         d=topo.total)
    # all N workers in ONE launch (models.SliceBatch): what the co-resident trainer runs
    subs = [models.SubnetLayout(a, w) for w in range(n)]
    tot = sum(s_.compact_total for s_ in subs)
    gb = models.SliceBatch([s_.host_gather for s_ in subs], DEV)
    sb = models.SliceBatch([s_.host_scatter for s_ in subs], DEV)
    comps = [torch.empty(max(1, s_.compact_total), device=DEV) for s_ in subs]
    fulls = [torch.empty(topo.total, device=DEV) for _ in subs]
    us, us_min = timed(lambda: gb.gather([theta] * n, comps))
    emit("k_gather(all workers)", tag, us, us_min, tot * 8, compact=tot, d=topo.total, n=n)
    us, us_min = timed(lambda: sb.scatter(comps, fulls))
    emit("k_scatter(zero-fill, all workers)", tag, us, us_min, tot * 4 + n * topo.total * 4, compact=tot,
         d=topo.total, n=n)
    us, us_min = timed(lambda: sb.scatter(comps, fulls, accumulate=True))
    emit("k_scatter(accumulate, all workers)", tag, us, us_min, tot * 12, compact=tot, d=topo.total, n=n)
    del fulls
    view = a.worker_view(0)
    out = torch.empty_like(theta)
    us, us_min = timed(lambda: N.call("sdp_masked_extract", 0, ptr(theta), ptr(view.param_mask_bool), 1,
                                      topo.total, 0, ptr(out), stream_ptr(DEV)))
    emit("k_masked_extract", tag, us, us_min, topo.total * 9, d=topo.total)
    if strategy == "neuron":
        # what width-wise training runs: flat <-> sync layout, compact <-> sync blocks
        from paper_2507_09029_b200.layout import SyncLayout, WorkerTransfer
        lay = SyncLayout(a)
        ts = torch.empty_like(theta)
        us, us_min = timed(lambda: lay.to_sync(theta, ts))
        emit("k_gather(to_sync)", tag, us, us_min, topo.total * 8, d=topo.total)
        us, us_min = timed(lambda: lay.from_sync(ts, theta))
        emit("k_gather(from_sync, reverse)", tag, us, us_min, topo.total * 8, d=topo.total)
        trs = [WorkerTransfer(lay, s_) for s_ in subs]
        tb = models.SliceBatch([t.host for t in trs], DEV)
        grads = [torch.zeros(topo.total, device=DEV) for _ in subs]
        us, us_min = timed(lambda: tb.gather(comps, [ts] * n, reverse=True))
        emit("k_gather(to_compact, reverse, all workers)", tag, us, us_min, tot * 8, compact=tot, d=topo.total, n=n)
        us, us_min = timed(lambda: tb.gather(comps, grads))
        emit("k_gather(from_compact, all workers)", tag, us, us_min, tot * 8, compact=tot, d=topo.total, n=n)
        del grads
        tr = WorkerTransfer(lay, sub)
        us, us_min = timed(lambda: tr.to_compact(ts, comp))
        emit("k_gather(to_compact, reverse)", tag, us, us_min, sub.compact_total * 8,
             compact=sub.compact_total, d=topo.total)
        us, us_min = timed(lambda: tr.from_compact(comp, ts))
        emit("k_gather(from_compact)", tag, us, us_min, sub.compact_total * 8,
             compact=sub.compact_total, d=topo.total)


def cpu_case(topo, tag, n, p, budget=3.0):
    from oracle import oracle as O
    a = O.build_assignment(topo, "block", n, p, 1)
    rng = np.random.default_rng(0)
    grads = [rng.standard_normal(topo.total) * a.param_masks[w] for w in range(n)]
    t0 = time.perf_counter()
    k = 0
    while time.perf_counter() - t0 < budget or k == 0:
        O.aggregate_f64(grads, a.param_masks, a.divisor)
        k += 1
    dt = (time.perf_counter() - t0) / k
    own = int(a.coverage.sum())
    print(json.dumps({"kernel": "cpu reference port (numpy f64 engine.aggregate, 1 thread)", "config": tag,
                      "us": round(dt * 1e6, 1), "sync_GBps": round(own * 4 / dt / 1e9, 3), "calls": k,
                      "host_cores": os.cpu_count()}), flush=True)


def main():
    global FLUSH_W, FLUSH_R
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--only", default="build,sync,sweep,slices,cpu",
                    help="comma-separated sections to run")
    args = ap.parse_args()
    only = set(args.only.split(","))
    N.load()
    FLUSH_W = torch.empty(64 << 20, device=DEV)
    FLUSH_R = torch.zeros(64 << 20, device=DEV)
    r18, gpt2 = zoo.resnet18_cifar_topology(), zoo.gpt2_small_topology()
    if "build" in only:  # mask builder
        build_case(r18, "C2 resnet18", "block", 8, 4)
        build_case(r18, "C2 resnet18 +[N,d]", "block", 8, 4, with_pm=True)
        build_case(r18, "C3 resnet18", "neuron", 8, 4)
        build_case(gpt2, "C4 gpt2", "block", 8, 4)
        build_case(gpt2, "C4 gpt2 neuron", "neuron", 8, 4)
    if "sync" in only:
        sync_case(r18, "C2 resnet18", "block", 8, 4)
        sync_case(r18, "C2 resnet18", "block", 8, 4, writeback=False, shadows=False)
        sync_case(r18, "C3 resnet18", "neuron", 8, 4)
        sync_case(r18, "C3 resnet18", "neuron", 8, 4, writeback=False, shadows=False)
        sync_case(r18, "C3 resnet18 (sync layout)", "neuron", 8, 4, sync_layout=True)
        sync_case(gpt2, "C4 gpt2", "block", 8, 4)
        sync_case(gpt2, "C4 gpt2 width-wise (sync layout)", "neuron", 8, 4, sync_layout=True)
        sync_case(gpt2, "C4 gpt2 width-wise", "neuron", 8, 4, writeback=False, shadows=False)
    if "sweep" in only:
        sizes = [1, 16, 256] if args.quick else [1, 4, 16, 64, 256, 1024]
        for mib in sizes:
            for p in (2, 4, 8):
                sync_case(zoo.sweep_topology(mib * (1 << 20) // 4), f"C5 sweep {mib} MiB", "block", 8, p)
                torch.cuda.empty_cache()
    if "sweep" in only:  # neuron variant, fragmented / uncovered owner sets
        mr = zoo.mini_resnet_topology(512, 8, 10, 2, 3, (8, 8))
        for p in (2, 4, 8):
            sync_case(mr, "C5 neuron mini-ResNet c=512 K=8", "neuron", 8, p)
            sync_case(mr, "C5 neuron mini-ResNet c=512 K=8 (sync layout)", "neuron", 8, p, sync_layout=True)
    if "slices" in only:  # width-wise extraction / write-back
        slices_case(r18, "C3 resnet18", "neuron", 8, 4)
        slices_case(gpt2, "C4 gpt2 (mlp units)", "neuron", 8, 4)
    if "cpu" in only and not args.no_cpu:
        for mib in (1, 16, 64):
            cpu_case(zoo.sweep_topology(mib * (1 << 20) // 4), f"C5 sweep {mib} MiB P=4", 8, 4)


if __name__ == "__main__":
    main()
