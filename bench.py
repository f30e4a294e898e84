"""Benchmark of the owner-subset sync (engine.aggregate, engine.py:60-79) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload resnet18|gpt2|sweep:<MiB>] [--p P]

A step = one owner-subset sync of the BASELINE configs[1] workload: ResNet-18
(CIFAR shape, d = 11,173,962), block dropping, N = 8 logical workers, P = 4,
seed 1.  At --gpus 1 the 8 worker replicas are co-resident in one HBM (the
reference's own in-process structure) and one k_owner_sync launch reads every
element from its owners, sums in ascending owner order in fp32, divides by the
owner count and writes the mean back into every owner's fp32 replica and bf16
training copy.  At --gpus G > 1 (torchrun) the 8 workers are placed
contiguously on the G GPUs and the same kernel reads/writes peer replicas over
NVLink (paper_2507_09029_b200/comm.py).

metric "subnet-sync GB/s": replica gradient bytes synchronised per second,
sum over elements j of |O_j| * 4 B (fp32-equivalent) / time -- the same count
for every arm, every N and the CPU reference.
"""

from __future__ import annotations

import argparse
import concurrent.futures
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "subnet-sync GB/s (owner-subset replica bytes synchronised per second)"
UNIT = "GB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="resnet18")
    ap.add_argument("--n-logical", type=int, default=8)
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--strategy", default="block")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-train", action="store_true")
    ap.add_argument("--train-steps", type=int, default=10)
    return ap.parse_args()


def workload(name: str):
    from paper_2507_09029_b200 import zoo
    if name == "resnet18":
        return zoo.resnet18_cifar_topology(), "resnet18-cifar (configs[1], C2)"
    if name == "gpt2":
        return zoo.gpt2_small_topology(), "gpt2-small 124M (configs[3], C4)"
    if name == "c1":  # the reference's own CPU-runnable case; use --n-logical 4 --p 2
        return (zoo.mini_resnet_topology(26, 8, 10, 2, 3, (32, 32)),
                "mini-ResNet 26ch x 8 blocks (configs[0], C1)")
    if name.startswith("sweep:"):
        mib = int(name.split(":")[1])
        return zoo.sweep_topology(mib * (1 << 20) // 4), f"sweep {mib} MiB fp32 (configs[4], C5)"
    raise SystemExit(f"unknown workload {name}")


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "_fallback": True}


def traffic_for(tag: str):
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        return json.loads(p.read_text()).get(tag)
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.15)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.06)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference arm: the reference algorithm (engine.py:71-74) ported to numpy
# f64 (oracle/oracle.py, verified bit-exact against the reference), split
# over host threads by contiguous element ranges.
# ---------------------------------------------------------------------------

def cpu_aggregate_threads(grads, masks, divisor, lo, hi, threads):
    chunks = np.linspace(lo, hi, threads + 1).astype(np.int64)
    out = np.empty(hi - lo, dtype=np.float64)

    def run(k):
        a, b = chunks[k], chunks[k + 1]
        from oracle.oracle import aggregate_f64
        out[a - lo:b - lo] = aggregate_f64([g[a:b] for g in grads], masks[:, a:b], divisor[a:b])

    if threads == 1:
        run(0)
    else:
        with concurrent.futures.ThreadPoolExecutor(threads) as ex:
            list(ex.map(run, range(threads)))
    return out


def host_workload(topo, strategy, n, p, seed=1):
    from oracle import oracle as O
    a = O.build_assignment(topo, strategy, n, p, seed)
    rng = np.random.default_rng(1000)
    grads = [(rng.standard_normal(topo.total, dtype=np.float32) * a.param_masks[w]).astype(np.float64)
             for w in range(n)]
    owned = int(a.coverage.sum())
    return a, grads, owned


def time_cpu(grads, masks, divisor, owned_per_elem, threads, budget_s, max_reps=1000):
    """Bounded sample: whole-vector calls until the budget is spent (>= 1 call);
    if one call exceeds the budget, a contiguous prefix sized to fit."""
    d = masks.shape[1]
    t0 = time.perf_counter()
    cpu_aggregate_threads(grads, masks, divisor, 0, min(d, 1 << 20), threads)
    est = (time.perf_counter() - t0) * d / min(d, 1 << 20)
    hi = d if est <= budget_s else max(1 << 16, int(d * budget_s / est))
    reps = max(1, min(max_reps, int(budget_s / max(est * hi / d, 1e-6))))
    t0 = time.perf_counter()
    for _ in range(reps):
        cpu_aggregate_threads(grads, masks, divisor, 0, hi, threads)
    dt = (time.perf_counter() - t0) / reps
    nbytes = float(owned_per_elem[:hi].sum()) * 4
    return nbytes / dt / 1e9, dt, hi, reps


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    topo, tag = workload(args.workload)
    a, grads, owned = host_workload(topo, args.strategy, args.n_logical, args.p)
    threads = os.cpu_count() or 1
    per_elem = a.coverage
    # size each step so warmup + steps end within ~2 minutes
    budget_total = 120.0
    d = topo.total
    t0 = time.perf_counter()
    cpu_aggregate_threads(grads, a.param_masks, a.divisor, 0, min(d, 1 << 20), threads)
    est_full = (time.perf_counter() - t0) * d / min(d, 1 << 20)
    per_step = budget_total / max(1, args.steps + args.warmup)
    hi = d if est_full <= per_step else max(1 << 16, int(d * per_step / est_full))
    for _ in range(args.warmup):
        cpu_aggregate_threads(grads, a.param_masks, a.divisor, 0, hi, threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cpu_aggregate_threads(grads, a.param_masks, a.divisor, 0, hi, threads)
        times.append(time.perf_counter() - t0)
    dt = float(np.mean(times))
    nbytes = float(per_elem[:hi].sum()) * 4
    value = nbytes / dt / 1e9
    sample = (f"{'whole vector' if hi == d else f'first {hi} of {d} elements'} per step; "
              f"numpy f64 port of engine.aggregate (oracle/oracle.py:aggregate_f64), "
              f"{threads} threads over contiguous element ranges")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": tag, "d": d, "n_logical": args.n_logical, "p": args.p,
                   "strategy": args.strategy, "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2507_09029_b200 import _native, engine, masking

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: every rank on GPU 0 (CUDA IPC within one device) with gloo plumbing
    if os.environ.get("SDP_BENCH_SAME_DEVICE") == "1":
        local = 0
    backend = os.environ.get("SDP_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _native.load()
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    red_dev = dev if backend == "nccl" else torch.device("cpu")  # where small all-reduces run
    topo, tag = workload(args.workload)
    n, p, d = args.n_logical, args.p, topo.total
    a = masking.build_assignment(topo, args.strategy, n, p, seed=1)

    if world > 1:
        from paper_2507_09029_b200 import comm
        step, plan_bytes, hbm_bytes, meta = comm.bench_setup(a, rank, world, dev)
        parallelism = f"{n} logical workers on {world} GPUs, NVLink P2P owner sync"
    else:
        pm = a.param_masks
        gen = torch.Generator(device=dev)
        reps, shadows = [], []
        for w in range(n):
            gen.manual_seed(1000 + w)
            reps.append(torch.randn(d, generator=gen, device=dev) * pm[w])
            shadows.append(torch.zeros(d, dtype=torch.bfloat16, device=dev))
        plan = a.sync_plan()
        prep = engine.PreparedSync(reps, a, writeback=True, shadows_bf16=shadows, plan=plan)
        step = prep.launch
        plan_bytes = plan.owned_elems * 4
        hbm_bytes = plan.owned_elems * (4 + 4 + 2)   # read fp32, write fp32 + bf16 per owner
        meta = {"tiles": plan.n_tiles, "uniform_tiles": plan.n_uniform, "grid": plan.grid,
                "tiles_per_cta": plan.tiles_per_cta}
        parallelism = f"{n} logical workers co-resident on 1 GPU"
        del pm

    # L2 flush between timed launches: write 256 MB (> 126 MB L2), then read
    # another 256 MB so the lines left behind are clean -- otherwise the timed
    # kernel pays for evicting the flush's dirty lines.
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    flush_rd = torch.zeros(64 << 20, dtype=torch.float32, device=dev)

    def flush_l2():
        flush.zero_()
        flush_rd.sum()

    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        step()
        flush_l2()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            starts[i].record(stream)
            step()
            ends[i].record(stream)
            flush_l2()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times = np.array([s.elapsed_time(e) for s, e in zip(starts, ends)])  # ms
    ms = float(times.mean())
    if world > 1:
        t = torch.tensor([ms], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # the step time is the slowest rank's
        ms = float(t.item())
        tot = torch.tensor([float(plan_bytes)], device=red_dev, dtype=torch.float64)
        dist.all_reduce(tot)
        total_bytes = float(tot.item())
    else:
        total_bytes = float(plan_bytes)
    value = total_bytes / (ms / 1e3) / 1e9

    peaks = measured_peaks()
    peak = float(peaks["hbm_gbs"])
    achieved = hbm_bytes / (float(times.mean()) / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic_for(f"{args.workload}:{world}"),
                "kernel": "k_owner_sync",
                "algorithmic_bytes_per_launch": hbm_bytes,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, read+write)"
                if not peaks.get("_fallback") else "fallback 6.65 TB/s (B200_PROFILING.md)"}
    if world > 1:
        roofline.update(meta.get("roofline", {}))
        # per direction each GPU carries ~ its own peer reads + peer writes
        # (peers write into it what it writes to them); measured P2P peak 770 GB/s
        nvl = meta.get("roofline", {}).get("nvlink_bytes_per_launch", 0)
        roofline["nvlink_achieved_GBps"] = nvl / (float(times.mean()) / 1e3) / 1e9
        roofline["nvlink_peak_GBps"] = 770.0
        roofline["nvlink_frac"] = roofline["nvlink_achieved_GBps"] / 770.0
        roofline["nvlink_peak_source"] = "B200_PROFILING.md measured peer copy per direction (900 nominal)"
        probe = meta.get("roofline", {}).get("p2p_copy_GBps_measured")
        if probe:  # this run's own ring peer-copy probe (all ranks at once)
            roofline["nvlink_frac_of_run_probe"] = roofline["nvlink_achieved_GBps"] / probe

    e2e = None
    cpu = None
    train = None
    builder = None
    if world > 1 and not args.no_train and args.workload == "resnet18":
        train = run_train_multi(args, dev, rank, world, red_dev)
    if rank == 0 and world == 1:
        e2e = run_e2e(args, a, dev, total_bytes)
        if not args.no_train and args.workload == "resnet18":
            train = run_train(args, dev)
            train["c4_gpt2"] = run_train_gpt2(args, dev)
        if not args.no_train and args.workload == "c1":
            train = run_train_c1(args, dev)
        if not args.no_cpu_baseline:
            cpu = run_cpu_baseline(args, topo)
            builder = run_mask_builder(args, topo, dev)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp32 (bf16 copy fused)", "data": "synthetic",
            "config": {"workload": tag, "d": d, "n_logical": n, "p": p, "strategy": args.strategy,
                       "seed": 1, "parallelism": parallelism,
                       "l2": "flushed between steps: 256 MB write + 256 MB read (cold, clean L2)", **meta},
            "gpu_launches": args.steps,
            "roofline": roofline,
            "clocks": clocks.summary(),
        }
        if e2e:
            line["e2e"] = e2e
        if train:
            line["train"] = train
        if cpu:
            line["cpu_baseline"] = cpu
        if builder:
            line["mask_builder"] = builder
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def gpu_local_cpus(index: int):
    """CPU set NVML reports as local to the GPU (pinned host buffers allocated
    from a thread bound there sit on the GPU's NUMA node)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * i + b for i, wd in enumerate(words) for b in range(64) if wd >> b & 1}
        return sorted(c for c in cpus if c < os.cpu_count())
    except Exception:
        return None


def run_e2e(args, a, dev, total_bytes):
    """The reference-facing call with HOST buffers: engine.aggregate(list of N
    numpy arrays backed by pinned memory, assignment) -> numpy gbar.  H2D of all
    N gradients, the sync kernel, and the D2H of the mean are inside the timing."""
    import torch

    from paper_2507_09029_b200 import engine
    n, d = a.n_workers, a.topology.total
    cpus = gpu_local_cpus(dev.index)
    if cpus:
        os.sched_setaffinity(0, cpus)
    pm = a.param_masks
    gen = torch.Generator(device=dev)
    host = []
    for w in range(n):
        gen.manual_seed(1000 + w)
        t = torch.empty(d, dtype=torch.float32, pin_memory=True)
        t.copy_(torch.randn(d, generator=gen, device=dev) * pm[w])
        host.append(t.numpy())
    del pm
    out = None
    for _ in range(3):  # warm-up exactly like the timed loop (the previous result is held)
        out = engine.aggregate(host, a)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.e2e_steps):
        t0 = time.perf_counter()
        out = engine.aggregate(host, a)
        ts.append(time.perf_counter() - t0)
    assert out.gbar.shape == (d,)
    print("e2e per-call ms:", " ".join(f"{t * 1e3:.2f}" for t in ts), file=sys.stderr)
    dt = float(np.mean(ts))
    plan = a.sync_plan()
    h2d = sum(ln for w in range(n) for _, ln in plan.worker_ranges(w)) * 4 \
        if a.uncovered_params == 0 else n * d * 4
    return {"value": total_bytes / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d * 4, "ms_per_step": dt * 1e3,
            "api": "paper_2507_09029_b200.engine.aggregate(list[np.ndarray pinned], assignment)",
            "host_cpus": f"{len(cpus)} GPU-local cores (NVML affinity)" if cpus else "unpinned",
            "timing": "host wall clock around the blocking call (returns numpy)"}


def run_train(args, dev):
    """BASELINE metric parts 2-3: train samples/s/GPU and peak memory per GPU
    vs full-replica DP (configs[1]: ResNet-18, N=8, P=4, batch 64/worker).
    Workers are co-resident on this GPU; a step = 8 subnetwork fwd/bwd (bf16
    autocast, dropped blocks skipped) + one fused sync/Nesterov launch.  The DP
    comparator is the same loop with P = N (every worker holds the full model)."""
    import torch

    from paper_2507_09029_b200 import masking, train
    batch, n = 64, args.n_logical
    gen = torch.Generator(device=dev)
    gen.manual_seed(0)
    batches = [(torch.randn(batch, 3, 32, 32, generator=gen, device=dev),
                torch.randint(0, 10, (batch,), generator=gen, device=dev)) for _ in range(n)]
    out = {"workload": f"ResNet-18 CIFAR-shape, N={n} co-resident workers, batch {batch}/worker, "
                       "bf16 autocast fwd/bwd, fused sync+Nesterov+bf16 cast, whole step in one CUDA graph",
           "data": "synthetic"}
    for tag, p, strategy in (("subnet", args.p, "block"), ("widthwise", args.p, "neuron"), ("dp", n, "block")):
        model = train.build_resnet18(dev)
        a = masking.build_assignment(model.topology, strategy, n, p, seed=1)
        tr = train.SubnetTrainer(model, a, lr=0.02, sync_layout=(strategy == "neuron"), graphed=True)
        out[f"{tag}_loss_first"] = float(tr.step(batches).item())
        for _ in range(2):
            tr.step(batches)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.train_steps):
            loss = tr.step(batches)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / args.train_steps
        out[f"{tag}_ms_per_step"] = ms
        out[f"{tag}_samples_per_s_per_gpu"] = n * batch / (ms / 1e3)
        out[f"{tag}_loss_last"] = float(loss.item())
        mems = [train.worker_memory(model, a, w if p < n else None, batch, dev)["peak_bytes"]
                for w in (range(n) if p < n else [0])]
        out[f"{tag}_peak_mem_per_worker_bytes"] = max(mems)  # the GPU that needs the most
        out[f"{tag}_peak_mem_mean_bytes"] = float(np.mean(mems))  # the paper's per-worker average
        del tr, model, a
        torch.cuda.empty_cache()
    out["mem_reduction_vs_dp"] = 1 - out["subnet_peak_mem_per_worker_bytes"] / out["dp_peak_mem_per_worker_bytes"]
    out["mem_reduction_vs_dp_mean"] = 1 - out["subnet_peak_mem_mean_bytes"] / out["dp_peak_mem_per_worker_bytes"]
    out["speedup_vs_dp_per_step"] = out["dp_ms_per_step"] / out["subnet_ms_per_step"]
    out["widthwise_mem_reduction_vs_dp"] = (1 - out["widthwise_peak_mem_per_worker_bytes"]
                                            / out["dp_peak_mem_per_worker_bytes"])
    out["widthwise_mem_reduction_vs_dp_mean"] = (1 - out["widthwise_peak_mem_mean_bytes"]
                                                 / out["dp_peak_mem_per_worker_bytes"])
    out["configs"] = {"subnet": "configs[1] C2: block dropping P=4", "widthwise": "configs[2] C3: "
                      "channel-slice compact subnetworks (gather/scatter kernels) P=4",
                      "dp": "full-replica DP comparator (P=N)"}
    out["note"] = ("peak memory = one worker's compact fp32 master + grad + momentum + bf16 copy + "
                   "activations of its fwd/bwd, i.e. what a GPU holding that worker needs (N = G); "
                   "*_peak_mem_per_worker_bytes / mem_reduction_vs_dp: the largest worker (block "
                   "sizes are unequal: the window holding layer4.1 keeps most parameters); "
                   "*_mean: averaged over the N workers, as PAPER.md reports per-worker savings")
    return out


def run_train_c1(args, dev, batch: int = 8):
    """configs[0] C1, the reference's own CPU-runnable case: mini-ResNet 26 ch
    x 8 blocks at 32x32, N=4 co-resident workers, P=2, batch 8/worker, block
    dropping; DP comparator at P=N.  Graphed steps; the config is tiny
    (launch-bound), not a kernel number."""
    import torch

    from paper_2507_09029_b200 import masking, models, train
    n, p = args.n_logical, args.p
    gen = torch.Generator(device=dev)
    gen.manual_seed(7)
    batches = [(torch.randn(batch, 3, 32, 32, generator=gen, device=dev),
                torch.randint(0, 10, (batch,), generator=gen, device=dev)) for _ in range(n)]
    out = {"workload": f"mini-ResNet 26ch x 8 blocks 32x32, N={n} co-resident workers, P={p}, batch {batch}/worker, "
                       "bf16 autocast, fused sync+Nesterov+bf16 cast, whole step in one CUDA graph",
           "data": "synthetic (the reference uses its blobs dataset)"}
    for tag, pp in (("subnet", p), ("dp", n)):
        model = models.build_mini_resnet(26, 8, 10, 2, 3, (32, 32), seed=1, device_=dev)
        a = masking.build_assignment(model.topology, "block", n, pp, seed=1)
        tr = train.SubnetTrainer(model, a, lr=0.002, graphed=True)
        for _ in range(3):
            tr.step(batches)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.train_steps):
            loss = tr.step(batches)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / args.train_steps
        out[f"{tag}_ms_per_step"] = ms
        out[f"{tag}_samples_per_s_per_gpu"] = n * batch / (ms / 1e3)
        out[f"{tag}_loss_last"] = float(loss.item())
        del tr, model, a
        torch.cuda.empty_cache()
    out["reference_cpu_samples_per_s"] = 69.8
    out["reference_cpu_note"] = ("SURVEY.md §8(d)/F9: the reference's engine at C1 on N CPU threads in the survey "
                                 "container (the reference is not installed on the GPU box, so not re-timed here)")
    return out


def run_train_multi(args, dev, rank: int, world: int, red_dev):
    """Train samples/s/GPU at G > 1 GPUs (BASELINE metric part 2 at 2/4/8 GPUs):
    one process per GPU, the N = 8 workers placed contiguously (N/G per rank),
    train.PeerTrainer (local fwd/bwd, peer-mapped owner sync, local fused
    Nesterov + bf16 cast).  CUDA events over the timed steps, max over ranks;
    peak memory = the largest local worker's step (train.worker_memory), max
    over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2507_09029_b200 import masking, train

    def all_gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    def rmax(x: float) -> float:
        t = torch.tensor([float(x)], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    batch, n = 64, args.n_logical
    out = {"workload": f"ResNet-18 CIFAR-shape, N={n} workers on {world} GPUs ({n // world} per GPU), "
                       f"batch {batch}/worker, bf16 autocast, peer-mapped owner sync + local fused Nesterov/bf16, "
                       "each rank's step replayed from a CUDA graph",
           "data": "synthetic", "timing": "CUDA events per rank, max over ranks"}
    for tag, p, strategy in (("subnet", args.p, "block"), ("widthwise", args.p, "neuron"), ("dp", n, "block")):
        model = train.build_resnet18(dev)
        a = masking.build_assignment(model.topology, strategy, n, p, seed=1)
        tr = train.PeerTrainer(model, a, rank, world, dev, all_gather, lr=0.02, graphed=True)
        gen = torch.Generator(device=dev)
        batches = {}
        for w in tr.local:
            gen.manual_seed(w)
            batches[w] = (torch.randn(batch, 3, 32, 32, generator=gen, device=dev),
                          torch.randint(0, 10, (batch,), generator=gen, device=dev))
        out[f"{tag}_loss_first"] = rmax(tr.step(batches).item())
        tr.step(batches)
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.train_steps):
            loss = tr.step(batches)
        e.record()
        torch.cuda.synchronize()
        tr.group.check()
        ms = rmax(s.elapsed_time(e) / args.train_steps)
        dist.barrier()
        out[f"{tag}_ms_per_step"] = ms
        out[f"{tag}_samples_per_s_per_gpu"] = n * batch / (ms / 1e3) / world
        out[f"{tag}_loss_last"] = rmax(loss.item())
        mem = max(train.worker_memory(model, a, w if p < n else None, batch, dev)["peak_bytes"]
                  for w in (tr.local if p < n else tr.local[:1]))
        out[f"{tag}_peak_mem_per_worker_bytes"] = int(rmax(mem))
        tr.close()
        del tr, model, a
        torch.cuda.empty_cache()
        dist.barrier()
    out["mem_reduction_vs_dp"] = 1 - out["subnet_peak_mem_per_worker_bytes"] / out["dp_peak_mem_per_worker_bytes"]
    out["widthwise_mem_reduction_vs_dp"] = (1 - out["widthwise_peak_mem_per_worker_bytes"]
                                            / out["dp_peak_mem_per_worker_bytes"])
    out["speedup_vs_dp_per_step"] = out["dp_ms_per_step"] / out["subnet_ms_per_step"]
    # configs[3] C4 at G GPUs: GPT-2 small, seq 1024, micro-batch 8 per worker
    g4 = {"workload": f"GPT-2 small 124M, seq 1024, N={n} workers on {world} GPUs x micro-batch 8, "
                      "bf16 autocast, flash SDPA, fused LM-head cross-entropy", "data": "synthetic tokens"}
    for tag, p in (("subnet", args.p), ("dp", n)):
        model = train.build_gpt2(dev)
        a = masking.build_assignment(model.topology, "block", n, p, seed=1)
        tr = train.PeerTrainer(model, a, rank, world, dev, all_gather, lr=1e-4, loss_fn=train.lm_loss,
                               graphed=True)
        gen = torch.Generator(device=dev)
        batches = {}
        for w in tr.local:
            gen.manual_seed(w)
            t = torch.randint(0, 50257, (8, 1024), generator=gen, device=dev)
            batches[w] = (t, t)
        tr.step(batches)
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = max(2, args.train_steps // 2)
        s.record()
        for _ in range(steps):
            loss = tr.step(batches)
        e.record()
        torch.cuda.synchronize()
        tr.group.check()
        ms = rmax(s.elapsed_time(e) / steps)
        dist.barrier()
        g4[f"{tag}_ms_per_step"] = ms
        g4[f"{tag}_tokens_per_s_per_gpu"] = n * 8 * 1024 / (ms / 1e3) / world
        g4[f"{tag}_loss_last"] = rmax(loss.item())
        tr.close()
        del tr, model, a
        torch.cuda.empty_cache()
        dist.barrier()
    g4["speedup_vs_dp_per_step"] = g4["dp_ms_per_step"] / g4["subnet_ms_per_step"]
    out["c4_gpt2"] = g4
    return out


def run_train_gpt2(args, dev, micro_batch: int = 8, seq: int = 1024):
    """configs[3] C4: GPT-2 small, seq 1024, block dropping P=4, N=8 co-resident
    workers x micro-batch 8: tokens/s/GPU and peak memory per worker vs DP."""
    import torch

    from paper_2507_09029_b200 import masking, train
    n = args.n_logical
    gen = torch.Generator(device=dev)
    gen.manual_seed(0)
    batches = [(lambda t: (t, t))(torch.randint(0, 50257, (micro_batch, seq), generator=gen, device=dev))
               for _ in range(n)]
    out = {"workload": f"GPT-2 small 124M, seq {seq}, N={n} co-resident workers x micro-batch "
                       f"{micro_batch}, bf16 autocast, flash SDPA, fused sync+Nesterov+bf16, whole step in one "
                       "CUDA graph", "data": "synthetic tokens"}
    for tag, p in (("subnet", args.p), ("dp", n)):
        model = train.build_gpt2(dev)
        a = masking.build_assignment(model.topology, "block", n, p, seed=1)
        tr = train.SubnetTrainer(model, a, lr=1e-4, loss_fn=train.lm_loss, graphed=True)
        out[f"{tag}_loss_first"] = float(tr.step(batches).item())
        tr.step(batches)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = max(2, args.train_steps // 2)
        s.record()
        for _ in range(steps):
            loss = tr.step(batches)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / steps
        out[f"{tag}_ms_per_step"] = ms
        out[f"{tag}_tokens_per_s_per_gpu"] = n * micro_batch * seq / (ms / 1e3)
        out[f"{tag}_loss_last"] = float(loss.item())
        del tr
        torch.cuda.empty_cache()
        mk = lambda: (batches[0][0], batches[0][1])  # noqa: E731
        mems = [train.worker_memory(model, a, w if p < n else None, micro_batch, dev, mk, train.lm_loss)["peak_bytes"]
                for w in (range(n) if p < n else (0,))]
        out[f"{tag}_peak_mem_per_worker_bytes"] = max(mems)
        out[f"{tag}_peak_mem_mean_bytes"] = float(np.mean(mems))
        del model, a
        torch.cuda.empty_cache()
    out["mem_reduction_vs_dp"] = 1 - out["subnet_peak_mem_per_worker_bytes"] / out["dp_peak_mem_per_worker_bytes"]
    out["mem_reduction_vs_dp_mean"] = 1 - out["subnet_peak_mem_mean_bytes"] / out["dp_peak_mem_per_worker_bytes"]
    out["speedup_vs_dp_per_step"] = out["dp_ms_per_step"] / out["subnet_ms_per_step"]
    return out


def run_mask_builder(args, topo, dev):
    """build_assignment through the public API on the GPU (seeded
    assignment + element expansion + tables, synchronised) and its kernels
    alone, beside the CPU restatement of the reference's build_assignment on
    1 core -- checked bit-exact against each other."""
    import torch

    from oracle import oracle as O  # noqa: F401  (checker/baseline only)
    from paper_2507_09029_b200 import masking
    n, p = args.n_logical, args.p
    masking.build_assignment(topo, args.strategy, n, p, seed=1)
    torch.cuda.synchronize()
    api = []
    for _ in range(5):
        t0 = time.perf_counter()
        a = masking.build_assignment(topo, args.strategy, n, p, seed=1)
        torch.cuda.synchronize()
        api.append(time.perf_counter() - t0)
    tables = masking._DeviceTables(topo, args.strategy, dev)
    t = tables.table
    kern = {}
    for name, fn in (("k_assign", lambda: masking._device_assign(t.groups, t.n_units, n, p, 1, dev)),
                     ("k_build_masks", lambda: masking._expand(topo, tables, ub, n, dev))):
        ub = masking._device_assign(t.groups, t.n_units, n, p, 1, dev)
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            fn()
        e.record()
        torch.cuda.synchronize()
        kern[name] = s.elapsed_time(e) / 5 * 1e3
    t0 = time.perf_counter()
    o = O.build_assignment(topo, args.strategy, n, p, 1)
    cpu_s = time.perf_counter() - t0
    exact = bool(np.array_equal(a.owner_mask.cpu().numpy().astype(np.uint64), o.owner_bits)
                 and np.array_equal(a.coverage.cpu().numpy(), o.coverage))
    return {"workload": f"build_assignment({args.workload}, {args.strategy}, N={n}, P={p}, seed=1)",
            "api_ms": float(np.median(api)) * 1e3,
            "stage_us": {k: round(v, 1) for k, v in kern.items()},
            "stage_timing": "CUDA events around each stage's host call (k_assign includes its group-table "
                            "upload; ncu kernel time 8 us)",
            "cpu_restatement_ms": cpu_s * 1e3, "cpu_cores": 1,
            "cpu_kind": "port (oracle/oracle.py:build_assignment, numpy; the reference itself is not on the box)",
            "bit_exact": exact}


def run_cpu_baseline(args, topo):
    from oracle import oracle as O  # noqa: F401  (checker/baseline only)
    a, grads, owned = host_workload(topo, args.strategy, args.n_logical, args.p)
    value, dt, hi, reps = time_cpu(grads, a.param_masks, a.divisor, a.coverage, 1, budget_s=10.0)
    d = topo.total
    return {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{reps} calls over {'the whole vector' if hi == d else f'{hi} of {d} elements'}"
                      f", numpy f64 port of engine.aggregate on 1 thread (host has {os.cpu_count()} cores)",
            "ms_per_call": dt * 1e3}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
