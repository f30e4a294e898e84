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
    ap.add_argument("--workload", default="gpt2")
    ap.add_argument("--n-logical", type=int, default=8)
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--strategy", default="block")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-train", action="store_true")
    ap.add_argument("--train-steps", type=int, default=10)
    ap.add_argument("--no-memory-ranks", action="store_true")
    ap.add_argument("--equal-loss-steps", type=int, default=1500,
                    help="steps of the equal-compute subnet-vs-DP loss run (0: skip)")
    ap.add_argument("--memory-child", action="store_true", help=argparse.SUPPRESS)
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
    """SM clock + throttle reasons sampled DURING the timed region: NVML polled
    every 2 ms from a thread (the timed region of a 20-step sync run is only a
    few tens of ms; nvidia-smi -lms 50 caught one sample), nvidia-smi as the
    fallback."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, index: int):
        self.index = index
        self.sm: list[float] = []
        self.reasons: set = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def poll():
                get_r = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
                while not self._stop.is_set():
                    self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                    r = int(get_r(h))
                    for bit, nm in self.REASONS.items():
                        if r & bit:
                            self.reasons.add(nm)
                    time.sleep(0.002)

            self._t = threading.Thread(target=poll, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)

    def summary(self) -> dict:
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "NVML, 2 ms poll"}


# ---------------------------------------------------------------------------
# CPU reference arm: the reference's OWN engine.aggregate (engine.py:60-79),
# staged into oracle/_ref by oracle/build_ref.py (pure Python; it travels to
# the GPU box with the snapshot) and called unmodified.  numpy ufuncs run on
# one core, so the all-threads form hands each host thread a contiguous range
# of the vector, with a reference MaskAssignment over that range (its own
# constructor, masking.py:188-207) -- every element still goes through the
# reference's code.
# ---------------------------------------------------------------------------

def reference_pkg():
    from oracle import build_ref  # checker / baseline only
    return build_ref.import_reference()


def reference_assignment(topo, strategy: str, n: int, p: int, seed: int = 1):
    """The reference's build_assignment (masking.py:305-359) on the same
    topology, declared through the reference's own types."""
    from oracle import build_ref
    S = reference_pkg()
    return S.build_assignment(build_ref.to_reference_topology(topo), strategy, n, p, seed)


def reference_grads(a, hi: int, seed: int = 1000):
    """N float64 gradients over [0, hi): fp32 normals, zero off-mask (the
    reference's nullity), upcast as the reference takes them."""
    rng = np.random.default_rng(seed)
    return [(rng.standard_normal(hi, dtype=np.float32) * a.param_masks[w, :hi]).astype(np.float64)
            for w in range(a.n_workers)]


def reference_chunks(a, hi: int, parts: int):
    """Contiguous ranges of [0, hi) with a reference MaskAssignment each."""
    import types
    S = reference_pkg()
    MA = S.masking.MaskAssignment
    bounds = np.linspace(0, hi, parts + 1).astype(np.int64)
    out = []
    for lo, up in zip(bounds[:-1], bounds[1:]):
        lo, up = int(lo), int(up)
        if up <= lo:
            continue
        ca = MA(a.n_workers, a.replication, a.strategy, a.seed, types.SimpleNamespace(total=up - lo),
                a.unit_workers, a.param_masks[:, lo:up], a.governors[lo:up])
        out.append((lo, up, ca))
    return out


def reference_aggregate(chunks, grads, pool=None):
    """One reference engine.aggregate call per chunk (all chunks = one step)."""
    S = reference_pkg()

    def run(c):
        lo, up, ca = c
        return S.engine.aggregate([g[lo:up] for g in grads], ca).gbar

    if pool is None:
        return [run(c) for c in chunks]
    return list(pool.map(run, chunks))


def _probe_seconds_per_elem(a, threads: int) -> float:
    m = min(a.topology.total, 1 << 20)
    g = reference_grads(a, m)
    ch = reference_chunks(a, m, threads)
    with concurrent.futures.ThreadPoolExecutor(threads) as pool:
        reference_aggregate(ch, g, pool if threads > 1 else None)
        t0 = time.perf_counter()
        reference_aggregate(ch, g, pool if threads > 1 else None)
        return (time.perf_counter() - t0) / m


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    topo, tag = workload(args.workload)
    d = topo.total
    a = reference_assignment(topo, args.strategy, args.n_logical, args.p)
    threads = os.cpu_count() or 1
    # size each step so warmup + steps end within ~2 minutes
    per_step = 120.0 / max(1, args.steps + args.warmup)
    est = _probe_seconds_per_elem(a, threads) * d
    hi = d if est <= per_step else max(1 << 16, int(d * per_step / est))
    grads = reference_grads(a, hi)
    chunks = reference_chunks(a, hi, threads)
    with concurrent.futures.ThreadPoolExecutor(threads) as pool:
        for _ in range(args.warmup):
            reference_aggregate(chunks, grads, pool)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            reference_aggregate(chunks, grads, pool)
            times.append(time.perf_counter() - t0)
    dt = float(np.mean(times))
    nbytes = float(a.coverage[:hi].sum()) * 4
    value = nbytes / dt / 1e9
    sample = (f"{'whole vector' if hi == d else f'first {hi} of {d} elements'} per step; the reference's own "
              f"subnetdp.engine.aggregate (oracle/_ref, unmodified, float64), {threads} host threads each "
              f"calling it on a contiguous range")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": tag, "d": d, "n_logical": args.n_logical, "p": args.p,
                   "strategy": args.strategy, "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
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
    # test hook: ranks share the visible GPUs round-robin (all on GPU 0 on a
    # 1-GPU box: CUDA IPC within one device), gloo plumbing
    if os.environ.get("SDP_BENCH_SAME_DEVICE") == "1":
        local = local % torch.cuda.device_count()
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
        rl = meta.get("roofline", {})
        roofline.update(rl)
        t_s = ms / 1e3  # the slowest rank's launch time (the collective ends with it)
        # SURVEY §8(d) busbw: sum over my elements of 2(k-1)/k * 4 B, k = owner GPUs
        busbw = rl.get("busbw_bytes_per_launch", 0) / t_s / 1e9
        probe = rl.get("p2p_copy_GBps_measured")
        roofline["busbw_GBps"] = busbw
        roofline["busbw_frac_900"] = busbw / 900.0
        roofline["busbw_frac_probe"] = busbw / probe if probe else None
        # what the ports actually carried, per direction (the leader's peer
        # reads and its writes of the mean + bf16 shadow, both ways)
        link = max(rl.get("nvlink_tx_bytes_per_launch", 0), rl.get("nvlink_rx_bytes_per_launch", 0))
        roofline["nvlink_achieved_GBps"] = link / t_s / 1e9
        roofline["nvlink_frac"] = roofline["nvlink_achieved_GBps"] / 900.0
        roofline["nvlink_peak_source"] = "900 GB/s per direction (NVLink 5 nominal); *_probe: this run's peer-copy probe"
        if probe:
            roofline["nvlink_frac_of_run_probe"] = roofline["nvlink_achieved_GBps"] / probe

    e2e = None
    cpu = None
    train = None
    builder = None
    if world > 1 and not args.no_train and args.workload in ("gpt2", "resnet18"):
        train = run_train_multi(args, dev, rank, world, red_dev)
    if rank == 0 and world == 1:
        e2e = run_e2e(args, a, dev, total_bytes)
        if not args.no_train and args.workload in ("gpt2", "resnet18"):
            train = {"c4_gpt2": run_train_gpt2(args, dev), "c2_c3_resnet18": run_train(args, dev)}
            if not args.no_memory_ranks and args.n_logical == 8:
                train["memory_n8_ranks"] = run_memory_ranks(args)
            if args.equal_loss_steps > 0 and args.n_logical == 8 and args.p == 4:
                train["equal_loss"] = run_equal_loss(args, dev, train.get("memory_n8_ranks"))
            if args.n_logical == 8 and args.p == 4:
                c1 = argparse.Namespace(**{**vars(args), "n_logical": 4, "p": 2})
                train["c1_mini_resnet"] = run_train_c1(c1, dev)
        if not args.no_train and args.workload == "c1":
            train = run_train_c1(args, dev)
        if not args.no_cpu_baseline:
            cpu, ref_a = run_cpu_baseline(args, topo)
            builder = run_mask_builder(args, topo, dev, ref_a)
            del ref_a
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
    # what a reference caller hands over: ordinary (pageable) numpy arrays
    # (engine.run's flat_gradient outputs) -> the chunked, pipelined copy path
    pageable = [np.array(h, copy=True) for h in host]
    del host, out
    out = None
    for _ in range(2):
        out = engine.aggregate(pageable, a)
    tp = []
    for _ in range(max(3, args.e2e_steps // 4)):
        t0 = time.perf_counter()
        out = engine.aggregate(pageable, a)
        tp.append(time.perf_counter() - t0)
    dtp = float(np.mean(tp))
    return {"value": total_bytes / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d * 4, "ms_per_step": dt * 1e3,
            "api": "paper_2507_09029_b200.engine.aggregate(list[np.ndarray pinned], assignment)",
            "host_cpus": f"{len(cpus)} GPU-local cores (NVML affinity)" if cpus else "unpinned",
            "timing": "host wall clock around the blocking call (returns numpy)",
            "pageable": {"value": total_bytes / dtp / 1e9, "unit": UNIT, "ms_per_step": dtp * 1e3,
                         "api": "engine.aggregate(list[np.ndarray pageable], assignment): "
                                "16 host threads copy each chunk's owned ranges into pinned staging slots, the copy "
                                "engine moves them to the device, overlapped with the sync and the mean's D2H",
                         "steps": len(tp)}}


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
        tr.check()
        del tr, model, a
        torch.cuda.empty_cache()
    out["speedup_vs_dp_per_step"] = out["dp_ms_per_step"] / out["subnet_ms_per_step"]
    out["configs"] = {"subnet": "configs[1] C2: block dropping P=4", "widthwise": "configs[2] C3: "
                      "channel-slice compact subnetworks (gather/scatter kernels) P=4",
                      "dp": "full-replica DP comparator (P=N)"}
    out["memory"] = "peak memory per GPU: train.memory_n8_ranks (measured in 8 real rank processes)"
    return out


def run_equal_loss(args, dev, memory: dict | None) -> dict:
    """North-star memory target "at equal loss": the C2 / C3 subnetwork runs
    and the P = N DP comparator trained for the same steps on the same
    learnable synthetic task (tools/equal_loss.py), next to the peak memory
    per GPU the 8-rank run measured for the same configurations."""
    sys.path.insert(0, str(ROOT / "tools"))
    from equal_loss import equal_loss
    out = equal_loss(dev, steps=args.equal_loss_steps)
    if memory and "resnet18_subnet" in memory and "resnet18_dp" in memory:
        dp = memory["resnet18_dp"]
        out["peak_memory_vs_dp"] = {"source": "train.memory_n8_ranks (ResNet-18, 8 PeerTrainer rank processes, "
                                              "owned-tile storage)"}
        for tag in ("subnet", "widthwise"):
            if f"resnet18_{tag}" in memory:
                m = memory[f"resnet18_{tag}"]
                out["peak_memory_vs_dp"][f"{tag}_largest_rank"] = m["peak_bytes_max"] / dp["peak_bytes_max"] - 1.0
                out["peak_memory_vs_dp"][f"{tag}_mean_rank"] = m["peak_bytes_mean"] / dp["peak_bytes_mean"] - 1.0
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
    out["reference_cpu"] = run_reference_c1(n, p, batch)
    out["reference_cpu_samples_per_s"] = out["reference_cpu"]["samples_per_s"]
    return out


def run_reference_c1(n: int = 4, p: int = 2, batch: int = 8, steps: int = 6) -> dict:
    """The reference's own training step at configs[0] timed on this host:
    mini-ResNet 26 ch x 8 blocks, synthetic blobs 32x32 (seed 7), N=4, P=2,
    batch 8/worker, block dropping, OPENBLAS 1 thread per worker thread and
    engine threads = N (SURVEY F9's fastest setting).  Set-up and step body
    are engine.run's (engine.py:155-223) calling the reference's functions
    from oracle/_ref unmodified -- the worker fan-out (_worker_step), aggregate
    and optimizer.update -- without run()'s held-out evaluation, which is not
    part of a training step."""
    from threadpoolctl import threadpool_limits
    S = reference_pkg()
    C, E = S.config, S.engine
    cfg = C.ExperimentConfig(
        model=C.ModelConfig(kind="mini_resnet", channels=26, blocks=8, classes=10, norm_groups=2,
                            in_channels=3, image_hw=(32, 32)),
        dataset=C.DatasetConfig(kind="synthetic-blobs", height=32, width=32, channels=3, classes=10, seed=7),
        n=n, p=p, strategy="block", batch_per_worker=batch, seed=1, threads=n)
    dataset = S.data.load_dataset(cfg.dataset)
    model = cfg.model.build(cfg.seed)
    a = E.build_assignment(model.topology, cfg.strategy, cfg.n, cfg.p, cfg.seed)
    model.theta = E.masked_kaiming_init(model, a, cfg.seed)
    opt = E.make_optimizer(cfg.optimizer.kind, model.topology.total, momentum=cfg.optimizer.momentum)
    streams = np.random.SeedSequence(cfg.seed).spawn(cfg.n)
    workers = [E.WorkerState(i, a.worker_view(i), np.random.default_rng(streams[i])) for i in range(cfg.n)]
    layers = (model.topology.default_alignment_layer,)
    times, losses = [], []
    with threadpool_limits(1, "blas"), concurrent.futures.ThreadPoolExecutor(cfg.threads) as pool:
        for t in range(steps + 1):
            t0 = time.perf_counter()
            futs = [pool.submit(E._worker_step, model, w, dataset, cfg.batch_per_worker, t, layers, False)
                    for w in workers]
            reports = [f.result() for f in futs]
            agg = E.aggregate([r.grad for r in reports], a)
            opt.update(model.theta, agg.gbar, 0.02)
            times.append(time.perf_counter() - t0)
            losses.append(float(np.mean([r.loss for r in reports])))
    dt = float(np.mean(times[1:]))  # the first step warms the BLAS / thread pool
    return {"samples_per_s": n * batch / dt, "ms_per_step": dt * 1e3, "cores": n, "steps_timed": steps,
            "loss_first": losses[0], "loss_last": losses[-1],
            "how": f"reference step body (engine.py:203-223: _worker_step fan-out, aggregate, optimizer.update; "
                   f"oracle/_ref unmodified), lr 0.02, OPENBLAS 1 thread, engine threads={n}; "
                   f"host has {os.cpu_count()} cores"}


def run_train_multi(args, dev, rank: int, world: int, red_dev):
    """Train samples/s/GPU at G > 1 GPUs (BASELINE metric part 2 at 2/4/8 GPUs):
    one process per GPU, the N = 8 workers placed contiguously (N/G per rank),
    train.PeerTrainer (local fwd/bwd, peer-mapped owner sync, local fused
    Nesterov + bf16 cast).  CUDA events over the timed steps, max over ranks;
    peak memory = torch.cuda.max_memory_allocated of each rank process over
    its steps (after the full init vector is freed), max over ranks."""
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
        model.theta = None  # the full init vector: the rank keeps only its workers' state
        gen = torch.Generator(device=dev)
        batches = {}
        for w in tr.local:
            gen.manual_seed(w)
            batches[w] = (torch.randn(batch, 3, 32, 32, generator=gen, device=dev),
                          torch.randint(0, 10, (batch,), generator=gen, device=dev))
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats(dev)
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
        out[f"{tag}_peak_mem_per_gpu_bytes"] = int(rmax(torch.cuda.max_memory_allocated(dev)))
        tr.close()
        del tr, model, a
        torch.cuda.empty_cache()
        dist.barrier()
    out["mem_reduction_vs_dp"] = 1 - out["subnet_peak_mem_per_gpu_bytes"] / out["dp_peak_mem_per_gpu_bytes"]
    out["widthwise_mem_reduction_vs_dp"] = (1 - out["widthwise_peak_mem_per_gpu_bytes"]
                                            / out["dp_peak_mem_per_gpu_bytes"])
    out["speedup_vs_dp_per_step"] = out["dp_ms_per_step"] / out["subnet_ms_per_step"]
    # configs[3] C4 at G GPUs: GPT-2 small, seq 1024, micro-batch 8 per worker
    g4 = {"workload": f"GPT-2 small 124M, seq 1024, N={n} workers on {world} GPUs x micro-batch 8, "
                      "bf16 autocast, flash SDPA, fused LM-head cross-entropy", "data": "synthetic tokens"}
    for tag, p in (("subnet", args.p), ("dp", n)):
        model = train.build_gpt2(dev)
        a = masking.build_assignment(model.topology, "block", n, p, seed=1)
        tr = train.PeerTrainer(model, a, rank, world, dev, all_gather, lr=1e-4, loss_fn=train.lm_loss,
                               graphed=True)
        model.theta = None
        gen = torch.Generator(device=dev)
        batches = {}
        for w in tr.local:
            gen.manual_seed(w)
            t = torch.randint(0, 50257, (8, 1024), generator=gen, device=dev)
            batches[w] = (t, t)
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats(dev)
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
        g4[f"{tag}_peak_mem_per_gpu_bytes"] = int(rmax(torch.cuda.max_memory_allocated(dev)))
        tr.close()
        del tr, model, a
        torch.cuda.empty_cache()
        dist.barrier()
    g4["speedup_vs_dp_per_step"] = g4["dp_ms_per_step"] / g4["subnet_ms_per_step"]
    g4["mem_reduction_vs_dp"] = 1 - g4["subnet_peak_mem_per_gpu_bytes"] / g4["dp_peak_mem_per_gpu_bytes"]
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
        tr.check()
        del tr, model, a
        torch.cuda.empty_cache()
    out["speedup_vs_dp_per_step"] = out["dp_ms_per_step"] / out["subnet_ms_per_step"]
    out["memory"] = "peak memory per GPU: train.memory_n8_ranks (measured in 8 real rank processes)"
    return out


def run_mask_builder(args, topo, dev, ref_a=None):
    """build_assignment through the public API on the GPU (seeded
    assignment + element expansion + tables, synchronised) and its kernels
    alone, beside the reference's own build_assignment (masking.py:305-359,
    oracle/_ref, 1 core) on the same topology -- checked bit-exact against
    each other (per-element owner sets)."""
    import torch

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
    ra = reference_assignment(topo, args.strategy, n, p) if ref_a is None else ref_a
    cpu_s = time.perf_counter() - t0 if ref_a is None else getattr(ra, "_bench_build_s", None)
    bits = np.zeros(topo.total, dtype=np.uint8 if n <= 8 else np.uint64)
    for w in range(n):
        bits |= ra.param_masks[w].astype(bits.dtype) << bits.dtype.type(w)
    ours = a.owner_mask.cpu().numpy()
    exact = bool(np.array_equal(ours.astype(np.uint64), bits.astype(np.uint64))
                 and np.array_equal(a.coverage.cpu().numpy(), ra.coverage)
                 and np.array_equal(a.governors.cpu().numpy(), ra.governors))
    return {"workload": f"build_assignment({args.workload}, {args.strategy}, N={n}, P={p}, seed=1)",
            "api_ms": float(np.median(api)) * 1e3,
            "stage_us": {k: round(v, 1) for k, v in kern.items()},
            "stage_timing": "CUDA events around each stage's host call (k_assign includes its group-table "
                            "upload)",
            "reference_cpu_ms": None if cpu_s is None else cpu_s * 1e3, "reference_cpu_cores": 1,
            "reference_kind": "reference (subnetdp.masking.build_assignment from oracle/_ref, unmodified)",
            "bit_exact_vs_reference": exact}


def run_cpu_baseline(args, topo):
    """The reference's own engine.aggregate on ONE core (numpy ufuncs are
    single-threaded) over a bounded prefix of the same workload."""
    t0 = time.perf_counter()
    a = reference_assignment(topo, args.strategy, args.n_logical, args.p)
    a._bench_build_s = time.perf_counter() - t0
    d = topo.total
    budget = 10.0  # seconds of timed calls; one call is sized to ~2.5 s
    est = _probe_seconds_per_elem(a, 1) * d
    hi = d if est <= budget / 4 else max(1 << 16, int(d * budget / 4 / est))
    grads = reference_grads(a, hi)
    chunks = reference_chunks(a, hi, 1)
    reps, t0 = 0, time.perf_counter()
    while True:
        reference_aggregate(chunks, grads)
        reps += 1
        if time.perf_counter() - t0 >= budget / 2 or reps >= 1000:
            break
    dt = (time.perf_counter() - t0) / reps
    value = float(a.coverage[:hi].sum()) * 4 / dt / 1e9
    return {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"{reps} calls over {'the whole vector' if hi == d else f'the first {hi} of {d} elements'}"
                      f" of the reference's own subnetdp.engine.aggregate (oracle/_ref, float64) on 1 thread "
                      f"(host has {os.cpu_count()} cores)",
            "ms_per_call": dt * 1e3}, a


def run_memory_child(args):
    """One rank of the N = G = 8 memory run (launched by run_memory_ranks):
    train.PeerTrainer with ONE worker on this rank, compact owned-tile
    storage, fused sync + Nesterov + bf16 cast; peak = this process's
    torch.cuda.max_memory_allocated over the training steps (all live state:
    compact theta / velocity / bf16 copy / gradient replica, activations,
    scratch), after the initial full theta that built the model was freed.
    Subnet (P = 4) and full-replica DP (P = N = 8) run the same steps on the
    same per-rank batches; their losses are reported side by side."""
    import torch
    import torch.distributed as dist

    from paper_2507_09029_b200 import _native, masking, train
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _native.load()
    dist.init_process_group("gloo")

    def all_gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    res = {}
    steps = max(2, args.train_steps // 2)
    for wl in ("gpt2", "resnet18"):
        runs = (("subnet", args.p, "block"), ("dp", world, "block"))
        if wl == "resnet18":  # configs[2]: width-wise compact subnetworks, owned-tile storage too
            runs += (("widthwise", args.p, "neuron"),)
        for tag, p, strategy in runs:
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
            model = train.build_gpt2(dev) if wl == "gpt2" else train.build_resnet18(dev)
            a = masking.build_assignment(model.topology, strategy, world, p, seed=1)
            kw = {"loss_fn": train.lm_loss, "lr": 1e-4} if wl == "gpt2" else {"lr": 0.02}
            tr = train.PeerTrainer(model, a, rank, world, dev, all_gather, graphed=False,
                                   timeout_cycles=60_000_000_000, **kw)
            model.theta = None  # the full init vector: every rank now holds only its compact state
            gen = torch.Generator(device=dev)
            gen.manual_seed(rank)
            if wl == "gpt2":
                t = torch.randint(0, 50257, (8, 1024), generator=gen, device=dev)
                batches = {w: (t, t) for w in tr.local}
            else:
                batches = {w: (torch.randn(64, 3, 32, 32, generator=gen, device=dev),
                               torch.randint(0, 10, (64,), generator=gen, device=dev)) for w in tr.local}
            torch.cuda.synchronize()
            torch.cuda.reset_peak_memory_stats(dev)
            losses = []
            for _ in range(steps):
                losses.append(float(tr.step(batches).item()))
            torch.cuda.synchronize()
            tr.check()
            res[f"{wl}_{tag}"] = {"peak_bytes": int(torch.cuda.max_memory_allocated(dev)),
                                  "state_bytes": int(tr.state_bytes()),
                                  "stored_params": int(sum(tr.theta[w].numel() for w in tr.local)),
                                  "losses": losses}
            tr.close()
            del tr, model, a, batches
            dist.barrier()
        res[f"{wl}_torch_ddp"] = torch_ddp_memory(wl, dev, rank, steps)
        dist.barrier()
    allr = all_gather(res)
    if rank == 0:
        print("MEMORY_RANKS " + json.dumps(allr), flush=True)
    dist.destroy_process_group()


def torch_ddp_memory(wl: str, dev, rank: int, steps: int) -> dict:
    """The stock comparator the north star names: torch DistributedDataParallel
    over the same model (one flat fp32 nn.Parameter holding every weight, cast
    to bf16 once per forward, the same forward kernels), bf16 autocast,
    torch.optim.SGD(momentum 0.9, nesterov), DDP's default 25 MB gradient
    buckets, on this rank's batch.
    Peak = torch.cuda.max_memory_allocated over the training steps."""
    import torch
    from torch.nn.parallel import DistributedDataParallel

    from paper_2507_09029_b200 import train

    class Flat(torch.nn.Module):
        def __init__(self, m):
            super().__init__()
            self.arch, self.topo = m.arch, m.topology
            self.theta = torch.nn.Parameter(m.theta.detach().clone())

        def forward(self, x):
            # AMP's weight cast, once for the whole flat vector (as the
            # trainers' bf16 copy): bf16 activations on the same kernels
            params = train.param_views(self.topo, self.theta.to(torch.bfloat16))
            if wl == "gpt2":
                params["__wte_padded"] = train._LinearCrossEntropy._padded(params["wte"].detach(), torch.bfloat16)
            return self.arch.forward(params, x)

    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    m = train.build_gpt2(dev) if wl == "gpt2" else train.build_resnet18(dev)
    net = Flat(m)
    m.theta = None
    ddp = DistributedDataParallel(net, device_ids=[dev.index])
    opt = torch.optim.SGD(ddp.parameters(), lr=1e-4 if wl == "gpt2" else 0.02, momentum=0.9, nesterov=True)
    gen = torch.Generator(device=dev)
    gen.manual_seed(rank)
    if wl == "gpt2":
        x = torch.randint(0, 50257, (8, 1024), generator=gen, device=dev)
        y = x
        loss_fn = train.lm_loss
    else:
        x = torch.randn(64, 3, 32, 32, generator=gen, device=dev)
        y = torch.randint(0, 10, (64,), generator=gen, device=dev)
        loss_fn = lambda out, t: torch.nn.functional.cross_entropy(out.float(), t)  # noqa: E731
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    losses = []
    for _ in range(steps):
        opt.zero_grad(set_to_none=False)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = loss_fn(ddp(x), y)
        loss.backward()
        opt.step()
        losses.append(float(loss.item()))
    torch.cuda.synchronize()
    out = {"peak_bytes": int(torch.cuda.max_memory_allocated(dev)),
           "state_bytes": int(3 * net.theta.numel() * 4), "stored_params": int(net.theta.numel()),
           "losses": losses}
    del ddp, net, opt, m
    return out


def run_memory_ranks(args, world: int = 8) -> dict:
    """BASELINE metric part 3 on the system that runs: peak memory per GPU at
    N = G = 8 (one worker per rank), measured by torch.cuda.max_memory_allocated
    inside each of 8 real PeerTrainer processes (torchrun, CUDA-IPC peer
    mapping, the fused sync kernel with its cross-process barrier).  On a
    1-GPU box the 8 processes share the device (time-sliced), which changes
    nothing about each process's own allocations; step time is not measured
    here."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, SDP_BENCH_SAME_DEVICE="1", SDP_DIST_BACKEND="gloo", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), "--memory-child",
           "--p", str(args.p), "--train-steps", str(args.train_steps)]
    import subprocess
    t0 = time.perf_counter()
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    line = next((ln for ln in r.stdout.splitlines() if ln.startswith("MEMORY_RANKS ")), None)
    if r.returncode != 0 or line is None:
        return {"error": (r.stdout[-1500:] + r.stderr[-1500:])}
    ranks = json.loads(line[len("MEMORY_RANKS "):])
    out = {"how": f"{world} PeerTrainer processes (one worker each, N = G = {world}), compact owned-tile storage, "
                  "fused sync+Nesterov+bf16; torch.cuda.max_memory_allocated per process over the training "
                  "steps; ranks share one GPU here (time-sliced)",
           "wall_s": round(time.perf_counter() - t0, 1)}
    for key in ranks[0]:
        peaks = [rk[key]["peak_bytes"] for rk in ranks]
        out[key] = {"peak_bytes_max": max(peaks), "peak_bytes_mean": float(np.mean(peaks)),
                    "peak_bytes_per_rank": peaks,
                    "state_bytes_max": max(rk[key]["state_bytes"] for rk in ranks),
                    "loss_per_step_rank_mean": [float(np.mean([rk[key]["losses"][i] for rk in ranks]))
                                                for i in range(len(ranks[0][key]["losses"]))]}
    for wl, tag in (("gpt2", "subnet"), ("resnet18", "subnet"), ("resnet18", "widthwise")):
        sub, dp = out[f"{wl}_{tag}"], out[f"{wl}_dp"]
        name = wl if tag == "subnet" else f"{wl}_{tag}"
        out[f"{name}_mem_reduction_vs_dp"] = 1 - sub["peak_bytes_max"] / dp["peak_bytes_max"]
        out[f"{name}_mem_reduction_vs_dp_mean"] = 1 - sub["peak_bytes_mean"] / dp["peak_bytes_mean"]
        ddp = out.get(f"{wl}_torch_ddp")
        if ddp:
            out[f"{name}_mem_reduction_vs_torch_ddp"] = 1 - sub["peak_bytes_max"] / ddp["peak_bytes_max"]
            out[f"{name}_mem_reduction_vs_torch_ddp_mean"] = 1 - sub["peak_bytes_mean"] / ddp["peak_bytes_mean"]
    return out


def main():
    args = parse()
    if args.memory_child:
        run_memory_child(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
