"""Timing probe for k_owner_sync variants (run under gpurun; not part of bench).

    python tools/sync_probe.py [--workload resnet18|gpt2|sweep:MiB] [--strategy block|neuron]

Prints per-variant microseconds per launch:
  events+flush   : per-launch CUDA events, L2 write+read flush between launches
  back-to-back   : K launches between two events, no flush (inputs > L2)
  graph          : K launches captured in one CUDA graph, no flush
"""

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2507_09029_b200 import engine, masking, zoo  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet18")
    ap.add_argument("--strategy", default="block")
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--no-shadow", action="store_true")
    ap.add_argument("--no-writeback", action="store_true")
    ap.add_argument("--tile", type=int, default=None)
    ap.add_argument("--tpc1", action="store_true", help="one tile per CTA (grid = #tiles)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    if args.workload == "resnet18":
        topo = zoo.resnet18_cifar_topology()
    elif args.workload == "gpt2":
        topo = zoo.gpt2_small_topology()
    else:
        topo = zoo.sweep_topology(int(args.workload.split(":")[1]) * (1 << 20) // 4)
    a = masking.build_assignment(topo, args.strategy, args.n, args.p, seed=1)
    d = topo.total
    reps = [torch.randn(d, device=dev) * a.param_masks[w] for w in range(args.n)]
    shadows = None if args.no_shadow else [torch.zeros(d, dtype=torch.bfloat16, device=dev) for _ in reps]
    out = torch.empty(d, device=dev) if args.no_writeback else None
    kw = {"tile": args.tile}
    if args.tpc1:
        kw["force_grid"] = -(-d // (args.tile or engine.auto_tile(d, 148)))  # one tile per CTA
    plan = a.sync_plan(**kw)
    prep = engine.PreparedSync(reps, a, writeback=not args.no_writeback, shadows_bf16=shadows,
                               out=out, plan=plan)
    per = (4 + (0 if args.no_writeback else 4) + (0 if (args.no_shadow or args.no_writeback) else 2))
    hbm = plan.owned_elems * per + (d * 4 if out is not None else 0)
    flush = torch.empty(64 << 20, device=dev)
    flush_rd = torch.zeros(64 << 20, device=dev)
    for _ in range(5):
        prep.launch()
    torch.cuda.synchronize()
    res = {}
    st = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    en = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        flush_rd.sum()
        st[i].record()
        prep.launch()
        en[i].record()
    torch.cuda.synchronize()
    res["events+flush"] = sum(s.elapsed_time(e) for s, e in zip(st, en)) / args.steps * 1e3
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.steps):
        prep.launch()
    e.record()
    torch.cuda.synchronize()
    res["back-to-back"] = s.elapsed_time(e) / args.steps * 1e3
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        with torch.cuda.graph(g, stream=cs):
            for _ in range(args.steps):
                prep.launch(cs)
    torch.cuda.synchronize()
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    res["graph"] = s.elapsed_time(e) / args.steps * 1e3
    out_d = {"tile": args.tile, "workload": args.workload, "strategy": args.strategy, "n": args.n, "p": args.p,
             "tiles": plan.n_tiles, "uniform": plan.n_uniform, "grid": plan.grid,
             "hbm_bytes": hbm, "us": res,
             "GBps": {k: hbm / v / 1e3 for k, v in res.items()}}
    print(json.dumps(out_d))


if __name__ == "__main__":
    main()
