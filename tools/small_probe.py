"""Small-buffer sync probe (C5 1-16 MiB; run under gpurun; not part of bench).

For each size / P: per-launch microseconds of k_owner_sync (cold L2 via a
flush, warm L2 without), a same-traffic device copy for the practical floor,
and an empty kernel for the event overhead.  One JSON line per row.

    python tools/small_probe.py [--sizes 1,4,16] [--ps 2,4,8] [--tiles 1024,2048]
"""

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2507_09029_b200 import _native as N  # noqa: E402

if "--lib" in sys.argv:  # an A/B variant (tools/variant_build.py) instead of the in-tree build
    N.load(sys.argv[sys.argv.index("--lib") + 1])
from paper_2507_09029_b200 import engine, masking, zoo  # noqa: E402

DEV = torch.device("cuda", 0)
FW = FR = None


def flush():
    FW.zero_()
    FR.sum()


def timed(fn, reps=30, cold=True):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    st = [torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    en = [torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    for i in range(reps):
        if cold:
            flush()
        st[i].record()
        fn()
        en[i].record()
    torch.cuda.synchronize()
    ts = sorted(s.elapsed_time(e) * 1e3 for s, e in zip(st, en))
    return ts[len(ts) // 2], ts[0]


def main():
    global FW, FR
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1,4,16")
    ap.add_argument("--ps", default="2,4,8")
    ap.add_argument("--tiles", default="auto")
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--strategy", default="block")
    ap.add_argument("--lib", default=None)
    ap.add_argument("--graph-only", action="store_true")
    ap.add_argument("--direct", type=int, default=None, help="force the small-buffer kernel on (1) / off (0)")
    ap.add_argument("--plans", default="{}", help="JSON list of extra sync_plan kwargs for the graph rows")
    args = ap.parse_args()
    FW = torch.empty(64 << 20, device=DEV)
    FR = torch.zeros(64 << 20, device=DEV)
    peak = json.load(open(Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json")).get("hbm_gbs", 6540.5)
    tiny = torch.zeros(1, device=DEV)
    med, mn = timed(lambda: tiny.add_(1))
    print(json.dumps({"row": "empty kernel", "us": round(med, 2), "us_min": round(mn, 2)}), flush=True)
    for mib in [float(x) for x in args.sizes.split(",")]:
        d = int(mib * (1 << 20)) // 4
        topo = zoo.sweep_topology(d)
        for p in [int(x) for x in args.ps.split(",")]:
            a = masking.build_assignment(topo, args.strategy, args.n, p, seed=1)
            reps = [torch.randn(d, device=DEV) * a.param_masks[w] for w in range(args.n)]
            shadows = [torch.zeros(d, dtype=torch.bfloat16, device=DEV) for _ in reps]
            own = int(a.owned_total())
            nbytes = own * 10
            src = torch.empty(nbytes // 8, device=DEV)
            dst = torch.empty_like(src)
            cm, cmn = timed(lambda: dst.copy_(src))
            print(json.dumps({"row": "copy same traffic", "MiB": mib, "p": p, "bytes": nbytes,
                              "us": round(cm, 2), "frac": round(nbytes / cm / 1e3 / peak, 3)}), flush=True)
            tiles = [None] if args.tiles == "auto" else [int(t) for t in args.tiles.split(",")]
            for t in ([] if args.graph_only else tiles):
                plan = a.sync_plan(tile=t)
                prep = engine.PreparedSync(reps, a, writeback=True, shadows_bf16=shadows, plan=plan)
                for cold in (True, False):
                    m, mn = timed(prep.launch, cold=cold)
                    print(json.dumps({"row": "sync", "MiB": mib, "p": p, "tile": plan.tile,
                                      "grid": plan.grid, "tiles": plan.n_tiles,
                                      "mixed": plan.n_tiles - plan.n_uniform, "cold": cold,
                                      "bytes": nbytes, "us": round(m, 2), "us_min": round(mn, 2),
                                      "frac": round(nbytes / m / 1e3 / peak, 3)}), flush=True)
            # graph-amortised: M back-to-back launches over K distinct replica
            # sets whose footprint is > 2x L2 (each launch reads cold HBM), so
            # the per-launch time is free of the ~6 us event / launch floor
            for pk in ([{}] + json.loads(args.plans) if args.plans != "{}" else [{}]):
                graph_row(args, a, d, mib, p, nbytes, peak, pk)
            del reps, shadows, src, dst


def graph_row(args, a, d, mib, p, nbytes, peak, pk):
    if True:
        if True:
            n_bytes_set = args.n * d * 6
            k_sets = max(2, min(64, -(-(300 << 20) // n_bytes_set)))
            sets = []
            for _ in range(k_sets):
                r_ = [torch.randn(d, device=DEV) * a.param_masks[w] for w in range(args.n)]
                s_ = [torch.zeros(d, dtype=torch.bfloat16, device=DEV) for _ in r_]
                sets.append(engine.PreparedSync(r_, a, writeback=True, shadows_bf16=s_,
                                                plan=a.sync_plan(direct=args.direct, **pk)))
            m_launch = 4 * k_sets
            cs = torch.cuda.Stream()
            with torch.cuda.stream(cs):
                for i in range(k_sets):
                    sets[i].launch(cs)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cs):
                for i in range(m_launch):
                    sets[i % k_sets].launch(cs)
            g.replay()
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3 / m_launch)
            m = sorted(ts)[len(ts) // 2]
            print(json.dumps({"row": "sync graph", "MiB": mib, "p": p, "direct": sets[0].args.flags & 0x40 != 0,
                              "plan": pk, "grid": sets[0].args.grid, "tile": sets[0].args.tile,
                              "sets": k_sets, "launches": m_launch,
                              "bytes": nbytes, "us": round(m, 2), "frac": round(nbytes / m / 1e3 / peak, 3)}),
                  flush=True)
            del sets, g


if __name__ == "__main__":
    main()
