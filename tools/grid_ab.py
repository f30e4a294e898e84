"""A/B the sync plan's CTA shape on one box: tiles per CTA 1 vs capped grid,
for several workloads and P (same process, same clocks)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2507_09029_b200 import engine, masking, zoo  # noqa: E402

dev = torch.device("cuda", 0)
fw = torch.empty(64 << 20, device=dev)
fr = torch.zeros(64 << 20, device=dev)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        fw.zero_()
        fr.sum()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return sum(ts) / len(ts)


for name, topo in (("resnet18", zoo.resnet18_cifar_topology()), ("gpt2", zoo.gpt2_small_topology()),
                   ("sweep256", zoo.sweep_topology(64 << 20))):
    for p in (2, 4):
        a = masking.build_assignment(topo, "block", 8, p, seed=1)
        reps = [torch.randn(topo.total, device=dev) * a.param_masks[w] for w in range(8)]
        sh = [torch.zeros(topo.total, dtype=torch.bfloat16, device=dev) for _ in range(8)]
        res = {}
        for tag, kw in (("tpc1", {}), ("cap4736", {"max_grid": 4736}), ("tile4096", {"tile": 4096})):
            plan = engine.SyncPlan(a, **kw)
            prep = engine.PreparedSync(reps, a, writeback=True, shadows_bf16=sh, plan=plan)
            us = timed(prep.launch)
            res[tag] = round(us, 1)
            res[tag + "_frac"] = round(plan.owned_elems * 10 / us / 1e3 / 6548.5, 3)
        print(json.dumps({"workload": name, "p": p, **res}), flush=True)
        del reps, sh
        torch.cuda.empty_cache()
