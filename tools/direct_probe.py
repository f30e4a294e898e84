"""SDP_SYNC_DIRECT vs the tiled kernel on the width-wise flat-layout aggregate
(C3 ResNet-18, C4 GPT-2 channel units) and the block configs.  Probe-only."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
if "--lib" in sys.argv:  # an A/B variant (tools/variant_build.py) instead of the in-tree build
    from paper_2507_09029_b200 import _native as _N  # noqa: E402
    _N.load(sys.argv[sys.argv.index("--lib") + 1])
import measure_all as M  # noqa: E402
from paper_2507_09029_b200 import engine, masking, zoo  # noqa: E402


def main():
    M.FLUSH_W = torch.empty(64 << 20, device=M.DEV)
    M.FLUSH_R = torch.zeros(64 << 20, device=M.DEV)
    for name, topo, strategy in (("C3", zoo.resnet18_cifar_topology(), "neuron"),
                                 ("C2", zoo.resnet18_cifar_topology(), "block"),
                                 ("C4n", zoo.gpt2_small_topology(), "neuron"),
                                 ("C4", zoo.gpt2_small_topology(), "block"),
                                 ("C5n", zoo.mini_resnet_topology(512, 8, 10, 2, 3, (8, 8)), "neuron")):
        a = masking.build_assignment(topo, strategy, 8, 4, seed=1)
        d = topo.total
        reps = [torch.randn(d, device=M.DEV) * a.param_masks[w] for w in range(8)]
        out = torch.empty(d, device=M.DEV)
        for direct, stream in ((False, False), (True, False), (True, True)):
            plan = engine.SyncPlan(a, direct=direct, stream=stream)
            prep = engine.PreparedSync(reps, a, writeback=False, out=out, plan=plan)
            us, mn = M.timed(prep.launch)
            own = plan.owned_elems
            nbytes = own * 4 + d * 4 + (plan.n_tiles - plan.n_uniform) * plan.tile
            auto = engine.SyncPlan(a)
            print(json.dumps({"cfg": name, "direct": direct, "stream": stream,
                              "auto": [auto.direct, auto.stream_mean],
                              "us": round(us, 1),
                              "frac": round(nbytes / us / 1e3 / M.PEAK, 3)}), flush=True)
        del reps


if __name__ == "__main__" and "--aggregate" not in sys.argv:
    main()


def aggregate_c3():
    """The drop-in engine.aggregate at C3 (leak check on: uncovered entries)."""
    topo = zoo.resnet18_cifar_topology()
    a = masking.build_assignment(topo, "neuron", 8, 4, seed=1)
    d = topo.total
    reps = [torch.randn(d, device=M.DEV) * a.param_masks[w] for w in range(8)]
    us, _ = M.timed(lambda: engine.aggregate(reps, a))
    plan = a.sync_plan()
    nbytes = plan.owned_elems * 4 + d * 4
    st = torch.zeros(1, dtype=torch.int32, device=M.DEV)
    out = torch.empty(d, device=M.DEV)
    prep = engine.PreparedSync(reps, a, writeback=False, out=out, check_uncovered=True, status=st)
    us_k, _ = M.timed(prep.launch)
    print(json.dumps({"cfg": "C3 kernel with the leak check", "lib": sys.argv[sys.argv.index("--lib") + 1]
                      if "--lib" in sys.argv else "in-tree", "us": round(us_k, 1),
                      "frac": round(nbytes / us_k / 1e3 / M.PEAK, 3)}), flush=True)
    print(json.dumps({"cfg": "C3 engine.aggregate", "direct": plan.direct, "stream_mean": plan.stream_mean,
                      "us": round(us, 1), "frac": round(nbytes / us / 1e3 / M.PEAK, 3)}), flush=True)


if __name__ == "__main__" and "--aggregate" in sys.argv:
    M.FLUSH_W = torch.empty(64 << 20, device=M.DEV)
    M.FLUSH_R = torch.zeros(64 << 20, device=M.DEV)
    aggregate_c3()
