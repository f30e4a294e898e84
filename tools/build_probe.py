"""Run k_assign + k_build_masks once per config (ncu target).

    ncu --set full -k regex:'k_build_masks|k_assign' python tools/build_probe.py [r18|gpt2|gpt2n]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2507_09029_b200 import _native as N  # noqa: E402
from paper_2507_09029_b200 import masking, zoo  # noqa: E402

N.load()
dev = torch.device("cuda", 0)
for name in [a for a in sys.argv[1:] if not a.startswith("--")] or ["r18", "gpt2"]:
    topo = zoo.resnet18_cifar_topology() if name.startswith("r18") else zoo.gpt2_small_topology()
    strategy = "neuron" if name.endswith("n") else "block"
    tables = masking._DeviceTables(topo, strategy, dev)
    t = tables.table
    ub = masking._device_assign(t.groups, t.n_units, 8, 4, 1, dev)
    masking._expand(topo, tables, ub, 8, dev)
    torch.cuda.synchronize()
    print(name, strategy, "d", topo.total, "units", t.n_units)

if "--time" in sys.argv[1:]:
    import time  # noqa: E402,F401

    from paper_2507_09029_b200._device import ptr, stream_ptr  # noqa: E402
    flush_w = torch.empty(64 << 20, device=dev)
    for name in ("r18", "gpt2", "r18n"):
        topo = zoo.resnet18_cifar_topology() if name.startswith("r18") else zoo.gpt2_small_topology()
        strategy = "neuron" if name.endswith("n") else "block"
        tables = masking._DeviceTables(topo, strategy, dev)
        t = tables.table
        ub = masking._device_assign(t.groups, t.n_units, 8, 4, 1, dev)
        d = topo.total
        om = torch.empty(d, dtype=torch.uint8, device=dev)
        cov = torch.empty(d, dtype=torch.int64, device=dev)
        div = torch.empty(d, dtype=torch.float64, device=dev)
        gov = torch.empty(d, dtype=torch.int64, device=dev)
        ac = torch.zeros(8, dtype=torch.int64, device=dev)

        def launch():
            N.call("sdp_build_masks", ptr(tables.params), tables.n_params, ptr(tables.rules), tables.n_rules,
                   ptr(ub), 8, d, ptr(om), 1, None, ptr(cov), ptr(div), ptr(gov), ptr(ac), stream_ptr(dev))

        for mode in ("kernel", "kernel on zeroed outputs", "_expand"):
            fn = (lambda: masking._expand(topo, tables, ub, 8, dev)) if mode == "_expand" else launch
            ts = []
            for i in range(8):
                if mode == "kernel on zeroed outputs":
                    for b in (om, cov, div, gov):
                        b.zero_()
                flush_w.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                fn()
                e.record()
                torch.cuda.synchronize()
                ts.append(s.elapsed_time(e) * 1e3)
            print(name, mode, "us", [round(x, 1) for x in ts], "GB/s", round(d * 25 / min(ts[2:]) / 1e3, 1))

if "--fill" in sys.argv[1:]:
    d = zoo.gpt2_small_topology().total
    bufs = [torch.empty(d, dtype=torch.int64, device=dev) for _ in range(3)] + [torch.empty(d, dtype=torch.uint8, device=dev)]
    for _ in range(3):
        for b in bufs:
            b.fill_(1)
    torch.cuda.synchronize()
    for rep in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for b in bufs:
            b.fill_(1)
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) * 1e3
        print("torch fill of the same 4 outputs (3.1 GB): us", round(us, 1), "GB/s", round(d * 25 / us / 1e3, 1))
    big = torch.empty(3 * d, dtype=torch.int64, device=dev)
    for rep in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        big.zero_()
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) * 1e3
        print("one 3 GB zero_: us", round(us, 1), "GB/s", round(3 * d * 8 / us / 1e3, 1))
