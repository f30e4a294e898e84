"""Where a co-resident training step's time goes (GPU kernel time vs wall).

    python tools/train_probe.py [--graphed] [subnet|widthwise|dp ...]
"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2507_09029_b200 import masking, train  # noqa: E402

dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(0)
n, batch = 8, 64
batches = [(torch.randn(batch, 3, 32, 32, generator=gen, device=dev),
            torch.randint(0, 10, (batch,), generator=gen, device=dev)) for _ in range(n)]
which = [a for a in sys.argv[1:] if not a.startswith("--")] or ["subnet", "widthwise", "dp"]
for tag, p, strategy in (("subnet", 4, "block"), ("widthwise", 4, "neuron"), ("dp", 8, "block")):
    if tag not in which:
        continue
    model = train.build_resnet18(dev)
    a = masking.build_assignment(model.topology, strategy, n, p, seed=1)
    tr = train.SubnetTrainer(model, a, lr=0.02, sync_layout=(strategy == "neuron"),
                             graphed="--graphed" in sys.argv)
    for _ in range(3):
        tr.step(batches)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        tr.step(batches)
    t_enq = time.perf_counter() - t0
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / 5
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        tr.step(batches)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    kern = sum(e.device_time_total for e in ev) / 1e3
    print(f"{tag}: wall {wall * 1e3:.1f} ms/step, host enqueue {t_enq / 5 * 1e3:.1f} ms/step, "
          f"GPU kernel time {kern:.1f} ms/step, kernels {len(ev)}")
    top = prof.key_averages().table(sort_by="cuda_time_total", row_limit=25)
    print("\n".join(ln[:60] + ln[100:200] for ln in top.splitlines()))
    if "--names" in sys.argv:
        ka = sorted(prof.key_averages(), key=lambda k: -k.device_time_total)[:12]
        for k in ka:
            print(f"{k.device_time_total / 1e3:8.3f} ms {k.count:5d}  {k.key[:300]}")
    del tr, model
    torch.cuda.empty_cache()
