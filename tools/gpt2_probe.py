"""Where a GPT-2 (C4) co-resident worker step's time goes.

    python tools/gpt2_probe.py
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2507_09029_b200 import masking, train  # noqa: E402

dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(0)
g = train.build_gpt2(dev)
a = masking.build_assignment(g.topology, "block", 8, 4, seed=1)
tr = train.SubnetTrainer(g, a, lr=1e-4, loss_fn=train.lm_loss, graphed=True)
tok = torch.randint(0, 50257, (8, 1024), generator=gen, device=dev)
batches = [(tok, tok)] * 8
for _ in range(2):
    tr.step(batches)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3):
    tr.step(batches)
e.record()
torch.cuda.synchronize()
print(f"step {s.elapsed_time(e) / 3:.1f} ms")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    tr.step(batches)
    torch.cuda.synchronize()
ka = sorted(prof.key_averages(), key=lambda k: -k.device_time_total)[:18]
tot = sum(k.device_time_total for k in prof.key_averages())
for k in ka:
    print(f"{k.device_time_total / 1e3:8.2f} ms {100 * k.device_time_total / tot:5.1f}% {k.count:5d}  {k.key[:150]}")
