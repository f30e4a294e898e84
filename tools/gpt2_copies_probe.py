"""Which host-level ops launch the copy kernels of a GPT-2 (C4) worker step:
one eager step under the torch profiler, CPU ops grouped by input shapes."""
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
tr = train.SubnetTrainer(g, a, lr=1e-4, loss_fn=train.lm_loss, graphed=False)
tok = torch.randint(0, 50257, (8, 1024), generator=gen, device=dev)
batches = [(tok, tok)] * 8
tr.step(batches)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA],
                            record_shapes=True, with_stack=True) as prof:
    tr.step(batches[:1] * 8)
    torch.cuda.synchronize()
rows = [k for k in prof.key_averages(group_by_input_shape=True)
        if k.key in ("aten::copy_", "aten::contiguous", "aten::clone", "aten::_to_copy", "aten::cat", "aten::stack")]
rows.sort(key=lambda k: -k.device_time_total)
for k in rows[:25]:
    print(f"{k.device_time_total / 1e3:8.2f} ms {k.count:5d}  {k.key:18s} {str(k.input_shapes)[:160]}")

print("-- stacks of the [8, 12, 1024, 64] copies")
for k in prof.key_averages(group_by_stack_n=6):
    if k.key == "aten::copy_" and k.device_time_total > 100:
        print(f"{k.device_time_total / 1e3:8.2f} ms x{k.count}", " <- ".join(k.stack[:6]))
