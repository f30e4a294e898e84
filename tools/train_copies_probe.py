"""Which host-level ops launch the copy kernels of a co-resident training
step: one eager step under the torch profiler, CPU ops grouped by input
shapes.   python tools/train_copies_probe.py [subnet|widthwise|dp|gpt2]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2507_09029_b200 import masking, train  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "widthwise"
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(0)
if which == "gpt2":
    g = train.build_gpt2(dev)
    a = masking.build_assignment(g.topology, "block", 8, 4, seed=1)
    tr = train.SubnetTrainer(g, a, lr=1e-4, loss_fn=train.lm_loss)
    tok = torch.randint(0, 50257, (8, 1024), generator=gen, device=dev)
    batches = [(tok, tok)] * 8
else:
    g = train.build_resnet18(dev)
    strategy, p = {"subnet": ("block", 4), "widthwise": ("neuron", 4), "dp": ("block", 8)}[which]
    a = masking.build_assignment(g.topology, strategy, 8, p, seed=1)
    tr = train.SubnetTrainer(g, a, lr=0.02, sync_layout=strategy == "neuron")
    batches = [(torch.randn(64, 3, 32, 32, generator=gen, device=dev),
                torch.randint(0, 10, (64,), generator=gen, device=dev)) for _ in range(8)]
tr.step(batches)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA],
                            record_shapes=True) as prof:
    tr.step(batches)
    torch.cuda.synchronize()
ops = ("aten::copy_", "aten::contiguous", "aten::clone", "aten::_to_copy", "aten::cat", "aten::stack",
       "aten::index_add_", "aten::index_select", "aten::scatter", "aten::gather", "aten::zero_", "aten::fill_")
rows = [k for k in prof.key_averages(group_by_input_shape=True) if k.key in ops]
rows.sort(key=lambda k: -k.device_time_total)
for k in rows[:30]:
    print(f"{k.device_time_total / 1e3:8.3f} ms {k.count:5d}  {k.key:18s} {str(k.input_shapes)[:150]}")
