"""One graphed co-resident training step inside cudaProfilerStart/Stop, for
an ncu launch list of exactly one step (warm-up and capture excluded):

    ncu --profile-from-start off --metrics gpu__time_duration.sum \\
        --clock-control none --csv --log-file L.csv \\
        python tools/train_step_once.py [subnet|widthwise|dp|gpt2]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2507_09029_b200 import masking, train  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "subnet"
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(0)
if which == "gpt2":
    g = train.build_gpt2(dev)
    a = masking.build_assignment(g.topology, "block", 8, 4, seed=1)
    tr = train.SubnetTrainer(g, a, lr=1e-4, loss_fn=train.lm_loss, graphed=True)
    tok = torch.randint(0, 50257, (8, 1024), generator=gen, device=dev)
    batches = [(tok, tok)] * 8
else:
    g = train.build_resnet18(dev)
    strategy, p = {"subnet": ("block", 4), "widthwise": ("neuron", 4), "dp": ("block", 8)}[which]
    a = masking.build_assignment(g.topology, strategy, 8, p, seed=1)
    tr = train.SubnetTrainer(g, a, lr=0.02, sync_layout=strategy == "neuron", graphed=True)
    batches = [(torch.randn(64, 3, 32, 32, generator=gen, device=dev),
                torch.randint(0, 10, (64,), generator=gen, device=dev)) for _ in range(8)]
for _ in range(2):
    tr.step(batches)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
tr.step(batches)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("one step done")
