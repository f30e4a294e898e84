"""One graphed ResNet-18 (C3 width-wise) and one GPT-2 (C4) worker step for
ncu: captures k_gn_fwd / k_gn_bwd / k_ce_fwd / k_ce_bwd launches.

    ncu --set full -k regex:'k_gn|k_ce' -c 8 python tools/train_kernels_probe.py
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2507_09029_b200 import masking, train  # noqa: E402

dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(0)
model = train.build_resnet18(dev)
a = masking.build_assignment(model.topology, "neuron", 8, 4, seed=1)
tr = train.SubnetTrainer(model, a, lr=0.02, sync_layout=True)
batches = [(torch.randn(64, 3, 32, 32, generator=gen, device=dev),
            torch.randint(0, 10, (64,), generator=gen, device=dev)) for _ in range(8)]
tr.step(batches)
g = train.build_gpt2(dev)
ag = masking.build_assignment(g.topology, "block", 8, 4, seed=1)
tg = train.SubnetTrainer(g, ag, lr=1e-4, loss_fn=train.lm_loss)
tok = torch.randint(0, 50257, (8, 1024), generator=gen, device=dev)
tg.step([(tok, tok)] * 8)
torch.cuda.synchronize()
print("ok")
