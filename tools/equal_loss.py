"""Equal-compute loss/accuracy of subnetwork DP vs full-replica DP (C2 / C3).

ResNet-18 CIFAR-shape, N = 8 co-resident workers, batch 64 per worker, the
same init, the same learning rate and the same number of steps (= the same
per-worker sample count); the only difference is the assignment:
  subnet    block dropping, P = 4 (configs[1])
  widthwise channel slices, P = 4 (configs[2], sync layout)
  dp        P = N: every worker holds the full model (the DP comparator)
Data: a learnable synthetic 10-class task (class-mean images + Gaussian
noise), fresh samples every step, a held-out set of 4096 for the full model.

    python tools/equal_loss.py [--steps 300] [--out path.json]
The bench runs the same function (bench.py: train.equal_loss).
"""

import argparse
import json
import sys
import time
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2507_09029_b200 import masking, train  # noqa: E402


class BlobImages:
    """x = amp * mean[y] + noise, mean[y] a fixed random 3x32x32 image per class."""

    def __init__(self, dev, classes: int = 10, amp: float = 0.2, seed: int = 123):
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        self.means = torch.randn(classes, 3, 32, 32, generator=g, device=dev) * amp
        self.classes, self.dev = classes, dev

    def batch(self, n: int, seed: int):
        g = torch.Generator(device=self.dev)
        g.manual_seed(seed)
        y = torch.randint(0, self.classes, (n,), generator=g, device=self.dev)
        x = self.means[y] + torch.randn(n, 3, 32, 32, generator=g, device=self.dev)
        return x, y


@torch.no_grad()
def evaluate(model, data: BlobImages, n: int = 4096) -> dict:
    x, y = data.batch(n, seed=10**9)
    params = train.param_views(model.topology, model.theta)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        logits = model.arch.forward(params, x)  # the full model (every block / channel)
    logits = logits.float()
    return {"eval_loss": float(F.cross_entropy(logits, y)), "eval_acc": float((logits.argmax(1) == y).float().mean())}


def equal_loss(dev, steps: int = 300, n: int = 8, p: int = 4, batch: int = 64, lr: float = 0.05,
               every: int = 10) -> dict:
    data = BlobImages(dev)
    out = {"workload": f"ResNet-18 CIFAR-shape, N={n} co-resident workers, batch {batch}/worker, {steps} steps, "
                       f"SGD-Nesterov lr {lr} momentum 0.9, bf16 autocast, same init and data for every run",
           "data": "synthetic learnable 10-class task: class-mean image (amplitude 0.2) + N(0,1) noise, "
                   "fresh samples each step; eval = full model on 4096 held-out samples",
           "runs": {}}
    for tag, pp, strategy in (("subnet", p, "block"), ("widthwise", p, "neuron"), ("dp", n, "block")):
        model = train.build_resnet18(dev, seed=1)
        a = masking.build_assignment(model.topology, strategy, n, pp, seed=1)
        tr = train.SubnetTrainer(model, a, lr=lr, sync_layout=(strategy == "neuron"), graphed=True)
        curve = []
        t0 = time.perf_counter()
        for s in range(steps):
            batches = [data.batch(batch, seed=s * 1000 + w) for w in range(n)]
            loss = tr.step(batches)
            if s % every == 0 or s == steps - 1:
                curve.append([s, round(float(loss.item()), 5)])
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        tr.check()
        tr.write_back()
        ev = evaluate(model, data)
        out["runs"][tag] = {"p": pp, "strategy": strategy, "loss_curve": curve,
                            "train_loss_last10_mean": round(sum(c[1] for c in curve[-10:]) / len(curve[-10:]), 5),
                            "wall_s": round(wall, 2), **ev}
        del tr, model, a
        torch.cuda.empty_cache()
    r = out["runs"]
    out["eval_acc_gap_subnet_vs_dp"] = round(r["subnet"]["eval_acc"] - r["dp"]["eval_acc"], 4)
    out["eval_acc_gap_widthwise_vs_dp"] = round(r["widthwise"]["eval_acc"] - r["dp"]["eval_acc"], 4)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    res = equal_loss(torch.device("cuda", 0), steps=args.steps)
    s = json.dumps(res)
    print(s)
    if args.out:
        Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
