"""Run each width-wise extraction / write-back kernel once per config (ncu target).

    ncu --set full -k regex:'k_gather|k_scatter' python tools/slices_probe.py

Configs: C3 ResNet-18 and C4 GPT-2 (mlp units), neuron strategy, N = 8, P = 4,
worker 0.  Launch order per config: gather, scatter(zero-fill),
scatter(accumulate), to_sync, from_sync, to_compact, from_compact.
"""

import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2507_09029_b200 import _native as N  # noqa: E402
from paper_2507_09029_b200 import masking, models, zoo  # noqa: E402
from paper_2507_09029_b200.layout import SyncLayout, WorkerTransfer  # noqa: E402


def main():
    N.load()
    dev = torch.device("cuda", 0)
    which = sys.argv[1:] or ["r18", "gpt2"]
    for name in which:
        topo = zoo.resnet18_cifar_topology() if name == "r18" else zoo.gpt2_small_topology()
        a = masking.build_assignment(topo, "neuron", 8, 4, seed=1)
        sub = models.SubnetLayout(a, 0)
        lay = SyncLayout(a)
        tr = WorkerTransfer(lay, sub)
        theta = torch.randn(topo.total, device=dev)
        comp = torch.empty(sub.compact_total, device=dev)
        full = torch.empty(topo.total, device=dev)
        ts = torch.empty_like(theta)
        torch.cuda.synchronize()
        sub.gather(theta, comp)
        sub.scatter(comp, full)
        sub.scatter(comp, full, accumulate=True)
        lay.to_sync(theta, ts)
        lay.from_sync(ts, theta)
        tr.to_compact(ts, comp)
        tr.from_compact(comp, ts)
        torch.cuda.synchronize()
        print(name, "compact", sub.compact_total, "d", topo.total, "tasks g/s", sub.n_gather,
              sub.n_scatter, "sync tasks", lay.n_tasks, "transfer tasks", tr.n_tasks)


if __name__ == "__main__":
    main()
