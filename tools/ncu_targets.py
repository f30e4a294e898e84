"""Launch a few libsdp kernels once each (after warm-up) for an ncu capture.

    ncu --set full --import-source on -k regex:'k_build|k_gather|k_scatter' -s <n> \
        python tools/ncu_targets.py
"""

import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2507_09029_b200 import masking, models, zoo  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    which = sys.argv[1:] or ["build_gpt2", "slices_r18", "sync_r18"]
    if "build_gpt2" in which:
        g = zoo.gpt2_small_topology()
        tables = masking._DeviceTables(g, "block", dev)
        ub = masking._device_assign(tables.table.groups, tables.table.n_units, 8, 4, 1, dev)
        for _ in range(3):
            masking._expand(g, tables, ub, 8, dev)
    if "slices_r18" in which or "slices_gpt2" in which:
        topo = zoo.resnet18_cifar_topology() if "slices_r18" in which else zoo.gpt2_small_topology()
        a = masking.build_assignment(topo, "neuron", 8, 4, seed=1)
        sub = models.SubnetLayout(a, 0)
        theta = torch.randn(topo.total, device=dev)
        comp = torch.empty(sub.compact_total, device=dev)
        full = torch.empty(topo.total, device=dev)
        for _ in range(3):
            sub.gather(theta, comp)
            sub.scatter(comp, full)
    if "slices_all_r18" in which:  # all 8 workers per launch (models.SliceBatch)
        topo = zoo.resnet18_cifar_topology()
        a = masking.build_assignment(topo, "neuron", 8, 4, seed=1)
        subs = [models.SubnetLayout(a, w) for w in range(8)]
        gb = models.SliceBatch([s.host_gather for s in subs], dev)
        sb = models.SliceBatch([s.host_scatter for s in subs], dev)
        theta = torch.randn(topo.total, device=dev)
        comps = [torch.empty(max(1, s.compact_total), device=dev) for s in subs]
        fulls = [torch.empty(topo.total, device=dev) for _ in subs]
        for _ in range(4):
            gb.gather([theta] * 8, comps)
            sb.scatter(comps, fulls)
            sb.scatter(comps, fulls, accumulate=True)
    if "sync_r18" in which:
        from paper_2507_09029_b200 import engine
        topo = zoo.resnet18_cifar_topology()
        for strategy in ("block", "neuron"):
            a = masking.build_assignment(topo, strategy, 8, 4, seed=1)
            reps = [torch.randn(topo.total, device=dev) * a.param_masks[w] for w in range(8)]
            sh = [torch.zeros(topo.total, dtype=torch.bfloat16, device=dev) for _ in range(8)]
            prep = engine.PreparedSync(reps, a, writeback=True, shadows_bf16=sh)
            for _ in range(3):
                prep.launch()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
