"""A/B of the slice task size (models.slice_tasks per_task) for the C3 / C4
width-wise gathers and scatters, per worker and all workers per launch.
Probe-only (run under gpurun)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import measure_all as M  # noqa: E402
from paper_2507_09029_b200 import masking, models, zoo  # noqa: E402


def main():
    M.FLUSH_W = torch.empty(64 << 20, device=M.DEV)
    M.FLUSH_R = torch.zeros(64 << 20, device=M.DEV)
    dev = M.DEV
    for name, topo in (("C3", zoo.resnet18_cifar_topology()), ("C4", zoo.gpt2_small_topology())):
        a = masking.build_assignment(topo, "neuron", 8, 4, seed=1)
        theta = torch.randn(topo.total, device=dev)
        for per in (2048, 4096, 8192, 16384, 32768):
            models.slice_tasks.__defaults__ = (per,)
            subs = [models.SubnetLayout(a, w) for w in range(8)]
            tot = sum(s.compact_total for s in subs)
            gb = models.SliceBatch([s.host_gather for s in subs], dev)
            sb = models.SliceBatch([s.host_scatter for s in subs], dev)
            comps = [torch.empty(max(1, s.compact_total), device=dev) for s in subs]
            fulls = [torch.empty(topo.total, device=dev) for _ in subs]
            row = {"cfg": name, "per_task": per}
            for key, fn, nbytes in (
                    ("gather_all", lambda: gb.gather([theta] * 8, comps), tot * 8),
                    ("scatter_zf_all", lambda: sb.scatter(comps, fulls), tot * 4 + 8 * topo.total * 4),
                    ("scatter_acc_all", lambda: sb.scatter(comps, fulls, accumulate=True), tot * 12),
                    ("scatter_zf_w0", lambda: subs[0].scatter(comps[0], fulls[0]),
                     subs[0].compact_total * 4 + topo.total * 4)):
                us, _ = M.timed(fn)
                row[key] = [round(us, 1), round(nbytes / us / 1e3 / M.PEAK, 3)]
            print(json.dumps(row), flush=True)
            del subs, gb, sb, comps, fulls
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
