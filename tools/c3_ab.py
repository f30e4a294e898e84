"""Same-box A/B of the sync plan shape for the width-wise (C3) sync layout:
tile size x grid x tile dispatch order (and C2 / C4 as controls)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import measure_all  # noqa: E402
from measure_all import sync_case  # noqa: E402

from paper_2507_09029_b200 import zoo  # noqa: E402

measure_all.FLUSH_W = torch.empty(64 << 20, device=measure_all.DEV)
measure_all.FLUSH_R = torch.zeros(64 << 20, device=measure_all.DEV)
r18 = zoo.resnet18_cifar_topology()
for order in ("index", "mixed_first", "cost"):
    for tile in (1024, 2048):
        for grid in (None, 148 * 8, 148 * 16):
            kw = {"order": order}
            if grid is not None:
                kw["force_grid"] = min(grid, -(-r18.total // tile))
            sync_case(r18, f"C3 sync layout tile {tile} grid {grid} {order}", "neuron", 8, 4, sync_layout=True,
                      tile=tile, **kw)
    sync_case(r18, f"C2 resnet18 {order}", "block", 8, 4, order=order)
    sync_case(r18, f"C3 flat {order}", "neuron", 8, 4, order=order)
