"""Sync plan shape A/B (grid, tile, dispatch order) on the ~50-100 us syncs:
C3 width-wise in the sync layout (what the trainer runs) and C2 block.
Probe-only (gpurun)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import measure_all as M  # noqa: E402
from paper_2507_09029_b200 import zoo  # noqa: E402

M.FLUSH_W = torch.empty(64 << 20, device=M.DEV)
M.FLUSH_R = torch.zeros(64 << 20, device=M.DEV)
r18 = zoo.resnet18_cifar_topology()
variants = [("default", {}), ("one tile per CTA", {"force_grid": 5457}), ("grid 2368", {"max_grid": 2368}),
            ("grid 1184", {"max_grid": 1184}), ("order cost", {"order": "cost"}), ("order index", {"order": "index"}),
            ("tile 1024", {"tile": 1024}), ("tile 4096", {"tile": 4096})]
for rep in range(2):
    for name, kw in variants:
        kw = dict(kw)
        tile = kw.pop("tile", None)
        if "force_grid" in kw and tile is None:
            pass
        M.sync_case(r18, f"C3 sync layout [{name}]", "neuron", 8, 4, sync_layout=True, tile=tile, **kw)
        M.sync_case(r18, f"C2 [{name}]", "block", 8, 4, tile=tile, **kw)
