"""A/B timing of libsdp variants built by tools/variant_build.py (probe-only).

    python tools/variant_probe.py tools/_variants/<name>/libsdp.so [cases]

cases: comma list of c2,c3,c3agg,c3lay,c4,c4nagg (default: all)
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
from paper_2507_09029_b200 import _native as N  # noqa: E402

N.load(sys.argv[1])
import measure_all as M  # noqa: E402
from paper_2507_09029_b200 import zoo  # noqa: E402


def main():
    cases = set((sys.argv[2] if len(sys.argv) > 2 else "c2,c3,c3agg,c3lay,c4,c4nagg").split(","))
    M.FLUSH_W = torch.empty(64 << 20, device=M.DEV)
    M.FLUSH_R = torch.zeros(64 << 20, device=M.DEV)
    tag = Path(sys.argv[1]).parent.name
    r18, gpt2 = zoo.resnet18_cifar_topology(), zoo.gpt2_small_topology()
    if "c2" in cases:
        M.sync_case(r18, f"[{tag}] C2 resnet18", "block", 8, 4)
    if "c3" in cases:
        M.sync_case(r18, f"[{tag}] C3 resnet18", "neuron", 8, 4)
    if "c3agg" in cases:
        M.sync_case(r18, f"[{tag}] C3 resnet18", "neuron", 8, 4, writeback=False, shadows=False)
    if "c3lay" in cases:
        M.sync_case(r18, f"[{tag}] C3 resnet18 (sync layout)", "neuron", 8, 4, sync_layout=True)
    if "c4" in cases:
        M.sync_case(gpt2, f"[{tag}] C4 gpt2", "block", 8, 4)
    if "c4nagg" in cases:
        M.sync_case(gpt2, f"[{tag}] C4 gpt2 width-wise", "neuron", 8, 4, writeback=False, shadows=False)


if __name__ == "__main__":
    main()
