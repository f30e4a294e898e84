"""A/B timing of libsdp variants built by tools/variant_build.py (probe-only).

    python tools/variant_probe.py tools/_variants/<name>/libsdp.so [cases]

cases: comma list of c2,c3,c3agg,c3lay,c4,c4nagg,c3s,c4ns,c4n,c5n (default: the first six)
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
    # block plans, mean-only: tiled (routed default) vs the streaming kernel
    if "blkagg" in cases:
        M.sync_case(r18, f"[{tag}] C2 resnet18", "block", 8, 4, writeback=False, shadows=False)
        M.sync_case(r18, f"[{tag}] C2 resnet18 stream", "block", 8, 4, writeback=False, shadows=False,
                    direct=True, stream=True)
        M.sync_case(gpt2, f"[{tag}] C4 gpt2", "block", 8, 4, writeback=False, shadows=False)
        M.sync_case(gpt2, f"[{tag}] C4 gpt2 stream", "block", 8, 4, writeback=False, shadows=False,
                    direct=True, stream=True)
    # the slice kernels (per worker and all workers per launch)
    if "s3" in cases:
        M.slices_case(r18, f"[{tag}] C3 resnet18", "neuron", 8, 4)
    if "s4" in cases:
        M.slices_case(gpt2, f"[{tag}] C4 gpt2 (mlp units)", "neuron", 8, 4)
    # the mask builder (k_assign + k_build_masks)
    if "b2" in cases:
        M.build_case(r18, f"[{tag}] C2 resnet18", "block", 8, 4)
    if "b3" in cases:
        M.build_case(r18, f"[{tag}] C3 resnet18", "neuron", 8, 4)
    if "b4" in cases:
        M.build_case(gpt2, f"[{tag}] C4 gpt2", "block", 8, 4)
        M.build_case(gpt2, f"[{tag}] C4 gpt2 neuron", "neuron", 8, 4)
    # the streaming kernel forced onto the write-back launches (routing A/B)
    if "c3s" in cases:
        M.sync_case(r18, f"[{tag}] C3 resnet18 stream", "neuron", 8, 4, direct=True, stream=True)
    if "c4ns" in cases:
        M.sync_case(gpt2, f"[{tag}] C4 gpt2 width-wise stream", "neuron", 8, 4, direct=True, stream=True)
    if "c4n" in cases:
        M.sync_case(gpt2, f"[{tag}] C4 gpt2 width-wise", "neuron", 8, 4)
    if "c5n" in cases:
        c5 = zoo.mini_resnet_topology(512, 8, 10, 2, 3, (8, 8))
        M.sync_case(c5, f"[{tag}] C5 neuron c=512", "neuron", 8, 4, writeback=False, shadows=False)
        M.sync_case(c5, f"[{tag}] C5 neuron c=512", "neuron", 8, 4)
        M.sync_case(c5, f"[{tag}] C5 neuron c=512 stream", "neuron", 8, 4, direct=True, stream=True)


if __name__ == "__main__":
    main()
