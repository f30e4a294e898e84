"""Time libsdp's LayerNorm kernels on the GPT-2 shape ([8192, 768] bf16)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2507_09029_b200 import train  # noqa: E402

dev = torch.device("cuda", 0)
x = torch.randn(8192, 768, device=dev).bfloat16().requires_grad_(True)
w = torch.ones(768, device=dev).bfloat16().requires_grad_(True)
b = torch.zeros(768, device=dev).bfloat16().requires_grad_(True)
dy = torch.randn(8192, 768, device=dev).bfloat16()
for _ in range(3):
    train._LayerNormBF16.apply(x, w, b, 1e-5).backward(dy)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(20):
        train._LayerNormBF16.apply(x, w, b, 1e-5).backward(dy)
    torch.cuda.synchronize()
for k in sorted(prof.key_averages(), key=lambda k: -k.device_time_total)[:8]:
    print(f"{k.device_time_total / k.count:8.2f} us x{k.count}  {k.key[:90]}")
