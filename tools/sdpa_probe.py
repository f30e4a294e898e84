"""SDPA backends on GPT-2's strided q/k/v views ([b, nh, t, hd] views of the
fused qkv GEMM output): fwd+bwd time and the copies each backend makes."""
import sys

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

b, t, nh, hd = 8, 1024, 12, 64
dev = torch.device("cuda", 0)
qkv = torch.randn(b * t, 3 * nh * hd, device=dev, dtype=torch.bfloat16, requires_grad=True)
gy = torch.randn(b, nh, t, hd, device=dev, dtype=torch.bfloat16)


def step():
    q, k, v = qkv.view(b, t, 3, nh, hd).permute(2, 0, 3, 1, 4)
    y = F.scaled_dot_product_attention(q, k, v, is_causal=True)
    y.backward(gy)


for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                 ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
    try:
        with sdpa_kernel([be]):
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(10):
                step()
            e.record()
            torch.cuda.synchronize()
            with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                                    torch.profiler.ProfilerActivity.CUDA]) as prof:
                step()
                torch.cuda.synchronize()
        cp = [k for k in prof.key_averages() if k.key in ("aten::copy_", "aten::contiguous", "aten::clone")]
        print(f"{name:10s} {s.elapsed_time(e) / 10 * 1e3:8.1f} us fwd+bwd;",
              ", ".join(f"{k.key} x{k.count} {k.device_time_total:.0f}us" for k in cp))
    except Exception as ex:  # noqa: BLE001
        print(name, "unavailable:", str(ex).splitlines()[0][:120])
sys.stdout.flush()
