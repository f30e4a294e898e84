"""A/B of two libsdp builds on the bench's device-resident sync (same box).

    python tools/sync_ab.py <path/to/libsdp.so|default> [workload] [reps]

Loads the given library in place of the in-tree one (an older build's
sdp_sync_args is a prefix of the current struct, so it ignores the new
fields), builds the bench workload (N=8, P=4, block, seed 1) and times `reps`
launches with the bench's L2 flush between them; prints one JSON line.
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2507_09029_b200 import _native  # noqa: E402

lib = sys.argv[1]
if lib != "default":
    _native.LIB_PATH = Path(lib)
    C_lib = __import__("ctypes").CDLL(lib)
    _native.ABI_VERSION = C_lib.sdp_abi_version()
_native.load(_native.LIB_PATH)
import bench  # noqa: E402
from paper_2507_09029_b200 import engine, masking  # noqa: E402

wl = sys.argv[2] if len(sys.argv) > 2 else "gpt2"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
dev = torch.device("cuda", 0)
topo, tag = bench.workload(wl)
a = masking.build_assignment(topo, "block", 8, 4, seed=1)
pm = a.param_masks
gen = torch.Generator(device=dev)
reps_ = []
for w in range(8):
    gen.manual_seed(1000 + w)
    reps_.append(torch.randn(topo.total, generator=gen, device=dev) * pm[w])
del pm
sh = [torch.zeros(topo.total, dtype=torch.bfloat16, device=dev) for _ in range(8)]
plan = a.sync_plan()
prep = engine.PreparedSync(reps_, a, writeback=True, shadows_bf16=sh, plan=plan)
flush = torch.empty(64 << 20, device=dev)
flush_rd = torch.zeros(64 << 20, device=dev)
for _ in range(5):
    prep.launch()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    flush.zero_()
    flush_rd.sum()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    prep.launch()
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
byt = plan.owned_elems * 10
print(json.dumps({"lib": lib, "workload": wl, "ms_median": float(np.median(ts)), "ms_mean": float(np.mean(ts)),
                  "frac_median": byt / (np.median(ts) / 1e3) / 1e9 / 6540.5}))
