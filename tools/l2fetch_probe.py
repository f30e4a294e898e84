"""A/B of the context's maximum L2 fetch granularity (CU_LIMIT_MAX_L2_FETCH_GRANULARITY,
0-128 B) on the fragmented-owner kernels: the width-wise flat-layout sync
(C3 aggregate / write-back: 9-element owner runs, DRAM reads 1.35x the owned
bytes on 128-B lines, profiles/r2_ncu_sync_c3_flat.md), the C3 slices, and the
block-strategy sync as a no-regression control.  Probe-only (gpurun)."""
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import measure_all as M  # noqa: E402
from paper_2507_09029_b200 import engine, masking, models, zoo  # noqa: E402

CU_LIMIT_MAX_L2_FETCH_GRANULARITY = 0x05
_cuda = ctypes.CDLL("libcuda.so.1")


def get_limit() -> int:
    v = ctypes.c_size_t(0)
    rc = _cuda.cuCtxGetLimit(ctypes.byref(v), CU_LIMIT_MAX_L2_FETCH_GRANULARITY)
    return int(v.value) if rc == 0 else -rc


def set_limit(b: int) -> int:
    torch.cuda.synchronize()
    return _cuda.cuCtxSetLimit(CU_LIMIT_MAX_L2_FETCH_GRANULARITY, ctypes.c_size_t(b))


def main():
    M.FLUSH_W = torch.empty(64 << 20, device=M.DEV)
    M.FLUSH_R = torch.zeros(64 << 20, device=M.DEV)
    torch.zeros(1, device=M.DEV)
    default = get_limit()
    print(json.dumps({"default_limit": default}), flush=True)
    cases = []
    r18, g2 = zoo.resnet18_cifar_topology(), zoo.gpt2_small_topology()
    for name, topo, strategy in (("C3", r18, "neuron"), ("C2", r18, "block"), ("C4n", g2, "neuron")):
        a = masking.build_assignment(topo, strategy, 8, 4, seed=1)
        d = topo.total
        reps = [torch.randn(d, device=M.DEV) * a.param_masks[w] for w in range(8)]
        sh = [torch.zeros(d, dtype=torch.bfloat16, device=M.DEV) for _ in range(8)]
        out = torch.empty(d, device=M.DEV)
        plan = a.sync_plan()
        own = plan.owned_elems
        mixed = plan.n_tiles - plan.n_uniform
        tiled = engine.SyncPlan(a, direct=False, stream=False)
        agg_s = engine.PreparedSync(reps, a, writeback=False, out=out, plan=plan)
        agg_t = engine.PreparedSync(reps, a, writeback=False, out=out, plan=tiled)
        wb = engine.PreparedSync(reps, a, writeback=True, shadows_bf16=sh, plan=plan)
        cases.append((f"{name} aggregate (routed)", agg_s.launch, own * 4 + d * 4 + mixed * plan.tile))
        cases.append((f"{name} aggregate (tiled)", agg_t.launch, own * 4 + d * 4 + mixed * plan.tile))
        cases.append((f"{name} write-back+bf16", wb.launch, own * 10 + mixed * plan.tile))
        if name == "C3":
            subs = [models.SubnetLayout(a, w) for w in range(8)]
            tot = sum(s_.compact_total for s_ in subs)
            theta = torch.randn(d, device=M.DEV)
            gb = models.SliceBatch([s_.host_gather for s_ in subs], M.DEV)
            sb = models.SliceBatch([s_.host_scatter for s_ in subs], M.DEV)
            comps = [torch.empty(max(1, s_.compact_total), device=M.DEV) for s_ in subs]
            fulls = [torch.zeros(d, device=M.DEV) for _ in subs]
            cases.append(("C3 gather (all workers)", lambda: gb.gather([theta] * 8, comps), tot * 8))
            cases.append(("C3 scatter zero-fill (all workers)", lambda: sb.scatter(comps, fulls),
                          tot * 4 + 8 * d * 4))
            cases.append(("C3 scatter accumulate (all workers)",
                          lambda: sb.scatter(comps, fulls, accumulate=True), tot * 12))
    for gran in (default, 32, 64, 128, default):
        rc = set_limit(gran)
        got = get_limit()
        for tag, fn, nbytes in cases:
            us, mn = M.timed(fn, reps=30)
            print(json.dumps({"case": tag, "set": gran, "rc": rc, "limit": got, "us": round(us, 2),
                              "us_min": round(mn, 2), "frac": round(nbytes / us / 1e3 / M.PEAK, 3)}), flush=True)


if __name__ == "__main__":
    main()
