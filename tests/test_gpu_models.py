"""Extraction / write-back (models.py:333-382) and the protocol step
(engine.py:202-223) on the GPU vs the reference's own outputs (golden vectors
from tests/golden/make_golden_models.py).

float64 throughout so the comparison isolates the math: losses within 1e-12
relative, gradients within 1e-10 of max|g| (cuDNN vs numpy summation order),
compact == full layout to 1e-12, extraction and scatter bit-exact."""

import json
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"
TOL_G = 1e-10


@lru_cache(maxsize=1)
def _golden():
    return json.loads((GOLDEN / "models.json").read_text()), dict(np.load(GOLDEN / "models.npz"))


def _case_ids():
    return [c["id"] for c in _golden()[0]["cases"]]


def _setup(ci, cuda):
    from paper_2507_09029_b200 import masking, models
    man, arr = _golden()
    c = man["cases"][ci]
    kw = dict(c["kw"])
    theta = torch.from_numpy(arr[f"m{ci}_theta0"]).to(cuda)
    if c["kind"] == "mini":
        kw["image_hw"] = tuple(kw["image_hw"])
        m = models.build_mini_resnet(**kw, dtype=torch.float64, theta=theta)
    else:
        m = models.build_residual_mlp(**kw, dtype=torch.float64, theta=theta)
    a = masking.build_assignment(m.topology, c["strategy"], c["n"], c["p"], c["seed"])
    return c, arr, m, a


@pytest.mark.parametrize("ci", _case_ids())
def test_masked_forward_and_flat_gradient_vs_reference(cuda, ci):
    from paper_2507_09029_b200 import models
    c, arr, m, a = _setup(ci, cuda)
    for w in range(c["n"]):
        view = a.worker_view(w)
        x, y = arr[f"m{ci}_x{w}"], arr[f"m{ci}_y{w}"]
        loss, tape, params = models.masked_forward(m, view, x, y)
        g = models.flat_gradient(m, tape, loss, params).cpu().numpy()
        ref_loss = arr[f"m{ci}_loss_w{w}"][0]
        ref_g = arr[f"m{ci}_grad_w{w}"]
        assert abs(loss.item() - ref_loss) <= 1e-12 * max(1.0, abs(ref_loss))
        assert np.max(np.abs(g - ref_g)) <= TOL_G * max(1.0, np.abs(ref_g).max())
        mask = view.param_mask_bool.cpu().numpy()
        assert np.all(g[~mask] == 0.0)  # masked gradients are exactly zero
        loss_m, _, _ = models.masked_forward(m, view, x, y, block_mode="multiply")
        assert abs(loss_m.item() - arr[f"m{ci}_lossmul_w{w}"][0]) <= 1e-12 * max(1.0, abs(ref_loss))


@pytest.mark.parametrize("ci", _case_ids())
def test_compact_subnetwork_matches_full_layout(cuda, ci):
    """Gather -> compact fwd/bwd -> scatter == masked full model."""
    from paper_2507_09029_b200 import models
    c, arr, m, a = _setup(ci, cuda)
    for w in range(c["n"]):
        view = a.worker_view(w)
        sub = models.SubnetLayout(a, w)
        x, y = arr[f"m{ci}_x{w}"], arr[f"m{ci}_y{w}"]
        loss_c, tape_c, cp = models.masked_forward(m, view, x, y, layout="compact", subnet=sub)
        g_c = models.flat_gradient(m, tape_c, loss_c, cp)
        ref_g = arr[f"m{ci}_grad_w{w}"]
        assert abs(loss_c.item() - arr[f"m{ci}_loss_w{w}"][0]) <= 1e-12 * max(1.0, abs(loss_c.item()))
        assert np.max(np.abs(g_c.cpu().numpy() - ref_g)) <= TOL_G * max(1.0, np.abs(ref_g).max())
        # compact size = the worker's active parameter count
        assert sub.compact_total == view.active_params


def test_extract_is_theta_times_mask_bitexact(cuda):
    from paper_2507_09029_b200 import models
    c, arr, m, a = _setup(0, cuda)
    th = m.theta.clone()
    th[::7] = -th[::7].abs()  # negative entries: theta * 0 must give -0.0 like numpy
    for w in range(c["n"]):
        view = a.worker_view(w)
        got = models._extract(th, view).cpu().numpy()
        want = th.cpu().numpy() * view.param_mask.cpu().numpy()
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("ci", _case_ids())
def test_gather_scatter_round_trip_bitexact(cuda, ci):
    from paper_2507_09029_b200 import models
    c, arr, m, a = _setup(ci, cuda)
    for w in range(c["n"]):
        sub = models.SubnetLayout(a, w)
        comp = sub.gather(m.theta)
        full = sub.scatter(comp).cpu().numpy()
        mask = a.worker_view(w).param_mask_bool.cpu().numpy()
        th = m.theta.cpu().numpy()
        assert np.array_equal(full[mask].view(np.uint64), th[mask].view(np.uint64))
        assert np.all(full[~mask] == 0.0)
        # compact tensors are the live rows/columns of the full ones
        views = sub.views(comp)
        for p in m.topology.params:
            if int(np.prod(sub.shapes[p.name])) == 0:
                continue
            full_p = th[p.offset:p.offset + p.size].reshape(p.shape)
            idx = []
            for axis in range(len(p.shape)):
                idx.append(np.arange(p.shape[axis]))
            for layer in m.topology.channel_layers:
                if a.strategy != "neuron" or not layer.maskable:
                    continue
                for pname, axis in tuple(layer.own_slices) + tuple(layer.consumer_slices):
                    if pname == p.name:
                        idx[axis] = np.nonzero(a.worker_view(w).channel_active[layer.layer_id])[0]
            want = full_p[np.ix_(*idx)]
            assert np.array_equal(views[p.name].cpu().numpy(), want)


@pytest.mark.parametrize("ci", _case_ids())
def test_compact_aggregate_bitexact_vs_full_aggregate(cuda, ci):
    from paper_2507_09029_b200 import engine, models
    c, arr, m, a = _setup(ci, cuda)
    subs = [models.SubnetLayout(a, w) for w in range(c["n"])]
    full_grads, comp_grads = [], []
    for w, sub in enumerate(subs):
        x, y = arr[f"m{ci}_x{w}"], arr[f"m{ci}_y{w}"]
        loss, tape, cp = models.masked_forward(m, a.worker_view(w), x, y, layout="compact", subnet=sub)
        (gc,) = torch.autograd.grad(loss, tape.leaf)
        comp_grads.append(gc.contiguous())
        full_grads.append(sub.scatter(gc.contiguous()))
    g1 = models.aggregate_compact(comp_grads, subs, a)
    g2 = engine.aggregate(full_grads, a).gbar
    assert torch.equal(g1.view(torch.int64), g2.view(torch.int64))


@pytest.mark.parametrize("ci", _case_ids())
def test_gradient_alignment_matches_reference(cuda, ci):
    """diagnostics.gradient_alignment (diagnostics.py:50-78) on the GPU reduction:
    same cosines within 1e-10, same absent-reason where the support is empty."""
    from paper_2507_09029_b200 import diagnostics
    c, arr, m, a = _setup(ci, cuda)
    layers = [p.name for p in m.topology.params if p.kind in ("conv_w", "linear_w")]
    for w in range(c["n"]):
        got = diagnostics.gradient_alignment(m, a.worker_view(w), arr[f"m{ci}_x{w}"], arr[f"m{ci}_y{w}"], layers)
        want = c["alignment"][w]
        assert [s.layer for s in got] == [x[0] for x in want]
        for s, (_, cos, reason) in zip(got, want):
            assert s.reason == reason
            if cos is None:
                assert s.cosine is None
            else:
                assert abs(s.cosine - cos) <= 1e-10


def test_restricted_cosine_edge_cases(cuda):
    from paper_2507_09029_b200 import diagnostics
    a = torch.tensor([1.0, 2.0, 0.0], device=cuda, dtype=torch.float64)
    b = torch.tensor([2.0, 4.0, 5.0], device=cuda, dtype=torch.float64)
    assert diagnostics.restricted_cosine(a, b, torch.tensor([0, 0, 0], device=cuda)) == (None, "empty-support")
    assert diagnostics.restricted_cosine(a, b, torch.tensor([0, 0, 1], device=cuda)) == (None, "zero-norm")
    cos, reason = diagnostics.restricted_cosine(a, b, torch.tensor([1, 1, 0], device=cuda))
    assert reason is None and abs(cos - 1.0) < 1e-15


@pytest.mark.parametrize("ci", _case_ids())
def test_two_protocol_steps_match_reference(cuda, ci):
    """per-worker masked grads -> owner sync with fused Nesterov, twice
    (engine.py:202-223): theta within 1e-10 of the reference's."""
    from paper_2507_09029_b200 import engine, models
    c, arr, m, a = _setup(ci, cuda)
    vel = torch.zeros_like(m.theta)
    for t, lr in enumerate(c["lrs"]):
        grads = []
        for w in range(c["n"]):
            k = t * c["n"] + w
            loss, tape, params = models.masked_forward(m, a.worker_view(w), arr[f"m{ci}_x{k}"], arr[f"m{ci}_y{k}"])
            grads.append(models.flat_gradient(m, tape, loss, params).contiguous())
        engine.owner_sync(grads, a, writeback=False,
                          nesterov={"theta": m.theta, "velocity": vel, "lr": lr, "momentum": 0.9})
        ref = arr[f"m{ci}_theta_step{t + 1}"]
        err = np.max(np.abs(m.theta.cpu().numpy() - ref))
        assert err <= TOL_G * max(1.0, np.abs(ref).max()), err


@pytest.mark.parametrize("strategy", ["block", "neuron"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_gather_scatter_all_paths_full_size(cuda, strategy, dtype):
    """ResNet-18 (C2/C3) through every slice-kernel path (16-B row copies,
    tiled column tables, flattened short rows, dropped tensors): gather then
    zero-fill scatter == theta on the worker's mask, 0 elsewhere; accumulate
    scatter == base + theta on the mask, base elsewhere (bit-exact)."""
    from paper_2507_09029_b200 import masking, models, zoo
    topo = zoo.resnet18_cifar_topology()
    a = masking.build_assignment(topo, strategy, 8, 4, seed=1)
    gen = torch.Generator(device=cuda)
    gen.manual_seed(9)
    theta = torch.randn(topo.total, generator=gen, device=cuda, dtype=dtype)
    base = torch.randn(topo.total, generator=gen, device=cuda, dtype=dtype)
    for w in (0, 5):
        sub = models.SubnetLayout(a, w)
        mask = a.worker_view(w).param_mask_bool
        comp = sub.gather(theta)
        assert comp.numel() >= sub.compact_total and int(mask.sum()) == sub.compact_total
        full = sub.scatter(comp)
        assert torch.equal(full, torch.where(mask, theta, torch.zeros((), dtype=dtype, device=cuda)))
        acc = sub.scatter(comp, base.clone(), accumulate=True)
        assert torch.equal(acc, torch.where(mask, base + theta, base))


@pytest.mark.parametrize("strategy,dtype", [("neuron", torch.float32), ("block", torch.float32),
                                            ("neuron", torch.float64), ("neuron", torch.bfloat16)])
def test_slice_batch_one_launch_equals_per_worker(cuda, strategy, dtype):
    """models.SliceBatch: all 8 workers' gathers (and zero-fill / accumulate
    scatters) in ONE sdp_*_slices_multi launch == the per-worker launches,
    bit for bit, for the flat layout and for the sync-layout transfers."""
    from paper_2507_09029_b200 import masking, models, zoo
    from paper_2507_09029_b200.layout import SyncLayout, WorkerTransfer
    topo = zoo.resnet18_cifar_topology()
    a = masking.build_assignment(topo, strategy, 8, 4, seed=1)
    gen = torch.Generator(device=cuda)
    gen.manual_seed(11)
    theta = torch.randn(topo.total, generator=gen, device=cuda).to(dtype)
    subs = [models.SubnetLayout(a, w) for w in range(8)]
    gb = models.SliceBatch([s.host_gather for s in subs], cuda)
    outs = [torch.empty(max(1, s.compact_total), dtype=dtype, device=cuda) for s in subs]
    gb.gather([theta] * 8, outs)
    for s, o in zip(subs, outs):
        ref = s.gather(theta)
        assert torch.equal(o[:s.compact_total].view(torch.uint8), ref[:s.compact_total].view(torch.uint8))
    if dtype == torch.bfloat16:
        return  # scatters are fp32 / fp64 only
    sb = models.SliceBatch([s.host_scatter for s in subs], cuda)
    fulls = [torch.full((topo.total,), 7.0, dtype=dtype, device=cuda) for _ in subs]
    sb.scatter(outs, fulls)
    base = torch.randn(topo.total, generator=gen, device=cuda).to(dtype)
    accs = [base.clone() for _ in subs]
    sb.scatter(outs, accs, accumulate=True)
    for s, o, f, acc in zip(subs, outs, fulls, accs):
        assert torch.equal(f, s.scatter(o))
        assert torch.equal(acc, s.scatter(o, base.clone(), accumulate=True))
    if strategy != "neuron" or dtype != torch.float32:
        return
    lay = SyncLayout(a)
    trs = [WorkerTransfer(lay, s) for s in subs]
    tb = models.SliceBatch([t.host for t in trs], cuda)
    ts = lay.to_sync(theta)
    comps = [torch.empty(max(1, s.compact_total), device=cuda) for s in subs]
    tb.gather(comps, [ts] * 8, reverse=True)
    grads = [torch.zeros(topo.total, device=cuda) for _ in subs]
    tb.gather(comps, grads)
    for t, c, g in zip(trs, comps, grads):
        assert torch.equal(c[:t.compact_total], t.to_compact(ts)[:t.compact_total])
        assert torch.equal(g, t.from_compact(c, torch.zeros(topo.total, device=cuda)))


@pytest.mark.parametrize("shape", [(64, (32, 32), 32), (16, (29, 35), 12), (8, (300, 212), 4), (64, (256, 256), 4),
                                   (4, (7, 1, 24), 16)])
def test_group_norm_backward_is_deterministic(cuda, shape):
    """k_gn_bwd + k_gn_bwd_fold: dx, dgamma and dbeta are bit-identical across
    repeated calls (per-CTA partial rows folded in a fixed order -- no
    floating-point atomics), for multi-CTA clusters, ragged groups and groups
    wider than the CTA (> 256 channels); dgamma / dbeta agree with fp32
    F.group_norm's to fold rounding."""
    import torch.nn.functional as F
    from paper_2507_09029_b200 import models
    b, counts, hw = shape
    c = sum(counts)
    gen = torch.Generator(device=cuda)
    gen.manual_seed(c + b)
    x = (torch.randn(b, c, hw, hw, generator=gen, device=cuda) * 2 + 0.5).to(torch.bfloat16)
    x = x.contiguous(memory_format=torch.channels_last).requires_grad_(True)
    gamma = torch.randn(c, generator=gen, device=cuda).requires_grad_(True)
    beta = torch.randn(c, generator=gen, device=cuda).requires_grad_(True)
    dy = torch.randn(b, c, hw, hw, generator=gen, device=cuda).to(torch.bfloat16)
    outs = []
    for _ in range(3):
        with torch.autocast("cuda", dtype=torch.bfloat16):
            y = models.ragged_group_norm(x, None, len(counts), gamma, beta, counts=counts, relu=True)
        outs.append(torch.autograd.grad(y, (x, gamma, beta), dy))
    for o in outs[1:]:
        for a_, b_ in zip(outs[0], o):
            assert torch.equal(a_.view(torch.int16) if a_.dtype == torch.bfloat16 else a_.view(torch.int32),
                               b_.view(torch.int16) if b_.dtype == torch.bfloat16 else b_.view(torch.int32))
    xr = x.detach().float().requires_grad_(True)
    gr, br = gamma.detach().float().requires_grad_(True), beta.detach().float().requires_grad_(True)
    parts, pos = [], 0
    for k in counts:
        parts.append(F.group_norm(xr[:, pos:pos + k], 1, gr[pos:pos + k], br[pos:pos + k]))
        pos += k
    rx, rg, rb = torch.autograd.grad(F.relu(torch.cat(parts, dim=1)), (xr, gr, br), dy.float())
    gx, gg, gb = outs[0]
    assert torch.allclose(gg, rg, rtol=1e-2, atol=1e-2 * rg.abs().max().item())
    assert torch.allclose(gb, rb, rtol=1e-2, atol=1e-2 * rb.abs().max().item())
    assert torch.allclose(gx.float(), rx, rtol=2e-2, atol=2e-2 * rx.abs().max().item())


@pytest.mark.parametrize("affine", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("relu", [False, True])
@pytest.mark.parametrize("counts", [(32, 32), (29, 35), (7, 1, 24)])
def test_channels_last_group_norm_matches_torch(cuda, relu, counts, affine):
    """libsdp's channels-last GroupNorm (+ReLU) over ragged contiguous groups
    == per-group F.group_norm in fp32 on the same bf16 input, forward and
    backward, to bf16 rounding."""
    import torch.nn.functional as F
    from paper_2507_09029_b200 import models
    gen = torch.Generator(device=cuda)
    gen.manual_seed(sum(counts) + relu)
    c = sum(counts)
    x = (torch.randn(8, c, 12, 12, generator=gen, device=cuda) * 2 + 0.5).to(torch.bfloat16)
    x = x.contiguous(memory_format=torch.channels_last).requires_grad_(True)
    gamma = torch.randn(c, generator=gen, device=cuda).to(affine).requires_grad_(True)
    beta = torch.randn(c, generator=gen, device=cuda).to(affine).requires_grad_(True)
    dy = torch.randn(8, c, 12, 12, generator=gen, device=cuda).to(torch.bfloat16)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        y = models.ragged_group_norm(x, None, len(counts), gamma, beta, counts=counts, relu=relu)
    assert y.is_contiguous(memory_format=torch.channels_last)
    gx, gg, gb = torch.autograd.grad(y, (x, gamma, beta), dy)
    # reference: fp32 per-group F.group_norm on the same values
    xr = x.detach().float().requires_grad_(True)
    gr, br = gamma.detach().float().requires_grad_(True), beta.detach().float().requires_grad_(True)
    outs, pos = [], 0
    for k in counts:
        outs.append(F.group_norm(xr[:, pos:pos + k], 1, gr[pos:pos + k], br[pos:pos + k]))
        pos += k
    yr = torch.cat(outs, dim=1)
    if relu:
        yr = F.relu(yr)
    rx, rg, rb = torch.autograd.grad(yr, (xr, gr, br), dy.float())
    assert torch.allclose(y.float(), yr, rtol=1e-2, atol=2e-2)
    assert torch.allclose(gx.float(), rx, rtol=2e-2, atol=2e-2 * rx.abs().max().item())
    assert gg.dtype == affine and gb.dtype == affine
    assert torch.allclose(gg.float(), rg, rtol=1e-2, atol=1e-2 * rg.abs().max().item())
    assert torch.allclose(gb.float(), rb, rtol=1e-2, atol=1e-2 * rb.abs().max().item())


def test_slice_batch_accumulate_stays_in_bounds(cuda):
    """Guard bands around every worker's full vector: the batched
    accumulate / zero-fill scatters and the gather write only inside their
    own [0, d) / [0, compact) ranges."""
    from paper_2507_09029_b200 import masking, models, zoo
    topo = zoo.mini_resnet_topology(26, 8, 10, 2, 3, (8, 8))
    a = masking.build_assignment(topo, "neuron", 8, 3, seed=21)
    d = topo.total
    subs = [models.SubnetLayout(a, w) for w in range(8)]
    guard = 4096
    gen = torch.Generator(device=cuda)
    gen.manual_seed(5)
    theta = torch.randn(d, generator=gen, device=cuda)
    cbig = [torch.full((max(1, s.compact_total) + guard,), 3.0, device=cuda) for s in subs]
    comps = [c[:max(1, s.compact_total)] for c, s in zip(cbig, subs)]
    models.SliceBatch([s.host_gather for s in subs], cuda).gather([theta] * 8, comps)
    fbig = [torch.full((d + guard,), 5.0, device=cuda) for _ in subs]
    fulls = [f[:d] for f in fbig]
    sb = models.SliceBatch([s.host_scatter for s in subs], cuda)
    sb.scatter(comps, fulls)
    sb.scatter(comps, fulls, accumulate=True)
    torch.cuda.synchronize()
    for c, s in zip(cbig, subs):
        assert torch.all(c[max(1, s.compact_total):] == 3.0)
    for f, s in zip(fbig, subs):
        assert torch.all(f[d:] == 5.0)
    # zero fill then accumulate == 2 * theta on the worker's mask, 0 elsewhere
    pm = a.param_masks
    for w, f in enumerate(fulls):
        assert torch.equal(f, torch.where(pm[w], theta + theta, torch.zeros_like(theta)))
