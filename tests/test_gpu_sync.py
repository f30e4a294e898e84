"""k_owner_sync vs the reference's aggregate (golden) and the fp32 restatement.

Criteria:
  1. float64: bit-identical to reference engine.aggregate;
  2. float32: bit-identical to the oracle's ordered fp32 recurrence, and within
     |out - ref| <= 1e-6 * max(|ref|, sum_owners|g| / P) of the float64 reference
     (the condition-scaled tolerance; north star: 1e-6 relative in fp32);
  3. bf16 output == RNE(fp32 output) bit for bit (=> <= 1 ulp vs bf16(ref)).
"""

import numpy as np
import pytest
import torch

import _golden as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu

REL_TOL_F32 = 1e-6


def _pkg():
    from paper_2507_09029_b200 import engine, masking
    return engine, masking


def _build(case):
    _, masking = _pkg()
    return masking.build_assignment(G.topology(case["model"]), case["strategy"], case["n"],
                                    case["p"], case["seed"])


@pytest.mark.parametrize("case", G.cases(with_grads=True), ids=lambda c: f"c{c['id']}-{c['strategy']}-N{c['n']}P{c['p']}")
def test_aggregate_f64_bitexact_vs_reference(cuda, case):
    engine, _ = _pkg()
    a = _build(case)
    masks = G.case_masks(case)
    grads, _, _ = G.case_inputs(case, masks)
    dev_grads = [torch.from_numpy(g).to(cuda) for g in grads]
    out = engine.aggregate(dev_grads, a)
    ref = G.arrays()[f"c{case['id']}_gbar"]
    assert np.array_equal(out.gbar.cpu().numpy().view(np.uint64), ref.view(np.uint64))
    assert torch.equal(out.divisor, a.divisor)
    # host numpy path (end-to-end) returns the same bits
    host = engine.aggregate(list(grads), a)
    assert np.array_equal(host.gbar.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("case", G.cases(with_grads=True), ids=lambda c: f"c{c['id']}")
def test_aggregate_f32_bitexact_vs_restatement_and_tolerance(cuda, case):
    engine, _ = _pkg()
    a = _build(case)
    masks = G.case_masks(case)
    grads, _, _ = G.case_inputs(case, masks)
    g32 = grads.astype(np.float32)
    out = engine.aggregate([torch.from_numpy(g).to(cuda) for g in g32], a).gbar.cpu().numpy()
    want = O.aggregate_f32_ordered(list(g32), masks)
    assert np.array_equal(out.view(np.uint32), want.view(np.uint32))
    ref = O.aggregate_f64(list(g32.astype(np.float64)), masks, np.maximum(masks.sum(0), 1).astype(np.float64))
    scale = np.maximum(np.abs(ref), (np.abs(g32.astype(np.float64)) * masks).sum(0) / np.maximum(masks.sum(0), 1))
    assert np.all(np.abs(out - ref) <= REL_TOL_F32 * scale)


def _pinned(arr):
    t = torch.empty(arr.shape, dtype=torch.from_numpy(arr).dtype, pin_memory=True)
    t.copy_(torch.from_numpy(arr))
    return t.numpy()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_host_paths_bitexact(cuda, dtype):
    """engine.aggregate on numpy inputs: pinned (zero-copy kernel reads over
    PCIe, writes the mean into pinned memory), pageable (pipelined copies) and
    device inputs give the same bits, and the reference's bits in float64."""
    engine, _ = _pkg()
    for case in G.cases(with_grads=True)[:6]:
        a = _build(case)
        masks = G.case_masks(case)
        grads, _, _ = G.case_inputs(case, masks)
        g = grads.astype(dtype)
        pinned = engine.aggregate([_pinned(x) for x in g], a).gbar
        pageable = engine.aggregate(list(g), a).gbar
        dev = engine.aggregate([torch.from_numpy(x).to(cuda) for x in g], a).gbar.cpu().numpy()
        view = np.uint64 if dtype == np.float64 else np.uint32
        assert np.array_equal(pinned.view(view), dev.view(view))
        assert np.array_equal(pageable.view(view), dev.view(view))
        if dtype == np.float64:
            ref = G.arrays()[f"c{case['id']}_gbar"]
            assert np.array_equal(pinned.view(np.uint64), ref.view(np.uint64))


def test_zero_copy_eligibility(cuda):
    """Only page-locked host memory mapped at the same device address takes the
    zero-copy path; pageable numpy and device tensors do not."""
    engine, _ = _pkg()
    pinned = torch.from_numpy(_pinned(np.zeros(64, dtype=np.float32)))
    assert engine._device_readable(pinned)
    assert not engine._device_readable(torch.from_numpy(np.zeros(64, dtype=np.float32)))
    assert not engine._device_readable(torch.zeros(64, device=cuda))


def test_host_results_are_fresh(cuda):
    """The pinned result pool never hands out a buffer the caller still holds
    (engine.py:60-79 returns a fresh gbar every call)."""
    engine, _ = _pkg()
    case = G.cases(with_grads=True)[0]
    a = _build(case)
    masks = G.case_masks(case)
    grads, _, _ = G.case_inputs(case, masks)
    g1 = [_pinned(x) for x in grads.astype(np.float32)]
    g2 = [_pinned(x * 2) for x in grads.astype(np.float32)]
    r1 = engine.aggregate(g1, a).gbar
    keep = r1.copy()
    sub = r1[1:]  # a view keeps the buffer in use too
    del r1
    r2 = engine.aggregate(g2, a).gbar
    assert np.array_equal(sub, keep[1:])
    assert np.shares_memory(sub, r2) is False
    assert np.array_equal(r2, keep * 2)


def test_uncovered_leak_pinned_host(cuda):
    engine, _ = _pkg()
    from paper_2507_09029_b200.errors import ProtocolError
    case = next(c for c in G.cases(with_grads=True) if c["uncovered_params"] > 0)
    a = _build(case)
    masks = G.case_masks(case)
    grads, _, _ = G.case_inputs(case, masks)
    unc = np.nonzero(~masks.any(0))[0]
    grads[1, unc[0]] = np.nan
    with pytest.raises(ProtocolError, match="zero mask coverage"):
        engine.aggregate([_pinned(x) for x in grads], a)


def test_uncovered_leak_pageable_host(cuda):
    """The staged pageable path (what engine.run passes) keeps the
    engine.py:75-78 leak check: every worker's full range is staged."""
    engine, _ = _pkg()
    from paper_2507_09029_b200.errors import ProtocolError
    case = next(c for c in G.cases(with_grads=True) if c["uncovered_params"] > 0)
    a = _build(case)
    masks = G.case_masks(case)
    grads, _, _ = G.case_inputs(case, masks)
    unc = np.nonzero(~masks.any(0))[0]
    grads[1, unc[-1]] = np.nan
    with pytest.raises(ProtocolError, match="zero mask coverage"):
        engine.aggregate([np.array(x) for x in grads], a)


@pytest.mark.parametrize("strategy", ["block", "neuron"])
def test_pageable_staged_many_chunks_bitexact(cuda, strategy, monkeypatch):
    """engine.aggregate on pageable numpy inputs with tiny staging chunks
    (many chunks, every staging slot reused several times): the same bits as
    the device-input path and the ordered restatement."""
    engine, masking = _pkg()
    from paper_2507_09029_b200 import zoo
    monkeypatch.setattr(engine, "STAGE_CHUNK_BYTES", 1 << 16)
    monkeypatch.setattr(engine, "STAGE_PIECE", 1 << 12)
    topo = zoo.mini_resnet_topology(26, 8, 10, 2, 3, (8, 8))
    a = masking.build_assignment(topo, strategy, 8, 3, seed=4)
    masks = a.param_masks.cpu().numpy()
    rng = np.random.default_rng(3)
    g32 = (rng.standard_normal((8, topo.total)) * masks).astype(np.float32)
    host = engine.aggregate([np.array(g) for g in g32], a).gbar
    dev = engine.aggregate([torch.from_numpy(g).to(cuda) for g in g32], a).gbar.cpu().numpy()
    assert np.array_equal(host.view(np.uint32), dev.view(np.uint32))
    assert np.array_equal(host.view(np.uint32), O.aggregate_f32_ordered(list(g32), masks).view(np.uint32))


@pytest.mark.parametrize("strategy", ["block", "neuron"])
def test_pinned_copy_pipeline_bitexact(cuda, strategy):
    """The copy-engine pipeline over pinned inputs (the measured alternative
    to the zero-copy path, profiles/r2_pinned_pipeline_ab.jsonl) with many
    small chunks == the zero-copy path == the ordered restatement."""
    engine, masking = _pkg()
    from paper_2507_09029_b200 import zoo
    topo = zoo.mini_resnet_topology(26, 8, 10, 2, 3, (8, 8))
    a = masking.build_assignment(topo, strategy, 8, 3, seed=9)
    masks = a.param_masks.cpu().numpy()
    rng = np.random.default_rng(8)
    g32 = (rng.standard_normal((8, topo.total)) * masks).astype(np.float32)
    pinned = [torch.from_numpy(g).pin_memory() for g in g32]
    check = a.uncovered_params > 0
    pipe = engine._host_staged(None, a, check, pinned=pinned, chunk_bytes=1 << 16).gbar.copy()
    zero = engine.aggregate([p.numpy() for p in pinned], a).gbar
    assert np.array_equal(pipe.view(np.uint32), zero.view(np.uint32))
    assert np.array_equal(pipe.view(np.uint32), O.aggregate_f32_ordered(list(g32), masks).view(np.uint32))


def test_disjoint_known_answer(cuda):
    """m1=[1,0], m2=[0,1], g1=[2,0], g2=[0,4] -> [2,4]."""
    engine, masking = _pkg()
    from paper_2507_09029_b200 import zoo
    topo = zoo.residual_mlp_topology(width=1, blocks=2, classes=1, in_dim=1)
    # blocks 0 and 1 (2 params each) on disjoint workers
    ba = np.array([[1, 0], [0, 1]], dtype=bool)
    pm = masking.induce_block_param_mask(topo, ba)
    a = masking.MaskAssignment(2, 1, "block", 0, topo, {}, pm, torch.zeros(topo.total, dtype=torch.int64))
    g = [torch.zeros(topo.total, dtype=torch.float64, device=cuda) for _ in range(2)]
    b0, b1 = topo.slice_of("block0.lin1.w"), topo.slice_of("block1.lin1.w")
    g[0][b0] = 2.0
    g[1][b1] = 4.0
    out = engine.aggregate(g, a).gbar
    assert out[b0].item() == 2.0 and out[b1].item() == 4.0


def test_wrong_count_raises_protocol_error(cuda):
    engine, _ = _pkg()
    from paper_2507_09029_b200.errors import ProtocolError
    case = G.cases(with_grads=True)[0]
    a = _build(case)
    with pytest.raises(ProtocolError, match="gradients for"):
        engine.aggregate([torch.zeros(case["d"], device=cuda)], a)


def test_uncovered_leak_raises_protocol_error(cuda):
    """engine.py:75-78: a non-finite entry at a zero-coverage parameter."""
    engine, _ = _pkg()
    from paper_2507_09029_b200.errors import ProtocolError
    case = next(c for c in G.cases(with_grads=True) if c["uncovered_params"] > 0)
    a = _build(case)
    masks = G.case_masks(case)
    grads, _, _ = G.case_inputs(case, masks)
    unc = np.nonzero(~masks.any(0))[0]
    grads[1, unc[0]] = np.inf
    with pytest.raises(ProtocolError, match="zero mask coverage"):
        engine.aggregate([torch.from_numpy(g).to(cuda) for g in grads], a)
    # finite junk at an uncovered entry is masked away exactly as 0*g is
    grads[1, unc[0]] = 3.0
    out = engine.aggregate([torch.from_numpy(g).to(cuda) for g in grads], a).gbar
    assert out[int(unc[0])].item() == 0.0


def _replicas(a, dtype, seed, cuda):
    """N logical replicas, seeded randn, zero off-mask (reference nullity)."""
    n, d = a.n_workers, a.topology.total
    gen = torch.Generator(device=cuda)
    reps = []
    pm = a.param_masks
    for w in range(n):
        gen.manual_seed(seed + w)
        reps.append(torch.randn(d, generator=gen, device=cuda, dtype=torch.float32).to(dtype) * pm[w])
    return reps


@pytest.mark.parametrize("strategy", ["block", "neuron"])
def test_writeback_bf16_and_replica_identity(cuda, strategy):
    """Replica mode: every owner ends with the identical mean; bf16 shadow == RNE(fp32)."""
    engine, masking = _pkg()
    from paper_2507_09029_b200 import zoo
    topo = zoo.mini_resnet_topology(26, 8, 10, 2, 3, (32, 32))
    a = masking.build_assignment(topo, strategy, 8, 3, seed=1)
    reps = _replicas(a, torch.float32, 1000, cuda)
    host = [r.cpu().numpy() for r in reps]
    masks = a.param_masks.cpu().numpy()
    want = O.aggregate_f32_ordered(host, masks)
    shadows = [torch.zeros(topo.total, dtype=torch.bfloat16, device=cuda) for _ in reps]
    out = torch.empty(topo.total, device=cuda)
    outb = torch.empty(topo.total, dtype=torch.bfloat16, device=cuda)
    engine.owner_sync(reps, a, out=out, out_bf16=outb, shadows_bf16=shadows)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32))
    wb = O.bf16_rne(want)
    assert np.array_equal(outb.view(torch.int16).cpu().numpy().view(np.uint16), wb)
    for w in range(8):
        m = masks[w]
        got = reps[w].cpu().numpy()
        assert np.array_equal(got[m].view(np.uint32), want[m].view(np.uint32))
        assert np.array_equal(got[~m], host[w][~m])  # non-owned entries untouched
        sh = shadows[w].view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(sh[m], wb[m]) and np.all(sh[~m] == 0)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_fused_nesterov_matches_reference_step(cuda, dtype):
    """SDP_SYNC_NESTEROV epilogue == aggregate then optim.SgdNesterov.update (optim.py:78-84)."""
    engine, _ = _pkg()
    for case in G.cases(with_grads=True)[:6]:
        a = _build(case)
        masks = G.case_masks(case)
        grads, theta0, vel0 = G.case_inputs(case, masks)
        npdt = np.float64 if dtype == torch.float64 else np.float32
        th = torch.from_numpy(theta0.astype(npdt)).to(cuda)
        ve = torch.from_numpy(vel0.astype(npdt)).to(cuda)
        reps = [torch.from_numpy(g.astype(npdt)).to(cuda) for g in grads]
        thb = torch.empty(case["d"], dtype=torch.bfloat16, device=cuda)
        engine.owner_sync(reps, a, writeback=False,
                          nesterov={"theta": th, "velocity": ve, "lr": 0.05, "momentum": 0.9,
                                    "theta_bf16": thb})
        if dtype == torch.float64:
            assert np.array_equal(th.cpu().numpy().view(np.uint64),
                                  G.arrays()[f"c{case['id']}_theta1"].view(np.uint64))
            assert np.array_equal(ve.cpu().numpy().view(np.uint64),
                                  G.arrays()[f"c{case['id']}_vel1"].view(np.uint64))
        else:
            g = O.aggregate_f32_ordered(list(grads.astype(np.float32)), masks)
            t1, v1 = O.nesterov_update(theta0.astype(np.float32), vel0.astype(np.float32), g, 0.05, 0.9)
            assert np.array_equal(th.cpu().numpy().view(np.uint32), t1.astype(np.float32).view(np.uint32))
            assert np.array_equal(ve.cpu().numpy().view(np.uint32), v1.astype(np.float32).view(np.uint32))
            assert np.array_equal(thb.view(torch.int16).cpu().numpy().view(np.uint16), O.bf16_rne(t1))


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_fused_adam_matches_reference_steps(cuda, dtype):
    """SDP_SYNC_ADAM epilogue, two steps == reference optim.Adam (optim.py:90-109)."""
    engine, _ = _pkg()
    npdt = np.float64 if dtype == torch.float64 else np.float32
    for case in G.cases(with_grads=True)[:6]:
        a = _build(case)
        masks = G.case_masks(case)
        grads, _, _ = G.case_inputs(case, masks)
        arr = G.arrays()
        th = torch.from_numpy(arr[f"c{case['id']}_theta1"].astype(npdt)).to(cuda)
        m = torch.zeros_like(th)
        v = torch.zeros_like(th)
        thb = torch.empty(case["d"], dtype=torch.bfloat16, device=cuda)
        for t, scale in ((1, 1.0), (2, 0.5)):
            reps = [torch.from_numpy((g * scale).astype(npdt)).to(cuda) for g in grads]
            engine.owner_sync(reps, a, writeback=False,
                              adam={"theta": th, "m": m, "v": v, "lr": 0.01, "t": t, "theta_bf16": thb})
        if dtype == torch.float64:
            # the scaled gradients aggregate to exactly 0.5 * gbar (power-of-two scaling)
            assert np.array_equal(th.cpu().numpy().view(np.uint64), arr[f"c{case['id']}_adam_theta2"].view(np.uint64))
            assert np.array_equal(m.cpu().numpy().view(np.uint64), arr[f"c{case['id']}_adam_m2"].view(np.uint64))
            assert np.array_equal(v.cpu().numpy().view(np.uint64), arr[f"c{case['id']}_adam_v2"].view(np.uint64))
        else:
            g32 = [grads.astype(np.float32), (grads * 0.5).astype(np.float32)]
            t0 = arr[f"c{case['id']}_theta1"].astype(np.float32)
            mm, vv = np.zeros_like(t0), np.zeros_like(t0)
            for t, gs in ((1, g32[0]), (2, g32[1])):
                gbar = O.aggregate_f32_ordered(list(gs), masks)
                t0, mm, vv = O.adam_update(t0, mm, vv, gbar, 0.01, t)
            assert np.array_equal(th.cpu().numpy().view(np.uint32), t0.view(np.uint32))
            assert np.array_equal(thb.view(torch.int16).cpu().numpy().view(np.uint16), O.bf16_rne(t0))


def test_fused_adam_device_step_equals_host_step(cuda):
    """The graph-replayable form of the fused Adam (a device int32 step and
    engine.adam_bias_table) == the host-t form, which the golden test pins to
    the reference's optim.Adam; the table holds 1 - beta**t exactly as
    optim.py:107-108 computes it and ends where both corrections are 1.0."""
    engine, _ = _pkg()
    tab = engine.adam_bias_table(0.9, 0.999, cuda).cpu().numpy().reshape(-1, 2)
    for t in (1, 2, 17, 300, len(tab) - 1):
        assert tab[t, 0] == 1 - 0.9 ** t and tab[t, 1] == 1 - 0.999 ** t
    assert tab[-1, 0] == 1.0 and tab[-1, 1] == 1.0 and tab[-2, 1] != 1.0
    case = G.cases(with_grads=True)[1]
    a = _build(case)
    masks = G.case_masks(case)
    grads, _, _ = G.case_inputs(case, masks)
    th0 = torch.from_numpy(G.arrays()[f"c{case['id']}_theta1"]).to(cuda)
    outs = []
    for mode in ("host", "device"):
        th, m, v = th0.clone(), torch.zeros_like(th0), torch.zeros_like(th0)
        step = torch.zeros(1, dtype=torch.int32, device=cuda)
        dtab = engine.adam_bias_table(0.9, 0.999, cuda)
        for t in (1, 2, 3):
            reps = [torch.from_numpy(g * (0.5 ** t)).to(cuda) for g in grads]
            opt = {"theta": th, "m": m, "v": v, "lr": 0.01}
            if mode == "host":
                opt["t"] = t
            else:
                step.add_(1)
                opt.update(step=step, bias_table=dtab)
            engine.owner_sync(reps, a, writeback=False, adam=opt)
        outs.append((th, m, v))
    for x, y in zip(*outs):
        assert torch.equal(x, y)


def test_standalone_nesterov_and_nonfinite(cuda):
    engine, _ = _pkg()
    from paper_2507_09029_b200.errors import NumericalError
    d = 10001
    rng = np.random.default_rng(3)
    th0, g = rng.standard_normal(d), rng.standard_normal(d)
    opt = engine.SgdNesterov(d, momentum=0.9, dtype=torch.float64)
    th = torch.from_numpy(th0).to(cuda)
    opt.update(th, torch.from_numpy(g).to(cuda), 0.1)
    t1, v1 = O.nesterov_update(th0, np.zeros(d), g, 0.1, 0.9)
    assert np.array_equal(th.cpu().numpy().view(np.uint64), t1.view(np.uint64))
    g[5] = np.nan
    with pytest.raises(NumericalError):
        opt.update(th, torch.from_numpy(g).to(cuda), 0.1)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_standalone_adam_and_make_optimizer(cuda, dtype):
    """engine.Adam / engine.make_optimizer: three optim.Adam.update steps
    (optim.py:101-109) bit-identical to the restatement (f64: the reference's
    own arithmetic); a non-finite gradient raises before t, m, v or theta move."""
    engine, _ = _pkg()
    from paper_2507_09029_b200.errors import ConfigError, NumericalError
    npdt = np.float64 if dtype == torch.float64 else np.float32
    d = 20011
    rng = np.random.default_rng(9)
    th0 = rng.standard_normal(d).astype(npdt)
    opt = engine.make_optimizer("adam", d)
    assert opt.kind == "adam" and engine.make_optimizer("sgd-nesterov", d).kind == "sgd-nesterov"
    with pytest.raises(ConfigError):
        engine.make_optimizer("lamb", d)
    th = torch.from_numpy(th0.copy()).to(cuda)
    tb = torch.empty(d, dtype=torch.bfloat16, device=cuda)
    want, m, v = th0.copy(), np.zeros(d, npdt), np.zeros(d, npdt)
    for t in (1, 2, 3):
        g = rng.standard_normal(d).astype(npdt)
        opt.update(th, torch.from_numpy(g).to(cuda), 0.01, theta_bf16=tb)
        want, m, v = O.adam_update(want, m, v, g, 0.01, t)
    bits = np.uint64 if dtype == torch.float64 else np.uint32
    assert opt.t == 3
    assert np.array_equal(th.cpu().numpy().view(bits), want.view(bits))
    assert np.array_equal(opt.m.cpu().numpy().view(bits), m.view(bits))
    assert np.array_equal(opt.v.cpu().numpy().view(bits), v.view(bits))
    if dtype == torch.float32:  # (a float64 theta rounds to bf16 directly)
        assert np.array_equal(tb.view(torch.int16).cpu().numpy().view(np.uint16), O.bf16_rne(want))
    g = rng.standard_normal(d).astype(npdt)
    g[7] = np.inf
    before = th.clone()
    with pytest.raises(NumericalError):
        opt.update(th, torch.from_numpy(g).to(cuda), 0.01)
    assert opt.t == 3 and torch.equal(th, before)


@pytest.mark.parametrize("n,p", [(2, 1), (4, 2), (8, 3), (8, 8), (16, 5), (33, 7), (64, 20)])
def test_mask_widths_and_partial_tiles(cuda, n, p):
    """uint8/16/32/64 owner masks; d not a multiple of the tile or of 4."""
    engine, masking = _pkg()
    from paper_2507_09029_b200 import zoo
    topo = zoo.residual_mlp_topology(width=37, blocks=max(n, 4), classes=3, in_dim=5)
    for strategy in ("block", "neuron"):
        a = masking.build_assignment(topo, strategy, n, p, seed=n * 100 + p)
        reps = _replicas(a, torch.float32, 7, cuda)
        masks = a.param_masks.cpu().numpy()
        want = O.aggregate_f32_ordered([r.cpu().numpy() for r in reps], masks)
        got = engine.aggregate(reps, a).gbar.cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (strategy, n, p)
        # the tiled kernel explicitly (small buffers default to SDP_SYNC_DIRECT at N <= 8)
        out = torch.empty(topo.total, device=cuda)
        engine.owner_sync(reps, a, out=out, writeback=False, plan=engine.SyncPlan(a, direct=False))
        assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32)), (strategy, n, p)


@pytest.mark.slow
def test_resnet18_and_gpt2_full_size_properties(cuda):
    """Full C2/C4 sizes: replicas bit-identical after writeback, mean of an
    all-equal input is that input, and linearity sync(a*x) == a*sync(x) for a=2."""
    engine, masking = _pkg()
    from paper_2507_09029_b200 import zoo
    for topo in (zoo.resnet18_cifar_topology(), zoo.gpt2_small_topology()):
        a = masking.build_assignment(topo, "block", 8, 4, seed=1)
        reps = _replicas(a, torch.float32, 11, cuda)
        doubled = [r * 2 for r in reps]
        out1 = torch.empty(topo.total, device=cuda)
        out2 = torch.empty(topo.total, device=cuda)
        engine.owner_sync(reps, a, out=out1)
        engine.owner_sync(doubled, a, out=out2)
        assert torch.equal(out2, out1 * 2)  # exact: scaling by 2 commutes with RN
        pm = a.param_masks
        for w in range(8):
            assert torch.equal(reps[w][pm[w]], out1[pm[w]])
        # identical inputs on every owner -> mean equals the input (values chosen so
        # every partial sum k*x is exact in fp32: small integers / 8)
        x = torch.randint(-1000, 1000, (topo.total,), device=cuda).float() / 8
        same = [x * pm[w] for w in range(8)]
        out3 = torch.empty_like(x)
        engine.owner_sync(same, a, out=out3, writeback=False)
        assert torch.equal(out3, x)
        del reps, doubled, same
        torch.cuda.empty_cache()


@pytest.mark.parametrize("strategy", ["block", "neuron"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_direct_small_buffer_kernel_equals_tiled(cuda, strategy, dtype):
    """SDP_SYNC_DIRECT (one round trip: masks + all N replicas loaded at once)
    == the tiled kernel bit for bit -- mean, bf16 mean, every owner's
    write-back and bf16 shadow, the fused Nesterov epilogue and the status
    word -- on sizes with a ragged tail (d not a multiple of the vector)."""
    engine, masking = _pkg()
    from paper_2507_09029_b200 import zoo
    for topo in (zoo.mini_resnet_topology(26, 8, 10, 2, 3, (8, 8)),
                 zoo.residual_mlp_topology(width=37, blocks=8, classes=3, in_dim=5)):
        a = masking.build_assignment(topo, strategy, 8, 3, seed=11)
        d = topo.total
        pm = a.param_masks
        gen = torch.Generator(device=cuda)
        gen.manual_seed(d)
        base = [(torch.randn(d, generator=gen, device=cuda) * pm[w]).to(dtype) for w in range(8)]
        th0 = torch.randn(d, generator=gen, device=cuda).to(dtype)
        res = {}
        for direct in (False, True):
            plan = engine.SyncPlan(a, direct=direct)
            assert plan.direct == direct
            reps = [b.clone() for b in base]
            sh = [torch.zeros(d, dtype=torch.bfloat16, device=cuda) for _ in reps]
            out = torch.empty(d, dtype=dtype, device=cuda)
            outb = torch.empty(d, dtype=torch.bfloat16, device=cuda)
            th, v = th0.clone(), torch.zeros_like(th0)
            tb = torch.empty(d, dtype=torch.bfloat16, device=cuda)
            status = torch.zeros(1, dtype=torch.int32, device=cuda)
            engine.PreparedSync(reps, a, writeback=True, shadows_bf16=sh, out=out, out_bf16=outb, plan=plan,
                                check_finite=True, check_uncovered=True, status=status,
                                nesterov={"theta": th, "velocity": v, "lr": 0.1, "momentum": 0.9,
                                          "theta_bf16": tb}).launch()
            res[direct] = [out, outb.view(torch.int16), th, v, tb.view(torch.int16), status] + reps + \
                [x.view(torch.int16) for x in sh]
        for x, y in zip(res[False], res[True]):
            assert torch.equal(x, y)
        assert int(res[True][5].item()) == 0
    # the leak check fires the same way
    reps = [b.clone() for b in base]
    unc = torch.nonzero(pm.sum(0) == 0)
    if len(unc):
        reps[3][int(unc[0])] = float("inf")
        st = torch.zeros(1, dtype=torch.int32, device=cuda)
        engine.PreparedSync(reps, a, writeback=False, out=torch.empty_like(reps[0]), check_uncovered=True,
                            status=st, plan=engine.SyncPlan(a, direct=True)).launch()
        assert int(st.item()) & 0x1


@pytest.mark.parametrize("strategy", ["block", "neuron"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_stream_kernel_equals_tiled(cuda, strategy, dtype):
    """SDP_SYNC_STREAM (grid-stride, owner-filtered loads, prefetched masks)
    == the tiled kernel bit for bit: mean, write-back, shadows, fused Nesterov."""
    engine, masking = _pkg()
    from paper_2507_09029_b200 import zoo
    for topo in (zoo.resnet18_cifar_topology(), zoo.residual_mlp_topology(width=37, blocks=8, classes=3, in_dim=5)):
        a = masking.build_assignment(topo, strategy, 8, 3, seed=5)
        d = topo.total
        pm = a.param_masks
        gen = torch.Generator(device=cuda)
        gen.manual_seed(d + 1)
        base = [(torch.randn(d, generator=gen, device=cuda) * pm[w]).to(dtype) for w in range(8)]
        th0 = torch.randn(d, generator=gen, device=cuda).to(dtype)
        res = {}
        for stream in (False, True):
            plan = engine.SyncPlan(a, direct=stream, stream=stream)
            assert plan.stream == stream
            reps = [b.clone() for b in base]
            sh = [torch.zeros(d, dtype=torch.bfloat16, device=cuda) for _ in reps]
            out = torch.empty(d, dtype=dtype, device=cuda)
            th, v = th0.clone(), torch.zeros_like(th0)
            st = torch.zeros(1, dtype=torch.int32, device=cuda)
            engine.PreparedSync(reps, a, writeback=True, shadows_bf16=sh, out=out, plan=plan, check_finite=True,
                                check_uncovered=True, status=st,
                                nesterov={"theta": th, "velocity": v, "lr": 0.1, "momentum": 0.9}).launch()
            res[stream] = [out, th, v, st] + reps + [x.view(torch.int16) for x in sh]
        for x, y in zip(res[False], res[True]):
            assert torch.equal(x, y)
        unc = torch.nonzero(pm.sum(0) == 0)
        if len(unc):  # the leak check fires on the streaming path too
            reps = [b.clone() for b in base]
            reps[6][int(unc[-1])] = float("nan")
            st = torch.zeros(1, dtype=torch.int32, device=cuda)
            engine.PreparedSync(reps, a, writeback=False, out=torch.empty_like(reps[0]), check_uncovered=True,
                                status=st, plan=engine.SyncPlan(a, direct=True, stream=True)).launch()
            assert int(st.item()) & 0x1


@pytest.mark.parametrize("strategy", ["block", "neuron"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_stream_kernel_mean_only_equals_tiled(cuda, strategy, dtype):
    """The mean-only instantiation of SDP_SYNC_STREAM (what the drop-in
    `aggregate` runs on width-wise flat plans: whole-vector stores of the
    per-element means, owners skipped warp-uniformly) == the tiled kernel bit
    for bit -- mean, bf16 mean, status -- replicas untouched; and the routed
    default plan picks it for a mixed-tile neuron plan."""
    engine, masking = _pkg()
    from paper_2507_09029_b200 import zoo
    for topo in (zoo.resnet18_cifar_topology(), zoo.residual_mlp_topology(width=37, blocks=8, classes=3, in_dim=5)):
        a = masking.build_assignment(topo, strategy, 8, 4, seed=3)
        d = topo.total
        pm = a.param_masks
        gen = torch.Generator(device=cuda)
        gen.manual_seed(d + 7)
        base = [(torch.randn(d, generator=gen, device=cuda) * pm[w]).to(dtype) for w in range(8)]
        res = {}
        for stream in (False, True):
            plan = engine.SyncPlan(a, direct=stream, stream=stream)
            reps = [b.clone() for b in base]
            out = torch.empty(d, dtype=dtype, device=cuda)
            outb = torch.empty(d, dtype=torch.bfloat16, device=cuda)
            st = torch.zeros(1, dtype=torch.int32, device=cuda)
            engine.PreparedSync(reps, a, writeback=False, out=out, out_bf16=outb, plan=plan, check_finite=True,
                                check_uncovered=True, status=st).launch()
            for r, b in zip(reps, base):
                assert torch.equal(r, b)
            res[stream] = [out, outb.view(torch.int16), st]
        for x, y in zip(res[False], res[True]):
            assert torch.equal(x, y)
        assert int(res[True][2].item()) == 0
        if strategy == "neuron" and topo.total > 1 << 20:
            assert a.sync_plan().stream_mean
            g = engine.aggregate(base, a).gbar
            assert torch.equal(g, res[False][0])


@pytest.mark.parametrize("d_extra", [0, 1, 3])
def test_stream_mean_writes_stay_in_bounds(cuda, d_extra):
    """Guard bands (compute-sanitizer is not available on the GPU pool): the
    mean-only streaming kernel writes `out` / `out_bf16` inside [0, d) only,
    on vectors with a ragged tail, and never touches the replicas."""
    engine, masking = _pkg()
    from paper_2507_09029_b200 import zoo
    topo = zoo.residual_mlp_topology(width=64 + d_extra, blocks=8, classes=3, in_dim=5)
    a = masking.build_assignment(topo, "neuron", 8, 4, seed=13)
    d = topo.total
    pm = a.param_masks
    gen = torch.Generator(device=cuda)
    gen.manual_seed(17)
    reps = [torch.randn(d, generator=gen, device=cuda) * pm[w] for w in range(8)]
    keep = [r.clone() for r in reps]
    guard = 1024
    big = torch.full((d + guard,), 7.0, device=cuda)
    bigb = torch.full((d + guard,), 7.0, device=cuda).to(torch.bfloat16)
    out, outb = big[:d], bigb[:d]
    plan = engine.SyncPlan(a, direct=True, stream=True)
    engine.PreparedSync(reps, a, writeback=False, out=out, out_bf16=outb, plan=plan).launch()
    torch.cuda.synchronize()
    assert torch.all(big[d:] == 7.0) and torch.all(bigb[d:] == 7.0)
    for r, k in zip(reps, keep):
        assert torch.equal(r, k)
    want = torch.empty(d, device=cuda)
    engine.PreparedSync(reps, a, writeback=False, out=want, plan=engine.SyncPlan(a, direct=False, stream=False)).launch()
    assert torch.equal(out, want)
