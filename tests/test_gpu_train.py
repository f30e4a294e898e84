"""Training-step integration (engine.py:202-223) on ResNet-18 (configs[1])."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_resnet18_subnet_step_matches_oracle(cuda):
    from paper_2507_09029_b200 import masking, train
    model = train.build_resnet18(cuda, seed=3)
    a = masking.build_assignment(model.topology, "block", 8, 4, seed=1)
    tr = train.SubnetTrainer(model, a, lr=0.05, autocast=False)
    gen = torch.Generator(device=cuda)
    gen.manual_seed(0)
    batches = [(torch.randn(4, 3, 32, 32, generator=gen, device=cuda),
                torch.randint(0, 10, (4,), generator=gen, device=cuda)) for _ in range(8)]
    th0 = model.theta.cpu().numpy().copy()
    tr.step(batches)
    grads = [g.cpu().numpy() for g in tr.grads]
    masks = a.param_masks.cpu().numpy()
    for w in range(8):  # a worker's gradient is exactly zero outside its subnetwork
        assert np.all(grads[w][~masks[w]] == 0.0)
    gbar = O.aggregate_f32_ordered(grads, masks)
    th1, v1 = O.nesterov_update(th0, np.zeros_like(th0), gbar, 0.05, 0.9)
    assert np.array_equal(model.theta.cpu().numpy().view(np.uint32), th1.astype(np.float32).view(np.uint32))
    assert np.array_equal(tr.theta_bf16.view(torch.int16).cpu().numpy().view(np.uint16), O.bf16_rne(th1))


def test_resnet18_adam_steps_match_oracle_and_graph_replay(cuda):
    """optimizer="adam" (optim.py:101-109 fused into the sync, device step
    counter + bias table): three steps == aggregate + the Adam restatement
    (fp32, the reference's bias corrections), and the graphed trainer
    replays the same three steps bit for bit (the step advances inside the
    graph)."""
    from paper_2507_09029_b200 import masking, train
    gen = torch.Generator(device=cuda)
    gen.manual_seed(0)
    steps = [[(torch.randn(4, 3, 32, 32, generator=gen, device=cuda),
               torch.randint(0, 10, (4,), generator=gen, device=cuda)) for _ in range(8)] for _ in range(3)]
    model = train.build_resnet18(cuda, seed=3)
    a = masking.build_assignment(model.topology, "block", 8, 4, seed=1)
    tr = train.SubnetTrainer(model, a, lr=0.01, autocast=False, optimizer="adam")
    th = model.theta.cpu().numpy().copy()
    m, v = np.zeros_like(th), np.zeros_like(th)
    masks = a.param_masks.cpu().numpy()
    for t, b in enumerate(steps, start=1):
        tr.step(b)
        gbar = O.aggregate_f32_ordered([g.cpu().numpy() for g in tr.grads], masks)
        th, m, v = O.adam_update(th, m, v, gbar, 0.01, t)
    tr.check()
    assert int(tr.adam_step.item()) == 3
    assert np.array_equal(model.theta.cpu().numpy().view(np.uint32), th.view(np.uint32))
    assert np.array_equal(tr.second.cpu().numpy().view(np.uint32), v.view(np.uint32))
    prev = torch.backends.cudnn.deterministic
    torch.backends.cudnn.deterministic = True  # eager vs graphed: same conv algorithms
    try:
        out = []
        for graphed in (False, True):
            mm = train.build_resnet18(cuda, seed=3)
            gtr = train.SubnetTrainer(mm, a, lr=0.01, autocast=False, optimizer="adam", graphed=graphed)
            for b in steps:
                gtr.step(b)
            assert int(gtr.adam_step.item()) == 3
            out.append(mm.theta)
        assert torch.equal(out[0], out[1])
    finally:
        torch.backends.cudnn.deterministic = prev


def test_resnet18_width_wise_compact_equals_masked_full(cuda):
    """C3: gather -> compact ResNet-18 fwd/bwd (ragged GN) -> scatter equals the
    reference semantics (theta*mask through the full model, active-channel GN)."""
    import torch.nn.functional as F
    from paper_2507_09029_b200 import masking, models, train
    model = train.build_resnet18(cuda, seed=2)
    model.theta = model.theta.double()
    a = masking.build_assignment(model.topology, "neuron", 8, 4, seed=1)
    gen = torch.Generator(device=cuda)
    gen.manual_seed(3)
    x = torch.randn(2, 3, 32, 32, generator=gen, device=cuda, dtype=torch.float64)
    y = torch.randint(0, 10, (2,), generator=gen, device=cuda)
    for w in (0, 5):
        view = a.worker_view(w)
        leaf = models._extract(model.theta, view).requires_grad_(True)
        loss_f = F.cross_entropy(model.arch.forward(train.param_views(model.topology, leaf), x, view), y)
        (g_f,) = torch.autograd.grad(loss_f, leaf)
        sub = models.SubnetLayout(a, w)
        leaf_c = sub.gather(model.theta).requires_grad_(True)
        loss_c = F.cross_entropy(model.arch.forward_compact(sub.views(leaf_c), x, sub), y)
        (g_c,) = torch.autograd.grad(loss_c, leaf_c)
        g_c = sub.scatter(g_c)
        assert abs(loss_f.item() - loss_c.item()) <= 1e-12 * abs(loss_f.item())
        assert torch.max(torch.abs(g_f - g_c)).item() <= 1e-10 * max(1.0, torch.max(torch.abs(g_f)).item())
        assert torch.all(g_c[~view.param_mask_bool] == 0)


def test_resnet18_width_wise_step_matches_oracle(cuda):
    from paper_2507_09029_b200 import masking, train
    model = train.build_resnet18(cuda, seed=3)
    a = masking.build_assignment(model.topology, "neuron", 8, 4, seed=1)
    tr = train.SubnetTrainer(model, a, lr=0.05, autocast=False)
    assert tr.compact
    gen = torch.Generator(device=cuda)
    gen.manual_seed(0)
    batches = [(torch.randn(4, 3, 32, 32, generator=gen, device=cuda),
                torch.randint(0, 10, (4,), generator=gen, device=cuda)) for _ in range(8)]
    th0 = model.theta.cpu().numpy().copy()
    tr.step(batches)
    grads = [g.cpu().numpy() for g in tr.grads]
    masks = a.param_masks.cpu().numpy()
    gbar = O.aggregate_f32_ordered(grads, masks)
    th1, _ = O.nesterov_update(th0, np.zeros_like(th0), gbar, 0.05, 0.9)
    assert np.array_equal(model.theta.cpu().numpy().view(np.uint32), th1.astype(np.float32).view(np.uint32))


def test_gpt2_block_dropping_skip_equals_multiply(cuda):
    """C4: a dropped GPT-2 block is the identity (skip == multiply-by-zero)
    and leaves exactly-zero gradients on its parameters."""
    from paper_2507_09029_b200 import masking, train
    model = train.build_gpt2(cuda)
    model.theta = model.theta.double()
    a = masking.build_assignment(model.topology, "block", 8, 4, seed=1)
    view = a.worker_view(3)
    tok = torch.randint(0, 50257, (2, 64), device=cuda)
    losses, grads = [], []
    for mode in ("skip", "multiply"):
        leaf = model.theta.detach().clone().requires_grad_(True)
        loss = train.lm_loss(model.arch.forward(train.param_views(model.topology, leaf), tok, view, mode), tok)
        (g,) = torch.autograd.grad(loss, leaf)
        losses.append(loss.item())
        grads.append(g)
    assert abs(losses[0] - losses[1]) <= 1e-12 * abs(losses[0])
    mask = view.param_mask_bool
    assert torch.all(grads[0][~mask] == 0) and torch.all(grads[1][~mask] == 0)
    assert torch.max(torch.abs(grads[0] - grads[1])).item() < 1e-12


def test_memory_subnet_below_full_replica(cuda):
    from paper_2507_09029_b200 import masking, train
    model = train.build_resnet18(cuda)
    a = masking.build_assignment(model.topology, "block", 8, 4, seed=1)
    sub = train.worker_memory(model, a, 0, 64, cuda)
    full = train.worker_memory(model, a, None, 64, cuda)
    assert sub["active_params"] == a.worker_view(0).active_params
    assert full["active_params"] == model.topology.total
    assert sub["peak_bytes"] < full["peak_bytes"]


@pytest.mark.parametrize("strategy", ["block", "neuron"])
def test_memory_step_gradient_is_the_worker_gradient(cuda, strategy):
    """worker_memory's hooked per-parameter backward produces the same compact
    gradient as autograd on the gathered compact leaf."""
    import torch.nn.functional as F
    from paper_2507_09029_b200 import masking, models, train
    model = train.build_resnet18(cuda, seed=6)
    a = masking.build_assignment(model.topology, strategy, 8, 4, seed=1)
    gen = torch.Generator(device=cuda)
    gen.manual_seed(2)
    x = torch.randn(8, 3, 32, 32, generator=gen, device=cuda)
    y = torch.randint(0, 10, (8,), generator=gen, device=cuda)
    got = train.worker_memory(model, a, 3, 8, cuda, make_batch=lambda: (x, y), return_grad=True)["grad"]
    sub = models.SubnetLayout(a, 3)
    leaf = sub.gather(model.theta).to(torch.bfloat16)  # workers train on the bf16 copy
    leaf.requires_grad_(True)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        if strategy == "neuron":
            logits = model.arch.forward_compact(sub.views(leaf), x, sub)
        else:
            logits = model.arch.forward(sub.views(leaf), x, a.worker_view(3))
        loss = F.cross_entropy(logits.float(), y)
    (want,) = torch.autograd.grad(loss, leaf)
    assert torch.allclose(got, want.float(), rtol=1e-5, atol=1e-7)


@pytest.mark.parametrize("strategy", ["block", "neuron"])
def test_graphed_step_equals_eager(cuda, strategy):
    """The CUDA-graph step (train.SubnetTrainer(graphed=True)) replays exactly
    the eager step: same theta after three steps (deterministic cuDNN, fp32),
    and the capture's warm-up steps leave no trace."""
    from paper_2507_09029_b200 import masking, train
    prev = torch.backends.cudnn.deterministic
    torch.backends.cudnn.deterministic = True
    try:
        gen = torch.Generator(device=cuda)
        gen.manual_seed(4)
        steps = [[(torch.randn(4, 3, 32, 32, generator=gen, device=cuda),
                   torch.randint(0, 10, (4,), generator=gen, device=cuda)) for _ in range(8)]
                 for _ in range(3)]
        out = []
        for graphed in (False, True):
            model = train.build_resnet18(cuda, seed=5)
            a = masking.build_assignment(model.topology, strategy, 8, 4, seed=1)
            tr = train.SubnetTrainer(model, a, lr=0.05, autocast=False, graphed=graphed,
                                     sync_layout=strategy == "neuron")
            losses = [float(tr.step(b).item()) for b in steps]
            out.append((tr.theta().cpu().numpy(), losses))
        assert out[0][1] == out[1][1]
        assert np.array_equal(out[0][0].view(np.uint32), out[1][0].view(np.uint32))
    finally:
        torch.backends.cudnn.deterministic = prev


def test_fused_lm_head_cross_entropy_matches_unfused(cuda):
    """train.lm_loss on the tied head (chunked, logits never whole) == the
    unfused F.cross_entropy over materialised logits: float64 to 1e-12, and
    under bf16 autocast to bf16 rounding."""
    from paper_2507_09029_b200 import train
    gen = torch.Generator(device=cuda)
    gen.manual_seed(1)
    tok = torch.randint(0, 50257, (3, 1500), generator=gen, device=cuda)  # 4497 rows: 3 chunks
    for dtype, autocast, tol in ((torch.float64, False, 1e-12), (torch.float32, True, 2e-2)):
        h = (torch.randn(3, 1500, 64, generator=gen, device=cuda) * 0.5).to(dtype).requires_grad_(True)
        w = (torch.randn(50257, 64, generator=gen, device=cuda) * 0.05).to(dtype).requires_grad_(True)
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=autocast):
            fused = train.lm_loss(train.LMHead(h, w), tok)
            plain = train.lm_loss(train.LMHead(h, w).logits(), tok)
        gf = torch.autograd.grad(fused, (h, w))
        gp = torch.autograd.grad(plain, (h, w))
        assert abs(fused.item() - plain.item()) <= tol * abs(plain.item())
        for a, b in zip(gf, gp):
            assert torch.allclose(a.double(), b.double(), rtol=tol, atol=tol * b.abs().max().item())


@pytest.mark.parametrize("rows,cols", [(8192, 768), (5, 768), (300, 256), (1000, 512), (77, 1024)])
def test_layer_norm_bf16_matches_fp32_reference(cuda, rows, cols):
    """libsdp k_ln_fwd / k_ln_bwd (train._LayerNormBF16) against torch fp32
    layer_norm of the same bf16 inputs: y and dx within bf16 rounding of the
    fp32 result, dgamma / dbeta (sums over the rows) to 1e-2 relative; the
    backward is deterministic (same bits on a second call)."""
    import torch.nn.functional as F
    from paper_2507_09029_b200 import train
    g = torch.Generator(device=cuda)
    g.manual_seed(rows + cols)
    x = (torch.randn(rows, cols, generator=g, device=cuda) * 2 + 0.5).bfloat16()
    w = (1 + 0.1 * torch.randn(cols, generator=g, device=cuda)).bfloat16()
    b = (0.1 * torch.randn(cols, generator=g, device=cuda)).bfloat16()
    dy = torch.randn(rows, cols, generator=g, device=cuda).bfloat16()
    xs, ws, bs = (t.clone().requires_grad_(True) for t in (x, w, b))
    y = train._LayerNormBF16.apply(xs, ws, bs, 1e-5)
    y.backward(dy)
    xr, wr, br = (t.float().requires_grad_(True) for t in (x, w, b))
    yr = F.layer_norm(xr, (cols,), wr, br, 1e-5)
    yr.backward(dy.float())
    assert y.dtype == torch.bfloat16 and xs.grad.dtype == torch.bfloat16
    tol = lambda r: 2 ** -7 * r.abs() + 1e-3  # noqa: E731  (one bf16 ulp of the fp32 value + slack)
    assert (y.float() - yr).abs().le(tol(yr)).all()
    assert (xs.grad.float() - xr.grad).abs().le(tol(xr.grad) + 1e-2 * xr.grad.abs().max()).all()
    for got, ref in ((ws.grad, wr.grad), (bs.grad, br.grad)):
        assert (got.float() - ref).abs().max() <= 1e-2 * ref.abs().max() + 1e-3
    xs2, ws2, bs2 = (t.clone().requires_grad_(True) for t in (x, w, b))
    train._LayerNormBF16.apply(xs2, ws2, bs2, 1e-5).backward(dy)
    assert torch.equal(xs2.grad, xs.grad) and torch.equal(ws2.grad, ws.grad) and torch.equal(bs2.grad, bs.grad)


@pytest.mark.parametrize("layout", ["bhtd", "bthd"])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_split_heads_backward_merges_bit_exact(cuda, dtype, layout):
    """train._SplitHeads: forward views equal the permute of qkv; backward
    (libsdp k_merge_heads) equals autograd's gradient of the plain
    view/permute bit for bit (a pure data movement)."""
    from paper_2507_09029_b200 import train
    b, t, nh, hd = 2, 37, 3, 64
    g = torch.Generator(device=cuda)
    g.manual_seed(3)
    qkv = torch.randn(b * t, 3 * nh * hd, generator=g, device=cuda).to(dtype)
    grads = [torch.randn(b, nh, t, hd, generator=g, device=cuda).to(dtype) for _ in range(3)]
    if layout == "bthd":  # the SDPA backward's [b, t, nh, hd]-major gradients
        grads = [x.transpose(1, 2).contiguous().transpose(1, 2) for x in grads]
    a = qkv.clone().requires_grad_(True)
    outs = train._SplitHeads.apply(a, b, t, nh, hd)
    r = qkv.clone().requires_grad_(True)
    refs = r.view(b, t, 3, nh, hd).permute(2, 0, 3, 1, 4)
    for o, ref in zip(outs, refs):
        assert torch.equal(o, ref)
    torch.autograd.backward(outs, grads)
    torch.autograd.backward(list(refs), grads)
    assert torch.equal(a.grad, r.grad)


def test_store_grads_bf16_channels_last_matches_slot_copy(cuda):
    """SubnetTrainer._store_grads: bf16 gradients (conv weights channels-last,
    as cuDNN's NHWC kernels return them) land in the fp32 replica exactly as
    a per-parameter g.float() copy into the reference-layout slots would put
    them (libsdp k_conv_grad_oihw + per-run casts); dropped parameters keep
    their zeros."""
    from paper_2507_09029_b200 import masking, train
    model = train.build_resnet18(cuda)
    a = masking.build_assignment(model.topology, "block", 8, 4, seed=1)
    tr = train.SubnetTrainer(model, a, lr=0.02)
    g = torch.Generator(device=cuda)
    g.manual_seed(11)
    for w in (0, 5):
        names = tr._live_params(w)
        spec = {p.name: p for p in model.topology.params}
        gs = []
        for k in names:
            t = torch.randn(spec[k].shape, generator=g, device=cuda).bfloat16()
            if t.dim() == 4:
                t = t.contiguous(memory_format=torch.channels_last)
            gs.append(t)
        tr.grads[w].zero_()
        tr._store_grads(w, names, gs)
        want = torch.zeros_like(tr.grads[w])
        slots = train.param_views(model.topology, want)
        for k, t in zip(names, gs):
            slots[k].copy_(t.float())
        assert torch.equal(tr.grads[w], want), w


def test_widthwise_bf16_per_parameter_leaves_match_single_leaf(cuda):
    """The width-wise bf16 step's per-parameter compact leaves (channels-last
    conv weights, fused gradient store + k_conv_grad_oihw) give the worker's
    fp32 sync-space gradient bit for bit as the single compact leaf whose
    gradient is one concatenation (deterministic cuDNN)."""
    from paper_2507_09029_b200 import masking, train
    prev = torch.backends.cudnn.deterministic
    torch.backends.cudnn.deterministic = True
    try:
        model = train.build_resnet18(cuda, seed=3)
        a = masking.build_assignment(model.topology, "neuron", 8, 4, seed=1)
        tr = train.SubnetTrainer(model, a, lr=0.02, sync_layout=True)
        g = torch.Generator(device=cuda)
        g.manual_seed(5)
        x = torch.randn(16, 3, 32, 32, generator=g, device=cuda)
        y = torch.randint(0, 10, (16,), generator=g, device=cuda)
        for w in (0, 3):
            tr.grads[w].zero_()
            tr._compact_step_bf16(w, x, y, cache=True)
            got = tr.grads[w].clone()
            sub = tr.subs[w]
            leaf = tr.transfers[w].to_compact(tr.theta_bf16).requires_grad_(True)
            with torch.autocast("cuda", dtype=torch.bfloat16):
                loss = tr.loss_fn(model.arch.forward_compact(sub.views(leaf), x, sub), y)
            (gl,) = torch.autograd.grad(loss, leaf)
            want = torch.zeros_like(tr.grads[w])
            tr.transfers[w].from_compact(gl.float(), want)
            assert torch.equal(got, want), (w, (got - want).abs().max().item())
    finally:
        torch.backends.cudnn.deterministic = prev


@pytest.mark.parametrize("rows,cols", [(8192, 768), (8192, 3072), (100, 2304), (3, 64)])
def test_col_sum_bf16_matches_fp32_sum(cuda, rows, cols):
    """libsdp column sums (the GPT-2 bias gradients) vs an fp64 sum of the
    same bf16 values: within bf16 rounding of the exact sum; deterministic."""
    import ctypes as C
    from paper_2507_09029_b200 import _native as N
    from paper_2507_09029_b200._device import ptr, stream_ptr
    g = torch.Generator(device=cuda)
    g.manual_seed(rows + cols)
    x = torch.randn(rows, cols, generator=g, device=cuda).bfloat16()
    parts = N.lib().sdp_col_sum_parts()

    def run():
        out = torch.empty(cols, dtype=torch.bfloat16, device=cuda)
        scratch = torch.empty(cols * parts, dtype=torch.float32, device=cuda)
        N.call("sdp_col_sum_bf16", ptr(x), rows, cols, ptr(out), ptr(scratch), stream_ptr(cuda))
        return out

    a, b = run(), run()
    assert torch.equal(a, b)
    ref = x.double().sum(0)
    assert (a.double() - ref).abs().le(2 ** -7 * ref.abs() + 1e-3 * rows ** 0.5).all()


def test_add_layer_norm_bf16_fused_matches_unfused(cuda):
    """train._AddLayerNormBF16 (libsdp residual-fused LayerNorm): the sum and
    the normalised rows equal the unfused bf16 add + LayerNorm kernels bit for
    bit; the gradients (dx with the residual branch's gradient folded in)
    agree with the unfused autograd to bf16 rounding."""
    from paper_2507_09029_b200 import train
    rows, cols = 4096, 768
    g = torch.Generator(device=cuda)
    g.manual_seed(9)
    a = torch.randn(rows, cols, generator=g, device=cuda).bfloat16()
    b = torch.randn(rows, cols, generator=g, device=cuda).bfloat16()
    w = (1 + 0.1 * torch.randn(cols, generator=g, device=cuda)).bfloat16()
    bias = (0.1 * torch.randn(cols, generator=g, device=cuda)).bfloat16()
    ds = torch.randn(rows, cols, generator=g, device=cuda).bfloat16()
    dy = torch.randn(rows, cols, generator=g, device=cuda).bfloat16()
    fa, fb, fw, fbias = (t.clone().requires_grad_(True) for t in (a, b, w, bias))
    s, y = train._AddLayerNormBF16.apply(fa, fb, fw, fbias, 1e-5)
    torch.autograd.backward([s, y], [ds, dy])
    ua, ub, uw, ubias = (t.clone().requires_grad_(True) for t in (a, b, w, bias))
    us = ua + ub
    uy = train._LayerNormBF16.apply(us, uw, ubias, 1e-5)
    torch.autograd.backward([us, uy], [ds, dy])
    assert torch.equal(s, us) and torch.equal(y, uy)
    for got, want in ((fa.grad, ua.grad), (fb.grad, ub.grad)):
        assert (got.float() - want.float()).abs().le(2 ** -7 * want.float().abs() + 2e-2).all()
    assert torch.equal(fw.grad, uw.grad) and torch.equal(fbias.grad, ubias.grad)
