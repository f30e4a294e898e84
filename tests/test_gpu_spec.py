"""SPEC.md acceptance criteria that concern the hot path.

  #1 DP-equivalence: at P = N the owner sync is the plain mean in worker order
     and, fused with SGD-Nesterov, reproduces the single-loop synchronous-DP
     trajectory (oracles.dp_reference_trajectory's update, oracles.py:112-143)
     -- here bit for bit over 100 steps in float64;
  #3 aggregation oracle: random mask / gradient instances equal the
     per-parameter brute-force loop (oracles.aggregate_loops, oracles.py:65-77)
     bit for bit;
  #10 memory accounting: a fully maskable model's active fraction is P/N.
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _aggregate_loops(grads, masks):
    """Per-parameter loop restatement of engine.aggregate (oracles.py:65-77)."""
    n, d = masks.shape
    out = np.zeros(d)
    for j in range(d):
        num, cnt = 0.0, 0
        for i in range(n):
            num += masks[i, j] * grads[i][j]
            cnt += int(masks[i, j])
        out[j] = num / max(cnt, 1)
    return out


def test_dp_equivalence_trajectory(cuda):
    """#1: N = P = 8, 100 steps, mini-ResNet d: fused sync + Nesterov (float64)
    == gbar = (sum in worker order) / N; v = mu v + gbar; th -= lr (gbar + mu v)."""
    from paper_2507_09029_b200 import engine, masking, zoo
    topo = zoo.mini_resnet_topology(26, 8, 10, 2, 3, (32, 32))
    a = masking.build_assignment(topo, "block", 8, 8, seed=1)
    assert a.dp_equivalent
    d = topo.total
    rng = np.random.default_rng(11)
    th_ref = rng.standard_normal(d)
    v_ref = np.zeros(d)
    theta = torch.from_numpy(th_ref.copy()).to(cuda)
    vel = torch.zeros(d, dtype=torch.float64, device=cuda)
    reps = [torch.empty(d, dtype=torch.float64, device=cuda) for _ in range(8)]
    for t in range(100):
        lr = 0.05 * 0.5 * (1 + np.cos(np.pi * t / 100))  # cosine schedule
        grads = [rng.standard_normal(d) * 0.1 for _ in range(8)]
        for r, g in zip(reps, grads):
            r.copy_(torch.from_numpy(g))
        engine.owner_sync(reps, a, writeback=False,
                          nesterov={"theta": theta, "velocity": vel, "lr": lr, "momentum": 0.9})
        total = np.zeros(d)
        for g in grads:
            total += g
        gbar = total / 8
        v_ref = 0.9 * v_ref + gbar
        th_ref = th_ref - lr * (gbar + 0.9 * v_ref)
    got = theta.cpu().numpy()
    assert np.max(np.abs(got - th_ref)) < 1e-6  # the SPEC bound ...
    assert np.array_equal(got.view(np.uint64), th_ref.view(np.uint64))  # ... and in fact bit-exact


def test_aggregate_random_instances_vs_loop_oracle(cuda):
    """#3: 300 random (N, d, mask density) instances with arbitrary masks."""
    from paper_2507_09029_b200 import engine, masking, zoo
    rng = np.random.default_rng(3)
    for inst in range(300):
        n = int(rng.integers(1, 10))
        width = int(rng.integers(1, 6))
        topo = zoo.residual_mlp_topology(width=width, blocks=2, classes=2, in_dim=3)
        d = topo.total
        masks = rng.random((n, d)) < rng.uniform(0.0, 1.0)
        grads = [rng.standard_normal(d) * masks[i] for i in range(n)]
        a = masking.MaskAssignment(n, 1, "block", 0, topo, {}, masks, torch.zeros(d, dtype=torch.int64))
        reps = [torch.from_numpy(g).to(cuda) for g in grads]
        got = engine.aggregate(reps, a).gbar.cpu().numpy()
        want = _aggregate_loops(grads, masks)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), inst
        # both kernels: the small-buffer one (the default here) and the tiled one
        out = torch.empty(d, dtype=torch.float64, device=cuda)
        engine.owner_sync(reps, a, out=out, writeback=False,
                          plan=engine.SyncPlan(a, direct=not a.sync_plan().direct))
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want.view(np.uint64)), inst
        if inst % 50 == 0:  # the vectorised oracle agrees too
            assert np.array_equal(want, O.aggregate_f64(grads, masks, np.maximum(masks.sum(0), 1).astype(np.float64)))


@pytest.mark.parametrize("n,p", [(8, 4), (8, 5), (6, 2)])
def test_active_fraction_fully_maskable(cuda, n, p):
    """#10: every parameter of the residual MLP except the stem/head sits in a
    maskable block; the active fraction of those is exactly P/N."""
    from paper_2507_09029_b200 import masking, zoo
    topo = zoo.residual_mlp_topology(width=16, blocks=n, classes=4, in_dim=8)
    a = masking.build_assignment(topo, "block", n, p, seed=2)
    gov = a.governors.cpu().numpy()
    pm = a.param_masks.cpu().numpy()
    maskable = gov > 0
    frac = pm[:, maskable].sum() / (n * maskable.sum())
    assert frac == p / n
