"""Pin the CPU oracle against the reference's own outputs (golden vectors)."""

import numpy as np
import pytest

import _golden as G
from oracle import oracle as O


def test_permutations_match_numpy_reference():
    p = G.permutations()
    off = 0
    for seed, n in zip(G.seeds(), p["n"]):
        n = int(n)
        assert np.array_equal(O.permutation(seed, n), p["values"][off:off + n]), (seed, n)
        off += n


def test_sequential_permutations_share_one_generator():
    p = G.permutations()
    g = O.Pcg64(int(p["seq_seed"][0]))
    off = 0
    for n in p["seq_sizes"]:
        assert np.array_equal(g.permutation(int(n)), p["seq_values"][off:off + int(n)])
        off += int(n)


@pytest.mark.parametrize("case", G.cases(), ids=lambda c: f"{c['model']}-{c['strategy']}-N{c['n']}P{c['p']}s{c['seed']}")
def test_oracle_assignment_matches_reference(case):
    topo = G.topology(case["model"])
    a = O.build_assignment(topo, case["strategy"], case["n"], case["p"], case["seed"])
    assert np.array_equal(a.param_masks, G.case_masks(case))
    arr = G.arrays()
    assert np.array_equal(a.governors, arr[f"c{case['id']}_governors"].astype(np.int64))
    assert np.array_equal(a.coverage, arr[f"c{case['id']}_coverage"].astype(np.int64))
    assert a.unit_workers() == {k: tuple(v) for k, v in case["unit_workers"].items()}
    assert a.param_masks.sum(axis=1).tolist() == case["active_param_counts"]
    assert int((a.coverage == 0).sum()) == case["uncovered_params"]


@pytest.mark.parametrize("case", G.cases(with_grads=True), ids=lambda c: f"c{c['id']}")
def test_oracle_aggregate_bitexact_f64(case):
    masks = G.case_masks(case)
    grads, theta0, vel0 = G.case_inputs(case, masks)
    divisor = np.maximum(masks.sum(axis=0), 1).astype(np.float64)
    ref = G.arrays()[f"c{case['id']}_gbar"]
    assert np.array_equal(O.aggregate_f64(list(grads), masks, divisor).view(np.uint64), ref.view(np.uint64))
    # owners-only restatement (what the kernel does) is bit-identical too
    assert np.array_equal(O._aggregate_f64_owners(list(grads), masks).view(np.uint64), ref.view(np.uint64))
    th, v = O.nesterov_update(theta0, vel0, ref, 0.05, 0.9)
    assert np.array_equal(th.view(np.uint64), G.arrays()[f"c{case['id']}_theta1"].view(np.uint64))
    assert np.array_equal(v.view(np.uint64), G.arrays()[f"c{case['id']}_vel1"].view(np.uint64))
    # Adam (optim.py:90-109): two steps from theta1 with zero moments
    m = np.zeros_like(th)
    vv = np.zeros_like(th)
    th, m, vv = O.adam_update(th, m, vv, ref, 0.01, 1)
    th, m, vv = O.adam_update(th, m, vv, ref * 0.5, 0.01, 2)
    arr = G.arrays()
    assert np.array_equal(th.view(np.uint64), arr[f"c{case['id']}_adam_theta2"].view(np.uint64))
    assert np.array_equal(m.view(np.uint64), arr[f"c{case['id']}_adam_m2"].view(np.uint64))
    assert np.array_equal(vv.view(np.uint64), arr[f"c{case['id']}_adam_v2"].view(np.uint64))


def test_known_answer_disjoint_masks():
    ka = G.manifest()["known_answers"]["disjoint"]
    m = np.array(ka["m"], dtype=bool)
    g = np.array(ka["g"], dtype=np.float64)
    out = O.aggregate_f64(list(g), m, np.maximum(m.sum(0), 1).astype(np.float64))
    assert out.tolist() == ka["gbar"]


def test_f32_restatement_condition_scaled_error():
    """fp32 ordered sum vs f64 reference within 1e-6 * max(|r|, sum|g|/P)."""
    case = G.cases(with_grads=True)[0]
    masks = G.case_masks(case)
    grads, _, _ = G.case_inputs(case, masks)
    g32 = grads.astype(np.float32)
    ref = O.aggregate_f64(list(g32.astype(np.float64)), masks, np.maximum(masks.sum(0), 1).astype(np.float64))
    out = O.aggregate_f32_ordered(list(g32), masks)
    scale = np.maximum(np.abs(ref), np.abs(g32.astype(np.float64) * masks).sum(0) / np.maximum(masks.sum(0), 1))
    assert np.all(np.abs(out - ref) <= 1e-6 * np.maximum(scale, 1e-300))


def test_bf16_rne():
    x = np.array([1.0, 1.00390625, 1.005859375, -2.5, 0.0, -0.0, 3.4e38], dtype=np.float32)
    import torch
    want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(O.bf16_rne(x), want)
