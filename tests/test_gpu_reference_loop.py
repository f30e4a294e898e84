"""The drop-in inside the reference's OWN training loop.

`subnetdp.engine.run` (engine.py:152-245, staged unmodified in oracle/_ref by
oracle/build_ref.py) is run twice on the same config: once as shipped, once
with its two hot-path calls swapped for this package's --
  engine.aggregate        -> paper_2507_09029_b200.engine.aggregate (k_owner_sync)
  engine.build_assignment -> masking.build_assignment (k_assign + k_build_masks),
                             handed back as the reference's MaskAssignment
                             (masking.to_reference)
-- and every theta bit, every metrics row and the saved masks.json must agree.
The runs happen in a subprocess whose sys.path holds the staged reference, so
this package's exceptions subclass the reference's (errors.py) and the
reference's own `except` clauses catch them.
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r'''
import json, sys, tempfile
import numpy as np
import subnetdp as S
from subnetdp import engine as E, config as C, errors as RE, masking as RM
from paper_2507_09029_b200 import engine as OE, masking as OM, errors as OERR

out = {}
for strategy in ("block", "neuron"):
    cfg = C.ExperimentConfig(
        model=C.ModelConfig(kind="mini_resnet", channels=8, blocks=3, classes=4, norm_groups=2,
                            in_channels=3, image_hw=(8, 8)),
        dataset=C.DatasetConfig(kind="synthetic-blobs", train_size=96, test_size=32, classes=4,
                                channels=3, height=8, width=8, seed=7),
        n=4, p=2, strategy=strategy, batch_per_worker=4, e_full=1, seed=3, threads=1, max_steps=4)
    orig_agg, orig_build = E.aggregate, E.build_assignment
    with tempfile.TemporaryDirectory() as d1, tempfile.TemporaryDirectory() as d2:
        ref = E.run(cfg, d1)
        calls = {"agg": 0, "build": 0}

        def agg(grads, assignment):
            calls["agg"] += 1
            return OE.aggregate(grads, assignment)

        def build(topology, strategy_, n, p, seed):
            calls["build"] += 1
            return OM.to_reference(OM.build_assignment(topology, strategy_, n, p, seed), topology)

        E.aggregate, E.build_assignment = agg, build
        try:
            ours = E.run(cfg, d2)
        finally:
            E.aggregate, E.build_assignment = orig_agg, orig_build
        masks_equal = open(f"{d1}/masks.json").read() == open(f"{d2}/masks.json").read()
        metrics_equal = open(f"{d1}/metrics.csv").read() == open(f"{d2}/metrics.csv").read()
    out[strategy] = {
        "theta_equal": bool(np.array_equal(ref.theta.view(np.uint64), ours.theta.view(np.uint64))),
        "masks_equal": masks_equal, "metrics_equal": metrics_equal,
        "steps": ref.summary["total_steps"], "calls": calls,
        "param_masks_equal": bool(np.array_equal(ref.assignment.param_masks, ours.assignment.param_masks)),
    }

# the reference's except clauses catch this package's errors
a = RM.build_assignment(S.build_mini_resnet(8, 2, 3, 2, 2, (4, 4), 0).topology, "block", 4, 2, 0)
try:
    OE.aggregate([np.zeros(a.topology.total)] * 3, a)
    out["protocol_caught"] = False
except RE.ProtocolError as exc:
    out["protocol_caught"] = isinstance(exc, OERR.ProtocolError)

# masks.json edge cases behave like the reference's assignment_from_dict
topo = S.build_mini_resnet(8, 2, 3, 2, 2, (4, 4), 0).topology
doc = RM.assignment_to_dict(RM.build_assignment(topo, "neuron", 4, 2, 5))
k = next(u for u in doc["units"] if u.startswith("channel:"))
lay = k.split(":")[1]
edge = {}
for tag, units in (("negative_index", {f"channel:{lay}:-1": [0, 1]}),
                   ("worker_out_of_range", {k: [0, 9]})):
    d2 = dict(doc, units=units)
    want = RM.assignment_from_dict(d2, topo).param_masks
    got = OM.assignment_from_dict(d2, topo).param_masks.cpu().numpy()
    edge[tag] = bool(np.array_equal(want, got))
for tag, units in (("index_too_large", {f"channel:{lay}:8": [0, 1]}),):
    d2 = dict(doc, units=units)
    errs = []
    for fn in (RM.assignment_from_dict, OM.assignment_from_dict):
        try:
            fn(d2, topo)
            errs.append(None)
        except Exception as exc:
            errs.append(type(exc).__name__)
    edge[tag] = errs
out["edge"] = edge

# read-only arrays, as the reference freezes them (test_masking.py:302-309)
oa = OM.build_assignment(topo, "block", 4, 2, 0)
ro = []
for arr in (oa.param_masks, oa.coverage, oa.divisor, oa.governors, oa.owner_mask):
    try:
        arr[0] = arr[0]
        ro.append(False)
    except ValueError:
        ro.append(True)
out["read_only"] = ro
print("RESULT " + json.dumps(out))
'''


def test_reference_engine_run_with_drop_in_is_bit_identical(cuda):
    from oracle import build_ref
    if build_ref.build() is None:
        pytest.skip("reference not staged in oracle/_ref")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(build_ref.OUT), str(ROOT), env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, env=env,
                       cwd=str(ROOT), timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    line = next(ln for ln in r.stdout.splitlines() if ln.startswith("RESULT "))
    res = json.loads(line[len("RESULT "):])
    for strategy in ("block", "neuron"):
        got = res[strategy]
        assert got["steps"] == 4 and got["calls"] == {"agg": 4, "build": 1}, got
        assert got["theta_equal"] and got["metrics_equal"] and got["masks_equal"], got
        assert got["param_masks_equal"], got
    assert res["protocol_caught"]
    assert res["edge"]["negative_index"] and res["edge"]["worker_out_of_range"]
    assert res["edge"]["index_too_large"] == ["IndexError", "IndexError"]
    assert all(res["read_only"])
