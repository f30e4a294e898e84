"""Checkpoint formats vs a checkpoint the REFERENCE wrote (tests/golden/ckpt_ref.*,
models.py:404-435): byte-identical output, bit-exact round trip (CPU)."""

from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2507_09029_b200 import checkpoint, zoo
from paper_2507_09029_b200.errors import DataError
from paper_2507_09029_b200.topology import GlobalModel

GOLDEN = Path(__file__).resolve().parent / "golden"


def _model(theta):
    topo = zoo.mini_resnet_topology(8, 3, 4, 2, 2, (4, 4))
    return GlobalModel(arch=None, topology=topo, theta=theta)


def test_reads_reference_checkpoint_and_writes_identical_bytes(tmp_path):
    theta, params = checkpoint.load_checkpoint(GOLDEN / "ckpt_ref")
    ref_raw = (GOLDEN / "ckpt_ref.bin").read_bytes()
    assert theta.dtype == torch.float64 and theta.numel() * 8 == len(ref_raw)
    assert np.array_equal(theta.numpy().view(np.uint64), np.frombuffer(ref_raw, "<u8"))
    m = _model(theta)
    assert params == {p.name: {"offset": p.offset, "shape": list(p.shape)} for p in m.topology.params}
    b, j = checkpoint.save_checkpoint(m, tmp_path / "ours")
    assert b.read_bytes() == ref_raw
    assert j.read_text() == (GOLDEN / "ckpt_ref.json").read_text()


def test_fp32_theta_round_trip_exact(tmp_path):
    th = torch.randn(_model(None).topology.total, dtype=torch.float32)
    m = _model(th)
    checkpoint.save_checkpoint(m, tmp_path / "c")
    back, _ = checkpoint.load_checkpoint(tmp_path / "c", dtype=torch.float32)
    assert torch.equal(back.view(torch.int32), th.view(torch.int32))


def test_truncated_and_missing_raise_data_error(tmp_path):
    with pytest.raises(DataError):
        checkpoint.load_checkpoint(tmp_path / "nope")
    m = _model(torch.zeros(_model(None).topology.total, dtype=torch.float64))
    b, _ = checkpoint.save_checkpoint(m, tmp_path / "t")
    b.write_bytes(b.read_bytes()[:-8])
    with pytest.raises(DataError, match="expected"):
        checkpoint.load_checkpoint(tmp_path / "t")


@pytest.mark.gpu
def test_training_state_resume_bitexact(cuda, tmp_path):
    from paper_2507_09029_b200 import masking
    topo = zoo.mini_resnet_topology(8, 3, 4, 2, 2, (4, 4))
    a = masking.build_assignment(topo, "neuron", 8, 3, seed=5)
    th = torch.randn(topo.total, device=cuda)
    vel = torch.randn(topo.total, device=cuda)
    m = GlobalModel(arch=None, topology=topo, theta=th)
    checkpoint.save_training_state(tmp_path / "run", m, a, 17, {"kind": "sgd-nesterov", "velocity": vel})
    th2, a2, step, opt = checkpoint.load_training_state(tmp_path / "run", topo, cuda, torch.float32)
    assert step == 17 and opt["kind"] == "sgd-nesterov"
    assert torch.equal(th2, th) and torch.equal(opt["velocity"], vel)
    assert torch.equal(a2.owner_mask, a.owner_mask) and a2.unit_workers == a.unit_workers
