"""Checkpoint and training-state formats.

* `save_checkpoint` / `load_checkpoint`: the reference's format exactly
  (models.py:404-435) -- theta as little-endian float64 in `<prefix>.bin` plus
  a JSON sidecar `{dtype, total, params: {name: {offset, shape}}}` -- so files
  written here load in the reference and vice versa, bit-exact.  The device
  theta (fp32 or f64) is widened to f64 on the way out (exact) and narrowed to
  the caller's dtype on the way in.
* `save_training_state` / `load_training_state`: what the reference never
  persisted (no optimizer state, no step counter, no resume) --
  theta + optimizer moments (same `<f8` layout) + step + the masks.json
  assignment document, enough to resume the protocol bit-exactly.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import torch

from .errors import DataError
from .masking import assignment_from_dict, assignment_to_dict


def _host_f64(t) -> np.ndarray:
    if torch.is_tensor(t):
        return t.detach().to("cpu", torch.float64).numpy()
    return np.asarray(t, dtype=np.float64)


def save_checkpoint(model, prefix) -> tuple[Path, Path]:
    """theta -> <prefix>.bin (<f8) + <prefix>.json (models.py:404-419)."""
    prefix = Path(prefix)
    bin_path, json_path = prefix.with_suffix(".bin"), prefix.with_suffix(".json")
    bin_path.write_bytes(_host_f64(model.theta).astype("<f8").tobytes())
    sidecar = {"dtype": "<f8", "total": model.topology.total,
               "params": {p.name: {"offset": p.offset, "shape": list(p.shape)} for p in model.topology.params}}
    json_path.write_text(json.dumps(sidecar, indent=2, sort_keys=True))
    return bin_path, json_path


def load_checkpoint(prefix, device=None, dtype=torch.float64):
    """-> (theta tensor, params sidecar) (models.py:422-435); DataError on a
    missing or truncated file."""
    prefix = Path(prefix)
    bin_path, json_path = prefix.with_suffix(".bin"), prefix.with_suffix(".json")
    if not bin_path.exists() or not json_path.exists():
        raise DataError(f"checkpoint files {bin_path} / {json_path} not found")
    sidecar = json.loads(json_path.read_text())
    raw = bin_path.read_bytes()
    expected = int(sidecar["total"]) * 8
    if len(raw) != expected:
        raise DataError(f"checkpoint {bin_path} holds {len(raw)} bytes, expected {expected}")
    theta = torch.from_numpy(np.frombuffer(raw, dtype="<f8").astype(np.float64))
    theta = theta.to(dtype)
    if device is not None:
        theta = theta.to(device)
    return theta, sidecar["params"]


def save_training_state(prefix, model, assignment, step: int, optimizer: dict) -> Path:
    """theta checkpoint + optimizer state + step + masks.json under one prefix.

    optimizer: {"kind": "sgd-nesterov"|"adam", <moment name>: tensor, ...,
    "t": adam step} -- moments are stored as <f8 like theta."""
    prefix = Path(prefix)
    save_checkpoint(model, prefix)
    state = {"step": int(step), "kind": optimizer["kind"], "moments": {}, "scalars": {}}
    for k, v in optimizer.items():
        if k == "kind":
            continue
        if torch.is_tensor(v) or isinstance(v, np.ndarray):
            path = prefix.with_name(prefix.name + f".{k}.bin")
            path.write_bytes(_host_f64(v).astype("<f8").tobytes())
            state["moments"][k] = path.name
        else:
            state["scalars"][k] = v
    state["masks"] = assignment_to_dict(assignment)
    out = prefix.with_name(prefix.name + ".state.json")
    out.write_text(json.dumps(state, indent=2, sort_keys=True))
    return out


def load_training_state(prefix, topology, device=None, dtype=torch.float32):
    """-> (theta, assignment, step, optimizer dict) on `device`."""
    prefix = Path(prefix)
    sp = prefix.with_name(prefix.name + ".state.json")
    if not sp.exists():
        raise DataError(f"training state {sp} not found")
    state = json.loads(sp.read_text())
    theta, _ = load_checkpoint(prefix, device, dtype)
    opt = {"kind": state["kind"], **state["scalars"]}
    for k, name in state["moments"].items():
        raw = (prefix.parent / name).read_bytes()
        if len(raw) != topology.total * 8:
            raise DataError(f"moment {name} holds {len(raw)} bytes, expected {topology.total * 8}")
        t = torch.from_numpy(np.frombuffer(raw, dtype="<f8").copy()).to(dtype)
        opt[k] = t.to(device) if device is not None else t
    assignment = assignment_from_dict(state["masks"], topology, device)
    return theta, assignment, int(state["step"]), opt
