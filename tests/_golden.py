"""Loader for the committed golden vectors (tests/golden/, made by running the
reference with tests/golden/make_golden.py)."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=1)
def manifest() -> dict:
    return json.loads((GOLDEN / "assignments.json").read_text())


@lru_cache(maxsize=1)
def arrays():
    return dict(np.load(GOLDEN / "assignments.npz"))


@lru_cache(maxsize=1)
def permutations():
    return dict(np.load(GOLDEN / "permutations.npz"))


def topology(model_key: str):
    from paper_2507_09029_b200 import zoo
    spec = dict(manifest()["models"][model_key])
    kind = spec.pop("kind")
    if kind == "mini_resnet":
        spec["image_hw"] = tuple(spec["image_hw"])
        return zoo.mini_resnet_topology(**spec)
    return zoo.residual_mlp_topology(**spec)


def cases(with_grads: bool = False):
    return [c for c in manifest()["cases"] if c.get("has_grads") or not with_grads]


def case_masks(case) -> np.ndarray:
    return np.unpackbits(arrays()[f"c{case['id']}_masks"], axis=1, count=case["d"]).astype(bool)


def case_inputs(case, masks: np.ndarray):
    """Regenerate the seeded f64 inputs exactly as make_golden.py drew them."""
    d, n = case["d"], case["n"]
    rng = np.random.default_rng(1000 + case["id"])
    grads = np.stack([rng.standard_normal(d) * masks[i] for i in range(n)])
    theta0 = rng.standard_normal(d)
    vel0 = rng.standard_normal(d) * 0.1
    return grads, theta0, vel0


def seeds():
    p = permutations()
    return [int(lo) | (int(hi) << 64) for lo, hi in zip(p["seed_lo"], p["seed_hi"])]
