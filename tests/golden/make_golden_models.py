"""Golden vectors for extraction / write-back and the training step, made by
running the REFERENCE (masked_forward / flat_gradient / aggregate / Nesterov).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_models.py

For each case: theta, the worker's batch, the reference loss and its flat
gradient (models.py:333-382), for every worker; plus two protocol steps
(engine.py:202-223 without the dataset/eval plumbing): per-worker gradients ->
aggregate -> SgdNesterov.update, recording theta after each step.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def main() -> None:
    import subnetdp as S
    from subnetdp.engine import aggregate
    from subnetdp.models import flat_gradient, masked_forward
    from subnetdp.optim import SgdNesterov

    cases = [
        ("mini", dict(channels=8, blocks=3, classes=4, norm_groups=2, in_channels=2, image_hw=(4, 4)),
         "neuron", 4, 2, 3),
        ("mini", dict(channels=8, blocks=3, classes=4, norm_groups=2, in_channels=2, image_hw=(4, 4)),
         "block", 4, 2, 3),
        ("mini", dict(channels=6, blocks=2, classes=3, norm_groups=3, in_channels=2, image_hw=(4, 4)),
         "neuron", 3, 2, 4),
        ("mlp", dict(width=12, blocks=4, classes=3, in_dim=5), "neuron", 4, 3, 7),
        ("mlp", dict(width=12, blocks=4, classes=3, in_dim=5), "block", 4, 2, 7),
    ]
    arrays = {}
    manifest = {"numpy": np.__version__, "cases": []}
    for ci, (kind, kw, strategy, n, p, seed) in enumerate(cases):
        model = S.build_mini_resnet(seed=seed, **kw) if kind == "mini" else S.build_residual_mlp(seed=seed, **kw)
        a = S.build_assignment(model.topology, strategy, n, p, seed)
        model.theta = S.masked_kaiming_init(model, a, seed)
        rng = np.random.default_rng(500 + ci)
        bsz = 5
        xs = [rng.standard_normal((bsz,) + model.topology.input_shape) for _ in range(2 * n)]
        ys = [rng.integers(0, kw["classes"], size=bsz) for _ in range(2 * n)]
        arrays[f"m{ci}_theta0"] = model.theta.copy()
        for w in range(n):
            view = a.worker_view(w)
            loss, tape, params = masked_forward(model, view, xs[w], ys[w])
            g = flat_gradient(model, tape, loss, params)
            arrays[f"m{ci}_loss_w{w}"] = np.array([float(loss.data)])
            arrays[f"m{ci}_grad_w{w}"] = g
            # multiply mode gives the same loss
            loss_m, _, _ = masked_forward(model, view, xs[w], ys[w], block_mode="multiply")
            arrays[f"m{ci}_lossmul_w{w}"] = np.array([float(loss_m.data)])
        # gradient alignment (diagnostics.py:50-78) per worker on its first batch
        from subnetdp.diagnostics import gradient_alignment
        layers = [p.name for p in model.topology.params if p.kind in ("conv_w", "linear_w")]
        align = []
        for w in range(n):
            samples = gradient_alignment(model, a.worker_view(w), xs[w], ys[w], layers)
            align.append([[s.layer, s.cosine, s.reason] for s in samples])
        # two protocol steps: worker w uses batch (step*n + w)
        opt = SgdNesterov(model.topology.total, momentum=0.9)
        lrs = [0.1, 0.05]
        for t in range(2):
            grads = []
            for w in range(n):
                view = a.worker_view(w)
                loss, tape, params = masked_forward(model, view, xs[t * n + w], ys[t * n + w])
                grads.append(flat_gradient(model, tape, loss, params))
            agg = aggregate(grads, a)
            opt.update(model.theta, agg.gbar, lrs[t])
            arrays[f"m{ci}_theta_step{t + 1}"] = model.theta.copy()
        for k in range(2 * n):
            arrays[f"m{ci}_x{k}"] = xs[k]
            arrays[f"m{ci}_y{k}"] = ys[k]
        manifest["cases"].append({"id": ci, "kind": kind, "kw": {k: (list(v) if isinstance(v, tuple) else v)
                                                                 for k, v in kw.items()},
                                  "strategy": strategy, "n": n, "p": p, "seed": seed, "lrs": lrs,
                                  "d": model.topology.total, "alignment": align})
    np.savez_compressed(HERE / "models.npz", **arrays)
    (HERE / "models.json").write_text(json.dumps(manifest, indent=1))
    print("ok", {k: v.shape for k, v in list(arrays.items())[:4]})


if __name__ == "__main__":
    main()
