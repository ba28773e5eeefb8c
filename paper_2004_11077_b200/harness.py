"""Monte-Carlo quantization-error experiment on the B200 layer.

Restates the reference's `run_error_benchmark` (harness.py:211-290) for the quantized pipelines:
trial t of seed s draws x then w from numpy.random.default_rng([s, t]) (harness.py:3-8, :219-221),
runs the quantized Winograd layer per image with valid padding (one reference call per trial), and
reports the mean / std / median / max of the max-abs and relative-L2 error against the fp64 direct
correlation (harness.py:201-208).  Because the layer is bit-exact with the reference, the means
reproduce the reference's published numbers (test_output.txt:156).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .layer import QuantWinogradConv
from .plan import build_plan
from .quantize import QuantConfig


@dataclass
class ErrorExperiment:
    trials: int = 1000
    seed: int = 1234
    channels: tuple = (3, 2)
    spatial: tuple = (13, 14)
    modes: tuple = ("canonical", "legendre")
    qconfigs: tuple = (("8b", QuantConfig.uniform(8)), ("8b+9b", QuantConfig.uniform(8, hadamard_bits=9)))
    distribution: str = "standard-normal"
    rows: list = field(default_factory=list)


def _draw(rng, dist, shape):
    return rng.uniform(-1.0, 1.0, shape) if dist == "uniform" else rng.standard_normal(shape)


def run_error_benchmark(cfg: ErrorExperiment, device=None) -> list[dict]:
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    plan = build_plan(4, 3, use_legendre=True)
    cin, cout = cfg.channels
    h, w_ = cfg.spatial
    xs, ws = [], []
    for t in range(cfg.trials):
        rng = np.random.default_rng([cfg.seed, t])
        xs.append(_draw(rng, cfg.distribution, (cin, h, w_)))
        ws.append(_draw(rng, cfg.distribution, (cout, cin, 3, 3)))
    X64 = torch.tensor(np.stack(xs), dtype=torch.float64, device=dev)
    W64 = torch.tensor(np.stack(ws), dtype=torch.float64, device=dev)
    # fp64 direct correlation (the metric's reference, not the measured path), all trials at once
    ref = torch.nn.functional.conv2d(X64.reshape(1, -1, h, w_), W64.reshape(-1, cin, 3, 3), groups=cfg.trials)
    ref = ref.reshape(cfg.trials, cout, h - 2, w_ - 2)
    rows = []
    for mode in cfg.modes:
        for qname, qc in cfg.qconfigs:
            r = QuantWinogradConv(plan, mode, qc, dev)
            out = torch.empty_like(ref)
            for t in range(cfg.trials):  # fp64 operands: the reference's own precision, bit-exact outputs
                r.forward(X64[t:t + 1], W64[t], padding=0, out=out[t:t + 1])
            diff = out - ref
            max_abs = diff.abs().flatten(1).max(dim=1).values
            rel = diff.flatten(1).norm(dim=1) / ref.flatten(1).norm(dim=1)
            for metric, vals in (("max_abs_err", max_abs), ("rel_l2_err", rel)):
                v = vals.cpu().numpy()
                rows.append({"mode": mode, "qconfig": qname, "metric": metric, "mean": float(np.mean(v)),
                             "std": float(np.std(v)), "median": float(np.median(v)), "max": float(np.max(v)),
                             "trials": cfg.trials, "seed": cfg.seed})
    cfg.rows = rows
    return rows
