"""Monte-Carlo quantization-error experiment on the B200 paths.

Restates the reference's ``run_error_benchmark`` (harness.py:211-290) and its ``ErrorReport``
(harness.py:145-182): trial t of seed s draws x then w from ``numpy.random.default_rng([s, t])``
(harness.py:3-8, :219-221); every pipeline is run once per trial with valid padding, exactly as the
reference calls it:

* ground truth: fp64 direct correlation, ``conv2d_direct`` on the GPU (bit-identical to the
  reference's, same operation order);
* (mode, "float"): the float Winograd path ``conv2d_winograd`` (fp32 on the GPU: these two rows carry
  fp32 rounding, ~1e-7 relative, where the fp64 reference shows ~1e-15);
* (mode, qconfig): the quantized layer on fp64 operands (bit-exact with the reference per trial);
* ("direct", "float") = (0, 0) and ("direct", qconfig): ``conv2d_direct_quantized`` (bit-exact).

Metrics are the reference's ``_error_metrics`` (max-abs and relative-L2 of y - ref, numpy fp64 on
the host), aggregated as mean / std / median / max per (mode, qconfig, metric); stage-stat rows
average each stage's max_abs and scale over trials; the condition table is ``condition_table``
(harness.py:185-197).  Since every quantized and direct output and the ground truth are bit-exact,
those rows equal the reference's report (tests/test_gpu_harness.py against tests/golden/mc_report.json
and the published acceptance means).
"""

from __future__ import annotations

from dataclasses import asdict, dataclass, field

import numpy as np
import torch

from .layer import QuantWinogradConv, conv2d_direct, conv2d_direct_quantized, conv2d_winograd
from .plan import build_plan, plan_to_float
from .quantize import QuantConfig

METRICS = ("max_abs_err", "rel_l2_err")
FLOAT_QCONFIG = "float"
DIRECT_MODE = "direct"


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
    stage_stats: list = field(default_factory=list)
    condition_table: list = field(default_factory=list)

    def describe(self) -> dict:
        return {"o": 4, "k": 3, "points": "0,1,-1,2,-2,inf", "modes": list(self.modes),
                "qconfigs": [{"name": n, **asdict(q)} for n, q in self.qconfigs], "trials": self.trials,
                "seed": self.seed, "input_distribution": self.distribution, "channels": list(self.channels),
                "spatial": list(self.spatial)}

    def json_dict(self) -> dict:
        """Same layout as the reference's ErrorReport.json_dict (harness.py:172-175)."""
        return {"config": self.describe(), "rows": self.rows, "stage_stats": self.stage_stats,
                "condition_numbers": self.condition_table}


def _draw(rng, dist, shape):
    return rng.uniform(-1.0, 1.0, shape) if dist == "uniform" else rng.standard_normal(shape)


def _error_metrics(y: np.ndarray, ref: np.ndarray) -> tuple[float, float]:
    # harness.py:201-208
    diff = y - ref
    max_abs = float(np.max(np.abs(diff))) if diff.size else 0.0
    denom = float(np.linalg.norm(ref.ravel()))
    num = float(np.linalg.norm(diff.ravel()))
    rel = num / denom if denom > 0 else (0.0 if num == 0.0 else float("inf"))
    return max_abs, rel


def _cond(mat, norm: str) -> float:
    """Condition number for the report: sigma_max / sigma_min (two-norm; also the Frobenius fallback
    for non-square factors), ||M||_F ||M^-1||_F for square factors; inf when numerically singular."""
    m = np.asarray(mat, dtype=np.float64)
    s = np.linalg.svd(m, compute_uv=False)
    if s[-1] <= s[0] * max(m.shape) * np.finfo(np.float64).eps:
        return float("inf")
    if norm == "frobenius" and m.shape[0] == m.shape[1]:
        return float(np.linalg.norm(m, "fro") * np.linalg.norm(np.linalg.inv(m), "fro"))
    return float(s[0] / s[-1])


def condition_table(plan) -> list[dict]:
    """harness.py:185-197: two-norm and Frobenius condition numbers of every pipeline factor."""
    plan = plan_to_float(plan)
    mats = [("B^T", plan.B.T), ("G", plan.G), ("A^T", plan.A.T)]
    if plan.base_change is not None:
        mats += [("B_P^T", plan.B_P.T), ("G_P", plan.G_P), ("A_P^T", plan.A_P.T), ("P^T", plan.base_change.P.T),
                 ("P^-T", plan.base_change.P_inv.T)]
    return [{"matrix": n, "two_norm": _cond(m, "two"), "frobenius": _cond(m, "frobenius")}
            for n, m in mats]


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
    ho, wo = h - 2, w_ - 2
    ref = torch.empty((cfg.trials, cout, ho, wo), dtype=torch.float64, device=dev)
    for t in range(cfg.trials):
        ref[t] = conv2d_direct(X64[t], W64[t])
    refh = ref.cpu().numpy()

    outs, stages = {}, {}
    for mode in cfg.modes:
        yf = torch.empty((cfg.trials, cout, ho, wo), dtype=torch.float32, device=dev)
        X32, W32 = X64.float(), W64.float()
        for t in range(cfg.trials):
            yf[t] = conv2d_winograd(X32[t], W32[t], plan, mode)
        outs[(mode, FLOAT_QCONFIG)] = yf.double().cpu().numpy()
        for qname, qc in cfg.qconfigs:
            r = QuantWinogradConv(plan, mode, qc, dev)
            out = torch.empty_like(ref)
            st = []
            for t in range(cfg.trials):  # fp64 operands: the reference's own precision, bit-exact outputs
                r.forward(X64[t:t + 1], W64[t], padding=0, out=out[t:t + 1])
                st.append([(s.stage, s.bits, s.max_abs, s.scale) for s in r.stats()[0]])
            outs[(mode, qname)] = out.cpu().numpy()
            stages[(mode, qname)] = st
    for qname, qc in cfg.qconfigs:
        yd = torch.empty_like(ref)
        for t in range(cfg.trials):
            yd[t] = conv2d_direct_quantized(X64[t], W64[t], qc)
        outs[(DIRECT_MODE, qname)] = yd.cpu().numpy()

    metrics = {key: np.array([_error_metrics(y[t], refh[t]) for t in range(cfg.trials)]) for key, y in outs.items()}
    metrics[(DIRECT_MODE, FLOAT_QCONFIG)] = np.zeros((cfg.trials, 2))
    rows = []
    for mode in list(cfg.modes) + [DIRECT_MODE]:  # harness.py:256-270
        for qname in [FLOAT_QCONFIG] + [n for n, _ in cfg.qconfigs]:
            per_trial = metrics[(mode, qname)]
            for idx, metric in enumerate(METRICS):
                v = per_trial[:, idx]
                rows.append({"mode": mode, "qconfig": qname, "metric": metric, "mean": float(np.mean(v)),
                             "std": float(np.std(v)), "median": float(np.median(v)), "max": float(np.max(v)),
                             "trials": cfg.trials, "seed": cfg.seed})
    stage_rows = []
    for mode in cfg.modes:  # harness.py:272-285
        for qname, _ in cfg.qconfigs:
            per_trial = stages[(mode, qname)]
            max_abs = np.array([[s[2] for s in t] for t in per_trial])
            scales = np.array([[s[3] for s in t] for t in per_trial])
            for j, s in enumerate(per_trial[0]):
                stage_rows.append({"mode": mode, "qconfig": qname, "stage": s[0], "bits": s[1],
                                   "mean_max_abs": float(np.mean(max_abs[:, j])),
                                   "mean_scale": float(np.mean(scales[:, j]))})
    cfg.rows, cfg.stage_stats, cfg.condition_table = rows, stage_rows, condition_table(plan)
    return rows
