"""Golden Monte-Carlo error reports generated from the UNMODIFIED reference
(build container only):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_mc_golden.py

Runs winoleg.harness.run_error_benchmark (harness.py:211-290) on small experiments — the published
acceptance geometry (F(4,3), C=(3,2), 13x14, seed 424242) with 100 trials, and a uniform-input,
C=(4,3), 10x11, 8b/6b-mixed experiment with 40 trials — and stores every metric row, stage-stat row
and the condition table.  Output: mc_report.json.
"""

from __future__ import annotations

import json
import os

from winoleg.harness import ExperimentConfig, run_error_benchmark
from winoleg.quantize import QuantConfig

HERE = os.path.dirname(os.path.abspath(__file__))

EXPERIMENTS = {
    "acceptance100": dict(trials=100, seed=424242),
    "uniform40": dict(trials=40, seed=7, input_distribution="uniform", channels=(4, 3), spatial=(10, 11),
                      qconfigs=(("8b", QuantConfig.uniform(8)),
                                ("6b/9b", QuantConfig(input_bits=6, weight_bits=6, hadamard_bits=9))),
                      ),
}


def main():
    out = {}
    for name, kw in EXPERIMENTS.items():
        cfg = ExperimentConfig(**kw)
        rep = run_error_benchmark(cfg)
        out[name] = rep.json_dict()
    with open(os.path.join(HERE, "mc_report.json"), "w") as fh:
        json.dump(out, fh, indent=1)
        fh.write("\n")


if __name__ == "__main__":
    main()
