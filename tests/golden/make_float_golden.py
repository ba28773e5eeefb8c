"""Golden fixtures for the float (unquantized) Winograd path and the direct baselines, generated
from the UNMODIFIED reference (build container only):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_float_golden.py

For each seeded case: fp32-representable x [c_in,H,W] (explicitly zero padded when pad > 0, as the
reference is valid-correlation only) and w [c_out,c_in,3,3]; the reference's
  conv2d_winograd(x, w, plan, mode) for both bases (pipeline.py:161-164),
  conv2d_direct(x, w)                  (reference.py:34-39),
  conv2d_direct_quantized(x, w, qc)    (quantize.py:151-160, 8-bit QuantConfig()).
Output: float_cases.npz.
"""

from __future__ import annotations

import json
import os

import numpy as np

import winoleg as R
from winoleg.quantize import conv2d_direct_quantized
from winoleg.reference import conv2d_direct

HERE = os.path.dirname(os.path.abspath(__file__))


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def main():
    plan = R.plan_to_float(R.build_plan(4, 3, use_legendre=True))
    out, meta = {}, []
    cases = [("rand_a", 0, 3, 5, 11, 13, 0), ("rand_b", 1, 6, 4, 9, 16, 1), ("rand_c", 2, 16, 8, 18, 18, 1),
             ("cfg1ish", 3, 32, 16, 16, 16, 1)]
    for name, seed, cin, cout, h, w_, pad in cases:
        rng = np.random.default_rng(100 + seed)
        x = f32(rng.standard_normal((cin, h, w_)))
        w = f32(rng.standard_normal((cout, cin, 3, 3)) * np.sqrt(2.0 / (9 * cin)))
        xp = np.pad(x, ((0, 0), (pad, pad), (pad, pad))) if pad else x
        out[f"{name}_x"], out[f"{name}_w"] = x.astype(np.float32), w.astype(np.float32)
        for mode in ("canonical", "legendre"):
            out[f"{name}_wino_{mode}"] = R.conv2d_winograd(xp, w, plan, mode)
        out[f"{name}_direct"] = conv2d_direct(xp, w)
        out[f"{name}_directq8"] = conv2d_direct_quantized(xp, w, R.QuantConfig())
        meta.append({"name": name, "pad": pad})
    np.savez_compressed(os.path.join(HERE, "float_cases.npz"), meta=json.dumps(meta), **out)


if __name__ == "__main__":
    main()
