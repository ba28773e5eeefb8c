"""Generate the golden fixtures in this directory from the UNMODIFIED reference.

Run in the build container only (the reference is not present on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

It imports the reference ``winoleg`` package (default numba backend) and records, for a set of
seeded cases, the inputs, the reference output, the reference StageStat list, and the integer
codes of every stage cast (captured with a cast hook that mirrors reference quantize.py:139-145).
Inputs are drawn in float64 and rounded to float32 first, so the same bytes feed the fp32 B200
layer.  Outputs: ``plans.json`` (exact F(o,3) matrices) and ``case_*.npz``.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

import winoleg as R
from winoleg.pipeline import run_pipeline
from winoleg.quantize import STAGE_BITS

HERE = os.path.dirname(os.path.abspath(__file__))


def capture_run(x, w, plan, mode, qc):
    """Reference quantized pipeline with a cast hook that also records each stage's codes."""
    stats, codes = [], {}

    def cast(stage, t):
        bits = getattr(qc, STAGE_BITS[stage])
        p = R.compute_scale(t, bits)
        mx = float(np.max(np.abs(t))) if t.size else 0.0
        stats.append((stage, bits, mx, p.scale))
        q = 2 ** (bits - 1) - 1
        codes[stage] = np.clip(np.rint(np.asarray(t, dtype=np.float64) / p.scale), -q, q).astype(np.int32)
        return R.fake_quant(t, bits)

    y = run_pipeline(x, w, plan, mode, cast=cast)
    # cross-check against the public entry point (quantize.py:129)
    y2, st2 = R.conv2d_winograd_quantized(x, w, plan, mode, qc)
    assert np.array_equal(y, y2)
    assert [(s.stage, s.bits, s.max_abs, s.scale) for s in st2] == stats
    return y, stats, codes


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def save_case(name, x, w, mode, qc, qname, pad, keep_weight_codes=True):
    plan = R.plan_to_float(R.build_plan(4, 3, use_legendre=True))
    xp = np.pad(x, ((0, 0), (pad, pad), (pad, pad))) if pad else x
    y, stats, codes = capture_run(xp, w, plan, mode, qc)
    arrays = {
        "x": x.astype(np.float32), "w": w.astype(np.float32), "y": y,
        "stat_bits": np.array([s[1] for s in stats], dtype=np.int32),
        "stat_max_abs": np.array([s[2] for s in stats]),
        "stat_scale": np.array([s[3] for s in stats]),
    }
    for stage, c in codes.items():
        if stage in ("weights", "weight_transform", "weight_base_change") and not keep_weight_codes:
            continue
        arrays["codes_" + stage] = c.astype(np.int8 if np.abs(c).max(initial=0) < 128 else np.int16)
    meta = {"mode": mode, "qconfig": qname, "pad": pad, "stages": [s[0] for s in stats],
            "bits": {f: getattr(qc, f) for f in ("input_bits", "weight_bits", "input_transform_bits",
                                                 "weight_transform_bits", "base_change_bits",
                                                 "hadamard_bits", "output_transform_bits")}}
    np.savez_compressed(os.path.join(HERE, f"case_{name}.npz"), meta=json.dumps(meta), **arrays)
    print("wrote", name, x.shape, w.shape, mode, qname, file=sys.stderr)


def main():
    # exact plans
    plans = {}
    for o in (2, 4, 6):
        p = R.build_plan(o, 3, use_legendre=True)
        d = {}
        for name, mat in (("G", p.G), ("BT", p.B.T), ("AT", p.A.T), ("P", p.base_change.P),
                          ("Pinv", p.base_change.P_inv), ("G_P", p.G_P), ("BPT", p.B_P.T),
                          ("APT", p.A_P.T)):
            d[name] = [[str(v) for v in row] for row in mat]
        plans[f"F({o},3)"] = d
    with open(os.path.join(HERE, "plans.json"), "w") as fh:
        json.dump(plans, fh, indent=1)

    # fake-quant known answers
    rng = np.random.default_rng(5)
    fq = []
    for bits in (2, 5, 8, 9, 12):
        v = rng.standard_normal(37) * 10.0 ** rng.uniform(-3, 3)
        fq.append({"bits": bits, "x": v.tolist(), "y": R.fake_quant(v, bits).tolist()})
    with open(os.path.join(HERE, "fake_quant.json"), "w") as fh:
        json.dump(fq, fh)

    u8 = R.QuantConfig.uniform(8)
    u89 = R.QuantConfig.uniform(8, hadamard_bits=9)
    odd = R.QuantConfig(input_bits=7, weight_bits=6, input_transform_bits=8, weight_transform_bits=8,
                        base_change_bits=7, hadamard_bits=9, output_transform_bits=13)
    # A. small random shapes, both bases, both widths, valid padding
    for seed in range(6):
        rng = np.random.default_rng(seed)
        cin, cout = (int(v) for v in rng.integers(1, 9, 2))
        h, wd = (int(v) for v in rng.integers(3, 20, 2))
        x = f32(rng.standard_normal((cin, h, wd)))
        w = f32(rng.standard_normal((cout, cin, 3, 3)))
        for mode in ("canonical", "legendre"):
            qc, qn = (u8, "8b") if seed % 2 == 0 else (u89, "8b+9b")
            save_case(f"rand{seed}_{mode}", x, w, mode, qc, qn, pad=seed % 2)
    # B. all-zero input
    save_case("zero_legendre", np.zeros((2, 6, 6)), f32(np.random.default_rng(9).standard_normal((3, 2, 3, 3))),
              "legendre", u8, "8b", 0)
    # C. integer-valued data: many exact rounding ties at every stage
    rng = np.random.default_rng(11)
    xi = rng.integers(-3, 4, (8, 12, 12)).astype(np.float64)
    wi = rng.integers(-2, 3, (8, 8, 3, 3)).astype(np.float64)
    for mode in ("canonical", "legendre"):
        save_case(f"ints_{mode}", xi, wi, mode, u8, "8b", 1)
        save_case(f"ints9_{mode}", xi, wi, mode, u89, "8b+9b", 1)
    # D. config-1 image (C=64, 32x32, pad 1, Kaiming weights fan_in 576)
    rng = np.random.default_rng(0)
    x = f32(rng.standard_normal((64, 32, 32)))
    w = f32(rng.standard_normal((64, 64, 3, 3)) * np.sqrt(2.0 / 576))
    save_case("cfg1img_legendre", x, w, "legendre", u8, "8b", 1)
    save_case("cfg1img_canonical", x, w, "canonical", u8, "8b", 1)
    # E. config-2 image, 9-bit Hadamard
    rng = np.random.default_rng(2)
    x = f32(rng.standard_normal((128, 16, 16)))
    w = f32(rng.standard_normal((32, 128, 3, 3)) * np.sqrt(2.0 / (9 * 128)))
    save_case("cfg2img_legendre9", x, w, "legendre", u89, "8b+9b", 1, keep_weight_codes=False)
    save_case("cfg2img_canonical9", x, w, "canonical", u89, "8b+9b", 1, keep_weight_codes=False)
    # F. C=256, 8x8, ReLU input (config-3c shape, tie-heavy input transform), fewer out channels
    rng = np.random.default_rng(3)
    x = f32(np.maximum(rng.standard_normal((256, 8, 8)), 0))
    w = f32(rng.standard_normal((16, 256, 3, 3)) * np.sqrt(2.0 / (9 * 256)))
    save_case("c256_canonical", x, w, "canonical", u8, "8b", 1, keep_weight_codes=False)
    save_case("c256_legendre", x, w, "legendre", u8, "8b", 1, keep_weight_codes=False)
    # G. non-uniform widths, odd extents (13x14 valid)
    rng = np.random.default_rng(424242)
    x = f32(rng.standard_normal((3, 13, 14)))
    w = f32(rng.standard_normal((2, 3, 3, 3)))
    for mode in ("canonical", "legendre"):
        save_case(f"odd_{mode}", x, w, mode, odd, "odd", 0)


if __name__ == "__main__":
    main()
