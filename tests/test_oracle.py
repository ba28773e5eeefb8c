"""Pin the CPU oracle to the reference: golden fixtures made by importing the unmodified reference
(tests/golden/make_golden.py) and the reference's own published known answers.  CPU only."""

import json
import os
from fractions import Fraction

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import GOLDEN, golden_cases, load_case
from oracle import oracle as O
from oracle import plan_ref


def test_plans_match_reference_exactly():
    plans = json.load(open(os.path.join(GOLDEN, "plans.json")))
    for o in (2, 4, 6):
        ep = plan_ref.exact_plan(o, 3)
        ref = plans[f"F({o},3)"]
        for name in ("G", "BT", "AT", "P", "Pinv", "G_P", "BPT", "APT"):
            got = [[str(Fraction(v)) for v in row] for row in ep[name]]
            assert got == ref[name], (o, name)


def test_golden_base_change_m6():
    # reference tests/test_legendre.py:8-23 (published P^T and P^-T for m=6)
    P, Pi = plan_ref.legendre_pair(6)
    PT = plan_ref.transpose(P)
    assert PT[2][0] == Fraction(-1, 3) and PT[4][0] == Fraction(3, 35) and PT[5][3] == Fraction(-10, 9)
    PiT = plan_ref.transpose(Pi)
    assert PiT[4][0] == Fraction(1, 5) and PiT[5][1] == Fraction(3, 7) and PiT[5][3] == Fraction(10, 9)
    assert sum(1 for r in P for v in r if v != 0) == 12


def test_fake_quant_known_answers():
    for case in json.load(open(os.path.join(GOLDEN, "fake_quant.json"))):
        got = O.fake_quant(np.array(case["x"]), case["bits"])
        assert np.array_equal(got, np.array(case["y"]))
    # reference tests/test_quantize.py:40-44
    assert np.array_equal(O.fake_quant(np.array([1.0, -1.0, 0.5]), 8), np.array([1.0, -1.0, 64.0 / 127.0]))
    assert np.array_equal(O.fake_quant(np.array([0.0]), 8), np.array([0.0]))


finite = st.floats(min_value=-1e300, max_value=1e300, allow_nan=False, allow_infinity=False,
                   allow_subnormal=False)


@settings(max_examples=200, deadline=None)
@given(st.lists(finite, min_size=1, max_size=48), st.integers(2, 16))
def test_fake_quant_laws(values, bits):
    # reference tests/test_quantize.py:54-74
    x = np.array(values)
    y = O.fake_quant(x, bits)
    assert np.array_equal(O.fake_quant(y, bits), y)
    assert np.array_equal(O.fake_quant(-x, bits), -y)
    mx = np.max(np.abs(x))
    assert np.max(np.abs(y)) <= mx
    if mx > 0:
        assert mx in np.abs(y)


@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: os.path.basename(p)[5:-4])
def test_oracle_bit_exact_vs_reference(path):
    c = load_case(path)
    meta = c["meta"]
    x = c["x"].astype(np.float64)[None]
    y, stats, codes = O.quant_conv_batch(x, c["w"].astype(np.float64), meta["mode"], meta["bits"],
                                         padding=meta["pad"], capture=True)
    assert np.array_equal(y[0], c["y"])
    got = [(s.stage, s.bits, s.max_abs, s.scale) for s in stats[0]]
    want = list(zip(meta["stages"], c["stat_bits"].tolist(), c["stat_max_abs"].tolist(),
                    c["stat_scale"].tolist()))
    assert got == want
    for stage in meta["stages"]:
        key = "codes_" + stage
        if key not in c:
            continue
        ref = c[key]
        mine = codes[stage]
        if stage in ("input_base_change", "input_transform", "hadamard", "output_base_change"):
            mine = mine[0]
            ref = ref.reshape(mine.shape)
        elif stage in ("input", "output"):
            mine = mine[0]
        elif stage != "weights":
            ref = ref.reshape(mine.shape)
        assert np.array_equal(mine, ref), stage


def _direct(x, w):
    cout, cin, k, _ = w.shape
    oh, ow = x.shape[1] - k + 1, x.shape[2] - k + 1
    out = np.zeros((cout, oh, ow))
    for p in range(k):
        for q in range(k):
            out += np.einsum("oc,chw->ohw", w[:, :, p, q], x[:, p:p + oh, q:q + ow])
    return out


def test_monte_carlo_known_answer():
    """Reference acceptance MC (harness.py:211-238; test_output.txt:156):
    F(4,3), C=(3,2), 13x14, N(0,1), seed 424242, 1000 trials -> mean rel-L2."""
    want = {("canonical", 8): 2.72492, ("canonical", 9): 1.52523,
            ("legendre", 8): 4.20480, ("legendre", 9): 3.58458}
    xs, ws = [], []
    for t in range(1000):
        rng = np.random.default_rng([424242, t])
        xs.append(rng.standard_normal((3, 13, 14)))
        ws.append(rng.standard_normal((2, 3, 3, 3)))
    refs = [_direct(x, w) for x, w in zip(xs, ws)]
    for (mode, hb), mean in want.items():
        rel = []
        for x, w, r in zip(xs, ws, refs):
            y, _ = O.conv2d_winograd_quantized(x, w, mode, O.uniform_bits(8, hb))
            rel.append(np.linalg.norm((y - r).ravel()) / np.linalg.norm(r.ravel()))
        assert round(float(np.mean(rel)), 5) == pytest.approx(mean, abs=1.5e-5), (mode, hb)


def test_per_image_groups_equal_independent_calls():
    rng = np.random.default_rng(7)
    x = rng.standard_normal((3, 4, 9, 10)).astype(np.float32).astype(np.float64)
    w = rng.standard_normal((5, 4, 3, 3)).astype(np.float32).astype(np.float64)
    for mode in ("canonical", "legendre"):
        y, st_, _ = O.quant_conv_batch(x, w, mode, O.uniform_bits(8), padding=1, images_per_group=1)
        for n in range(3):
            yn, sn = O.conv2d_winograd_quantized(np.pad(x[n], ((0, 0), (1, 1), (1, 1))), w, mode,
                                                 O.uniform_bits(8))
            assert np.array_equal(y[n], yn)
            assert st_[n] == sn
