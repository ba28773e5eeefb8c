"""CPU checks of the product host side: construction vs the reference's golden plans, the public
API types, and the C-ABI library (loads without a GPU and exports every symbol of
include/winoleg_b200.h).  No device compute here."""

import ctypes
import json
import os
import re
from fractions import Fraction

import numpy as np
import pytest

import paper_2004_11077_b200 as W
from conftest import GOLDEN, ROOT
from paper_2004_11077_b200 import _lib


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "winoleg_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(wl_\w+)\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    names = header_symbols()
    assert len(names) >= 15
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(_lib.EXPORTS) == set(names)


def test_plan_matches_reference_golden():
    plans = json.load(open(os.path.join(GOLDEN, "plans.json")))
    for o in (2, 4, 6):
        p = W.build_plan(o, 3, use_legendre=True)
        mats = {"G": p.G, "BT": p.B.T, "AT": p.A.T, "P": p.base_change.P, "Pinv": p.base_change.P_inv,
                "G_P": p.G_P, "BPT": p.B_P.T, "APT": p.A_P.T}
        for name, m in mats.items():
            assert [[str(Fraction(v)) for v in row] for row in m] == plans[f"F({o},3)"][name], (o, name)


def test_stage_tables_match_generated_header():
    # the compiled tables are the integer stage matrices of the host construction
    hdr = open(os.path.join(ROOT, "paper_2004_11077_b200", "csrc", "wl_tables.cuh")).read()
    plan = W.build_plan(4, 3, use_legendre=True)
    for mode, prefix in (("canonical", "Can_"), ("legendre", "Leg_")):
        for name, sm in W.stage_matrices(plan, mode).items():
            body = "{" + ", ".join("{" + ", ".join(str(int(v)) for v in r) + "}" for r in sm.L_int) + "}"
            assert f"struct {prefix}{name.upper()}" in hdr and body in hdr, (mode, name)
            assert f"{prefix}{name.upper()}_D = {sm.D};" in hdr


def test_known_construction_facts():
    p = W.plan_to_float(W.build_plan(4, 3, use_legendre=True))
    assert np.allclose(p.base_change.P_inv @ p.B_P, p.B)        # P^-1 B_P = B  (pipeline.py:9-11)
    assert np.allclose(p.base_change.P_inv @ p.A_P, p.A)
    assert W.monic_legendre(4) == [Fraction(3, 35), 0, Fraction(-6, 7), 0, 1]
    # F(2,3): A^T ((G g) * (B^T d)) == correlation (reference test_construct.py:91-96 style)
    q = W.build_plan(2, 3)
    g, d = np.array([1, 2, 3], dtype=object), np.array([1, 2, 3, 4], dtype=object)
    assert list(q.A.T @ ((q.G @ g) * (q.B.T @ d))) == [14, 20]


def test_quant_config_api():
    assert W.QuantConfig.from_name("8b+9b").hadamard_bits == 9
    assert W.QuantConfig.from_name("8b") == W.QuantConfig.uniform(8)
    with pytest.raises(ValueError):
        W.QuantConfig.from_name("fast")
    with pytest.raises(ValueError):
        W.QuantConfig(input_bits=1)
    assert W.QuantParams(bits=8, scale=1.0).q_max == 127
    assert set(W.STAGE_BITS) == set(W.STAGE_ORDER["legendre"])


def test_points_and_errors():
    with pytest.raises(W.InvalidPointsError):
        W.InterpolationPoints.parse("0,1,1,inf")
    with pytest.raises(W.DimensionError):
        W.build_plan(4, 3, points=W.InterpolationPoints.parse("0,1,inf"))
    assert str(W.InterpolationPoints.default(6)) == "0,1,-1,2,-2,inf"
    from paper_2004_11077_b200.layer import _require_mode
    with pytest.raises(ValueError):
        _require_mode(W.build_plan(4, 3), "legendre")
    with pytest.raises(ValueError):
        _require_mode(W.build_plan(4, 3), "fourier")
