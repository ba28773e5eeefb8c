"""CPU: the closed-form STE backward (what the sm_100a path implements) equals torch fp64 autograd
of the staged quantized pipeline with straight-through casts.  Pins oracle.backward_ref."""

import numpy as np
import pytest

from oracle import backward_ref as BR
from oracle import oracle as O


@pytest.mark.parametrize("mode", ["canonical", "legendre"])
@pytest.mark.parametrize("seed,cin,cout,h,w,pad", [(0, 3, 4, 8, 8, 1), (1, 2, 5, 9, 11, 0), (2, 4, 3, 6, 13, 1)])
def test_closed_form_equals_autograd(mode, seed, cin, cout, h, w, pad):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((2, cin, h, w))
    wt = rng.standard_normal((cout, cin, 3, 3))
    bits = O.uniform_bits(8, 9)
    ho, wo = h + 2 * pad - 2, w + 2 * pad - 2
    dy = rng.standard_normal((2, cout, ho, wo))
    # one scale group over the whole (2-image) batch, as the autograd pipeline casts whole tensors
    _, dx_a, dw_a, U, V = BR.ste_autograd(x, wt, mode, bits, pad, dy)
    dx_f, dw_f, db_f = BR.ste_formula(dy, U, V, h, w, pad)
    assert np.allclose(dx_f, dx_a, rtol=1e-10, atol=1e-10)
    assert np.allclose(dw_f, dw_a, rtol=1e-10, atol=1e-10)
    assert np.allclose(db_f, dy.sum(axis=(0, 2, 3)))


def test_quantised_operands_shapes():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 3, 7, 7))
    w = rng.standard_normal((4, 3, 3, 3))
    U, V = BR.quantised_operands(x, w, "legendre", O.uniform_bits(8), 1)
    assert U.shape == (4, 3, 6, 6) and V.shape == (2, 3, 4, 6, 6)
