"""GPU: the quantized direct-convolution baseline, §8f row 3 — the reference's
conv2d_direct_quantized (quantize.py:151-160) — bit-exact against the reference's own outputs
(tests/golden/float_cases.npz, key *_directq8, made by importing the reference) and against the
pinned fp64 oracle (oracle/float_ref.py) on batched, padded, per-image / per-batch, 8/9/4-bit cases."""
import json
import os

import numpy as np
import pytest
import torch

import paper_2004_11077_b200 as W
from oracle import float_ref as F
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "float_cases.npz")


def _oracle(x, w, qin, qw, qout):
    return O.fake_quant(F.direct(O.fake_quant(x, qin), O.fake_quant(w, qw)), qout)


def test_direct_quantized_vs_reference_golden():
    z = np.load(GOLD, allow_pickle=False)
    for m in json.loads(str(z["meta"])):
        n, pad = m["name"], m["pad"]
        y = W.conv2d_direct_quantized(z[f"{n}_x"], z[f"{n}_w"], W.QuantConfig(), padding=pad)
        assert y.dtype == np.float64 and np.array_equal(y, z[f"{n}_directq8"]), n


@pytest.mark.parametrize("groups", ["image", "batch"])
@pytest.mark.parametrize("bits", [(8, 8, 8), (8, 8, 9), (4, 6, 5)])
def test_direct_quantized_batched_vs_oracle(groups, bits):
    rng = np.random.default_rng(11)
    x = rng.standard_normal((3, 7, 10, 9))
    x[1] = np.maximum(x[1], 0.0)
    w = rng.standard_normal((5, 7, 3, 3)) * np.sqrt(2 / 63)
    qin, qw, qout = bits
    qc = W.QuantConfig(input_bits=qin, weight_bits=qw, output_transform_bits=qout)
    y = W.conv2d_direct_quantized(torch.as_tensor(x, device="cuda"), torch.as_tensor(w, device="cuda"), qc,
                                  padding=1, scale_groups=groups).cpu().numpy()
    xp = np.pad(x, ((0, 0), (0, 0), (1, 1), (1, 1)))
    if groups == "image":
        ref = np.stack([_oracle(xp[i], w, qin, qw, qout) for i in range(3)])
    else:  # one cast over the whole [N, ...] tensor at each quantisation point
        xq = O.fake_quant(xp, qin)
        wq = O.fake_quant(w, qw)
        ref = O.fake_quant(np.stack([F.direct(xq[i], wq) for i in range(3)]), qout)
    assert np.array_equal(y, ref)


def test_direct_quantized_fp32_and_zero():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 4, 6, 6)).astype(np.float32)
    x[1] = 0.0  # all-zero image: scales 1.0, output zero (quantize.py:115-117)
    w = rng.standard_normal((3, 4, 3, 3)).astype(np.float32)
    y = W.conv2d_direct_quantized(torch.as_tensor(x, device="cuda"), torch.as_tensor(w, device="cuda")).cpu().numpy()
    assert y.dtype == np.float32
    ref = np.stack([_oracle(x[i].astype(np.float64), w.astype(np.float64), 8, 8, 8) for i in range(2)])
    assert np.array_equal(y, ref.astype(np.float32))
    assert not np.any(y[1])


def test_direct_quantized_errors():
    with pytest.raises(W.DimensionError):
        W.conv2d_direct_quantized(np.zeros((2, 2, 2)), np.zeros((1, 2, 3, 3)))
    with pytest.raises(W.DimensionError):
        W.conv2d_direct_quantized(np.zeros((3, 6, 6)), np.zeros((1, 2, 3, 3)))


def test_direct_f64_vs_reference_golden():
    # the reference's conv2d_direct (reference.py:34-39), bit for bit, valid and padded
    z = np.load(GOLD, allow_pickle=False)
    for m in json.loads(str(z["meta"])):
        n, pad = m["name"], m["pad"]
        y = W.conv2d_direct(z[f"{n}_x"], z[f"{n}_w"], padding=pad)
        assert np.array_equal(y, z[f"{n}_direct"]), n
