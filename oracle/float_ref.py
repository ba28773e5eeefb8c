"""TEST INFRASTRUCTURE ONLY — fp64 restatements of the reference's unquantized Winograd path and
its direct baselines (checkers for the GPU float path, §8f rows 2-3).

* ``winograd_float(x, w, mode)``  run_pipeline with the identity cast (pipeline.py:106-158 via
  conv2d_winograd, :161-164): tiles of m=6 at stride 4 with pad-to-tile (pipeline.py:79-91),
  sandwiches L . X . L^T in the numba order tmp = X . R, then L . tmp (_kernels.py:69-92),
  Hadamard sum over c (_kernels.py:94-105), crop (pipeline.py:94-99).  Pinned to the reference's
  own outputs (tests/golden/float_cases.npz) to 1e-12 relative.
* ``direct(x, w)``                _conv2d_direct_nb (_kernels.py:53-66), same summation order
  (c, p, q ascending, product then add): bit-identical.
* ``direct_quantized(x, w, bits)`` quantize.py:151-160: fake_quant input and weights, direct
  correlation, fake_quant the output (the C oracle's fake_quant).

Only ``tests/`` may import this module; the product package never does.
"""

from __future__ import annotations

import numpy as np

from . import oracle as O
from . import plan_ref


def _mats(mode: str):
    ep = plan_ref.exact_plan(4, 3)
    f = {k: plan_ref.to_f64(ep[k]) for k in ("G", "BT", "AT", "Pinv", "G_P", "BPT", "APT")}
    if mode == "canonical":
        return {"wt": [f["G"]], "it": [f["BT"]], "ot": [f["AT"]]}
    pinv_t = np.ascontiguousarray(f["Pinv"].T)
    # weight: G_P then P^-1; input: P^-T then B_P^T; output: P^-T then A_P^T   (pipeline.py:132-155)
    return {"wt": [f["G_P"], f["Pinv"]], "it": [pinv_t, f["BPT"]], "ot": [pinv_t, f["APT"]]}


def _sandwich(L, X):
    """L . X . L^T over the leading batch axes, numba order (tmp = X . L^T, then L . tmp)."""
    return np.matmul(L, np.matmul(X, L.T))


def winograd_float(x, w, mode: str):
    """Reference conv2d_winograd for one image x [c_in, H, W] (valid correlation), fp64."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    c_in, h, wd = x.shape
    c_out = w.shape[0]
    o, m = 4, 6
    ho, wo = h - 2, wd - 2
    th, tw = -(-ho // o), -(-wo // o)
    xp = np.zeros((c_in, (th - 1) * o + m, (tw - 1) * o + m))
    xp[:, :h, :wd] = x
    tiles = np.stack([xp[:, o * i: o * i + m, o * j: o * j + m] for i in range(th) for j in range(tw)], axis=1)
    M = _mats(mode)
    u = w
    for L in M["wt"]:
        u = _sandwich(L, u)
    v = tiles
    for L in M["it"]:
        v = _sandwich(L, v)
    acc = np.einsum("oimn,itmn->otmn", u, v)  # [c_out, T, 6, 6]
    y = acc
    for L in M["ot"]:
        y = _sandwich(L, y)
    out = np.zeros((c_out, th * o, tw * o))
    for idx in range(th * tw):
        i, j = divmod(idx, tw)
        out[:, o * i: o * i + o, o * j: o * j + o] = y[:, idx]
    return out[:, :ho, :wo]


def direct(x, w):
    """_conv2d_direct_nb: out[oc,i,j] += w[oc,c,p,q] * x[c,i+p,j+q], c, p, q ascending."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    c_out, c_in, k, _ = w.shape
    oh, ow = x.shape[1] - k + 1, x.shape[2] - k + 1
    out = np.zeros((c_out, oh, ow))
    for c in range(c_in):
        for p in range(k):
            for q in range(k):
                out += w[:, c, p, q][:, None, None] * x[c, p:p + oh, q:q + ow][None]
    return out


def direct_quantized(x, w, bits: int = 8, out_bits: int = 8):
    """quantize.py:151-160 with QuantConfig widths input=weights=bits, output_transform=out_bits."""
    return O.fake_quant(direct(O.fake_quant(x, bits), O.fake_quant(w, bits)), out_bits)
