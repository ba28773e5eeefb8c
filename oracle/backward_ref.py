"""TEST INFRASTRUCTURE ONLY — fp64 oracles for the straight-through-estimator backward.

The reference has no backward ("parity unpinned by the reference").  Two
independent fp64 restatements pin the B200 backward instead:

* ``ste_autograd``: the staged quantized pipeline of reference pipeline.py:106-158 written in torch
  fp64 with every cast as ``t + (fake_quant(t) - t).detach()`` (quantize.py:112-126 semantics,
  scales detached) and differentiated by autograd;
* ``ste_formula``: the closed form the CUDA path implements — dM = A dY A^T, dV = sum_k U (.) dM,
  dU = sum_t V (.) dM, dX = col2im(B dV B^T), dW = G^T dU G — evaluated in numpy fp64 from the
  quantised operands (dequantised U and V codes).

tests/test_backward_oracle.py checks the two against each other on CPU; the GPU tests compare the
sm_100a backward with ``ste_formula`` fed by the pinned C oracle's codes.
"""

from __future__ import annotations

import numpy as np

from . import plan_ref
from .oracle import quant_conv_batch

_EP = plan_ref.exact_plan(4, 3)
A = plan_ref.to_f64(plan_ref.transpose(_EP["AT"]))   # 6 x 4
BT = plan_ref.to_f64(_EP["BT"])                      # 6 x 6
G = plan_ref.to_f64(_EP["G"])                        # 6 x 3


def _tiles_geometry(h, w, pad):
    ho, wo = h + 2 * pad - 2, w + 2 * pad - 2
    th, tw = -(-ho // 4), -(-wo // 4)
    return ho, wo, th, tw


def ste_formula(dy, U, V, h, w, pad):
    """dy [n,K,Ho,Wo]; U [K,C,6,6] dequantised; V [n,C,T,6,6] dequantised -> (dx, dw, db) fp64."""
    n, K, ho, wo = dy.shape
    C = U.shape[1]
    _, _, th, tw = _tiles_geometry(h, w, pad)
    dyp = np.zeros((n, K, th * 4, tw * 4))
    dyp[:, :, :ho, :wo] = dy
    tiles = dyp.reshape(n, K, th, 4, tw, 4).transpose(0, 1, 2, 4, 3, 5).reshape(n, K, th * tw, 4, 4)
    dM = np.einsum("ia,nktab,jb->nktij", A, tiles, A)
    dV = np.einsum("kcij,nktij->nctij", U, dM)
    dU = np.einsum("nctij,nktij->kcij", V, dM)
    dXt = np.einsum("ai,nctab,bj->nctij", BT, dV, BT)  # B dV B^T with B = BT^T
    hp, wp = (th - 1) * 4 + 6, (tw - 1) * 4 + 6
    dxp = np.zeros((n, C, max(hp, h + 2 * pad), max(wp, w + 2 * pad)))
    for ty in range(th):
        for tx in range(tw):
            dxp[:, :, 4 * ty:4 * ty + 6, 4 * tx:4 * tx + 6] += dXt[:, :, ty * tw + tx]
    dx = dxp[:, :, pad:pad + h, pad:pad + w]
    dw = np.einsum("ap,kcab,bq->kcpq", G, dU, G)
    db = dy.sum(axis=(0, 2, 3))
    return dx, dw, db


def _deq(codes, st):
    q = 2 ** (st.bits - 1) - 1
    out = codes.astype(np.float64) * st.scale
    out[codes == q] = st.max_abs
    out[codes == -q] = -st.max_abs
    return out


def quantised_operands(x, w, mode, bits, pad, images_per_group=1):
    """Dequantised U [K,C,6,6] and V [n,C,T,6,6] as the (pinned) C oracle quantises them."""
    _, st, cap = quant_conv_batch(x, w, mode, bits, padding=pad, images_per_group=images_per_group, capture=True)
    wname = "weight_base_change" if mode == "legendre" else "weight_transform"
    names = [s.stage for s in st[0]]
    U = _deq(cap[wname], st[0][names.index(wname)])
    V = np.empty(cap["input_transform"].shape)
    for g in range(len(st)):
        sl = slice(g * images_per_group, (g + 1) * images_per_group)
        V[sl] = _deq(cap["input_transform"][sl], st[g][names.index("input_transform")])
    return U, V


def ste_autograd(x, w, mode, bits, pad, dy):
    """torch fp64 autograd of the staged pipeline with straight-through casts (one scale group)."""
    import torch

    ep = _EP
    f = lambda M: torch.tensor(plan_ref.to_f64(M), dtype=torch.float64)  # noqa: E731
    Gm, BTm, ATm = f(ep["G"]), f(ep["BT"]), f(ep["AT"])
    Pinv = f(ep["Pinv"])
    G_P, BPT, APT = f(ep["G_P"]), f(ep["BPT"]), f(ep["APT"])

    def cast(t, b):
        q = 2 ** (b - 1) - 1
        m = t.detach().abs().max()
        if m == 0:
            return t
        s = m / q
        c = torch.clamp(torch.round(t.detach() / s), -q, q)
        v = c * s
        v = torch.where(c == q, m, torch.where(c == -q, -m, v))
        return t + (v - t).detach()

    xt = torch.tensor(np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad))), dtype=torch.float64, requires_grad=True)
    wt = torch.tensor(w, dtype=torch.float64, requires_grad=True)
    n, C, H, W = xt.shape
    K = wt.shape[0]
    ho, wo = H - 2, W - 2
    th, tw = -(-ho // 4), -(-wo // 4)
    xq = cast(xt, bits["input_bits"])
    wq = cast(wt, bits["weight_bits"])
    hp, wp = (th - 1) * 4 + 6, (tw - 1) * 4 + 6
    xp = torch.zeros((n, C, hp, wp), dtype=torch.float64)
    xp = xp + torch.nn.functional.pad(xq, (0, wp - W, 0, hp - H))[:, :, :hp, :wp]
    tiles = xp.unfold(2, 6, 4).unfold(3, 6, 4).reshape(n, C, th * tw, 6, 6)
    if mode == "canonical":
        U = cast(Gm @ wq @ Gm.T, bits["weight_transform_bits"])
        V = cast(BTm @ tiles @ BTm.T, bits["input_transform_bits"])
    else:
        U = cast(G_P @ wq @ G_P.T, bits["weight_transform_bits"])
        U = cast(Pinv @ U @ Pinv.T, bits["base_change_bits"])
        V = cast(Pinv.T @ tiles @ Pinv, bits["base_change_bits"])
        V = cast(BPT @ V @ BPT.T, bits["input_transform_bits"])
    acc = torch.einsum("kcij,nctij->nktij", U, V)
    acc = cast(acc, bits["hadamard_bits"])
    if mode == "canonical":
        yt = ATm @ acc @ ATm.T
    else:
        mid = cast(Pinv.T @ acc @ Pinv, bits["base_change_bits"])
        yt = APT @ mid @ APT.T
    y = yt.reshape(n, K, th, tw, 4, 4).permute(0, 1, 2, 4, 3, 5).reshape(n, K, th * 4, tw * 4)[:, :, :ho, :wo]
    y = cast(y, bits["output_transform_bits"])
    y.backward(torch.tensor(dy, dtype=torch.float64))
    dx = xt.grad.numpy()[:, :, pad:pad + x.shape[2], pad:pad + x.shape[3]]
    return y.detach().numpy(), dx, wt.grad.numpy(), U.detach().numpy(), V.detach().numpy()
