"""GPU: straight-through-estimator backward through the C ABI (wl_backward) against the fp64
closed form fed by the pinned oracle's quantised operands (oracle/backward_ref.py, itself checked
against torch fp64 autograd on CPU).  Tolerance: relative L2 error <= 1e-5 (fp32 GEMMs and
transforms vs fp64)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2004_11077_b200 as W  # noqa: E402
from oracle import backward_ref as BR  # noqa: E402
from oracle import oracle as O  # noqa: E402

PLAN = W.build_plan(4, 3, use_legendre=True)
TOL = 1e-5


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-30))


def run(x, w, dy, mode, qc, pad, bias=True):
    layer_w = torch.tensor(w, device="cuda", requires_grad=True)
    b = torch.zeros(w.shape[0], device="cuda", requires_grad=True) if bias else None
    xt = torch.tensor(x, device="cuda", requires_grad=True)
    r = W.QuantWinogradConv(PLAN, mode, qc)
    y = W.winograd_conv2d(xt, layer_w, b, r, pad)
    y.backward(torch.tensor(dy, device="cuda"))
    torch.cuda.synchronize()
    return y, xt.grad.cpu().numpy(), layer_w.grad.cpu().numpy(), (b.grad.cpu().numpy() if bias else None)


@pytest.mark.parametrize("mode", ["legendre", "canonical"])
@pytest.mark.parametrize("n,c,k,hw,pad", [(4, 16, 24, 12, 1), (2, 3, 64, 32, 1), (3, 33, 10, 9, 0),
                                          (256, 64, 64, 32, 1)])
def test_backward_matches_fp64_closed_form(mode, n, c, k, hw, pad):
    rng = np.random.default_rng(n * 7 + c)
    x = np.maximum(rng.standard_normal((n, c, hw, hw)), 0).astype(np.float32)
    w = (rng.standard_normal((k, c, 3, 3)) * np.sqrt(2 / (9 * c))).astype(np.float32)
    ho = hw + 2 * pad - 2
    dy = rng.standard_normal((n, k, ho, ho)).astype(np.float32)
    qc = W.QuantConfig.uniform(8)
    y, dx, dw, db = run(x, w, dy, mode, qc, pad)
    sample = slice(0, min(n, 8))  # per-image scales: the oracle may use any subset of images for dx
    U, V = BR.quantised_operands(x[sample].astype(np.float64), w.astype(np.float64), mode,
                                 {f: getattr(qc, f) for f in O.BIT_FIELDS}, pad)
    dx_r, _, _ = BR.ste_formula(dy[sample].astype(np.float64), U, V, hw, hw, pad)
    assert rel(dx[sample], dx_r) <= TOL
    if n <= 8:
        _, dw_r, db_r = BR.ste_formula(dy.astype(np.float64), U, V, hw, hw, pad)
        assert rel(dw, dw_r) <= TOL
        assert rel(db, db_r) <= TOL


def test_module_training_step_runs_and_learns():
    torch.manual_seed(0)
    m = W.WinogradAwareConv2d(8, 8, bias=True).cuda()
    x = torch.randn(4, 8, 16, 16, device="cuda")
    target = torch.randn(4, 8, 16, 16, device="cuda")
    opt = torch.optim.SGD(m.parameters(), lr=0.05, momentum=0.9)
    losses = []
    for _ in range(8):
        opt.zero_grad()
        loss = torch.nn.functional.mse_loss(m(x), target)
        loss.backward()
        opt.step()
        losses.append(float(loss.detach()))
    assert all(np.isfinite(losses)) and losses[-1] < losses[0]
