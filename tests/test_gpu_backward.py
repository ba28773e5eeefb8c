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


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("WL_RANDOM_SEEDS_BWD", "12"))))
def test_backward_random_shapes(seed):
    """Seeded random shapes (ragged, non-square, C / K not multiples of the MMA tiles, padding 0..2, both modes,
    8b and 8b+9b): dx, dW, db against the fp64 closed form."""
    rng = np.random.default_rng(7000 + seed)
    n, c, k = int(rng.choice([1, 2, 5])), int(rng.choice([1, 3, 17, 48, 64, 100])), int(rng.choice([1, 6, 33, 64, 130]))
    h, w_ = int(rng.integers(3, 21)), int(rng.integers(3, 21))
    pad = int(rng.integers(0, 3))
    if h + 2 * pad < 3 or w_ + 2 * pad < 3:
        pad = 1
    mode = str(rng.choice(["legendre", "canonical"]))
    x = rng.standard_normal((n, c, h, w_)).astype(np.float32)
    w = (rng.standard_normal((k, c, 3, 3)) * np.sqrt(2 / (9 * c))).astype(np.float32)
    ho, wo = h + 2 * pad - 2, w_ + 2 * pad - 2
    dy = rng.standard_normal((n, k, ho, wo)).astype(np.float32)
    qc = W.QuantConfig.from_name("8b+9b" if seed % 2 else "8b")
    y, dx, dw, db = run(x, w, dy, mode, qc, pad)
    U, V = BR.quantised_operands(x.astype(np.float64), w.astype(np.float64), mode,
                                 {f: getattr(qc, f) for f in O.BIT_FIELDS}, pad)
    dx_r, dw_r, db_r = BR.ste_formula(dy.astype(np.float64), U, V, h, w_, pad)
    assert rel(dx, dx_r) <= TOL
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


def test_graphed_training_step_equals_eager_forward_and_updates():
    """make_graphed_step: the loss of a replay is the eager loss of the same state (the forward is
    deterministic), and the replay updates the weights."""
    from paper_2004_11077_b200 import training as TR
    torch.manual_seed(1)
    dev = torch.device("cuda")
    m = TR.ResNet18(TR.winograd_conv_factory("legendre")).to(dev)
    opt = TR.make_optimizer(m, lr=0.01)
    x, y = TR.synthetic_batch(32, 0, seed=3, device=dev)
    step = TR.make_graphed_step(m, opt, x, y, warmup=2)
    for _ in range(2):
        ref = TR.ResNet18(TR.winograd_conv_factory("legendre")).to(dev)
        ref.load_state_dict(m.state_dict())
        ref.train()
        with torch.no_grad():
            l_ref = float(torch.nn.functional.cross_entropy(ref(x), y))
        w_before = m.stem.weight.detach().clone()
        l = float(step())
        torch.cuda.synchronize()
        assert abs(l - l_ref) <= 1e-6 * max(1.0, abs(l_ref)), (l, l_ref)
        assert not torch.equal(w_before, m.stem.weight.detach())
    TR.invalidate_weight_caches(m)


def _deq_t(codes, qmax, maxabs, scale):
    """Dequantised value as the reference holds it after fake_quant (quantize.py:120-125)."""
    c = codes.double()
    v = c * scale
    v = torch.where(c == qmax, torch.full_like(v, maxabs), v)
    return torch.where(c == -qmax, torch.full_like(v, -maxabs), v)


def _ste_torch(dy, U, V, h, w, pad):
    """ste_formula (oracle/backward_ref.py) in torch fp64 on the device: dy [n,K,Ho,Wo], U [K,C,6,6],
    V [n,C,TP,6,6] dequantised -> (dx, dw, db)."""
    A = torch.tensor(BR.A, dtype=torch.float64, device=dy.device)
    BT = torch.tensor(BR.BT, dtype=torch.float64, device=dy.device)
    G = torch.tensor(BR.G, dtype=torch.float64, device=dy.device)
    n, K, ho, wo = dy.shape
    C = U.shape[1]
    th, tw = -(-ho // 4), -(-wo // 4)
    dyp = torch.zeros((n, K, th * 4, tw * 4), dtype=torch.float64, device=dy.device)
    dyp[:, :, :ho, :wo] = dy
    tiles = dyp.reshape(n, K, th, 4, tw, 4).permute(0, 1, 2, 4, 3, 5).reshape(n, K, th * tw, 4, 4)
    dM = torch.einsum("ia,nktab,jb->nktij", A, tiles, A)
    dV = torch.einsum("kcij,nktij->nctij", U, dM)
    dU = torch.einsum("nctij,nktij->kcij", V, dM)
    dXt = torch.einsum("ai,nctab,bj->nctij", BT, dV, BT)
    hp, wp = (th - 1) * 4 + 6, (tw - 1) * 4 + 6
    dxp = torch.zeros((n, C, max(hp, h + 2 * pad), max(wp, w + 2 * pad)), dtype=torch.float64, device=dy.device)
    for ty in range(th):
        for tx in range(tw):
            dxp[:, :, 4 * ty:4 * ty + 6, 4 * tx:4 * tx + 6] += dXt[:, :, ty * tw + tx]
    dx = dxp[:, :, pad:pad + h, pad:pad + w]
    dw = torch.einsum("ap,kcab,bq->kcpq", G, dU, G)
    return dx, dw, dy.sum(dim=(0, 2, 3))


@pytest.mark.parametrize("mode", ["legendre", "canonical"])
@pytest.mark.parametrize("c,hw", [(64, 32), (128, 16), (256, 8), (512, 4)])
def test_backward_config3_full_batch_dx_dw_db(mode, c, hw):
    """Config 3 at its full batch (N=256, every ResNet-18 3x3 shape): dx, dw and db against the fp64
    closed form over ALL images.  The quantised operands are the layer's own U / V codes and stage
    scales (their bit-exactness against the reference is tests/test_gpu_parity.py's job)."""
    n, pad = 256, 1
    rng = np.random.default_rng(c + hw)
    x = np.maximum(rng.standard_normal((n, c, hw, hw)), 0).astype(np.float32)
    w = (rng.standard_normal((c, c, 3, 3)) * np.sqrt(2 / (9 * c))).astype(np.float32)
    dy = rng.standard_normal((n, c, hw, hw)).astype(np.float32)
    qc = W.QuantConfig.uniform(8)
    y, dx, dw, db = run(x, w, dy, mode, qc, pad)
    r = W.QuantWinogradConv(PLAN, mode, qc)
    y2 = r.forward(torch.tensor(x, device="cuda"), torch.tensor(w, device="cuda"), padding=pad)
    assert torch.equal(y, y2)
    views, st = r.debug_views(), r.stats()
    names = [s.stage for s in st[0]]
    wi, vi = names.index("weight_base_change" if mode == "legendre" else "weight_transform"), names.index("input_transform")
    su, qmax = st[0][wi], 127
    U = _deq_t(views["U"], qmax, su.max_abs, su.scale).permute(1, 2, 0).reshape(c, c, 6, 6)
    TP = views["V"].shape[1] // n
    Vc = views["V"].reshape(36, n, TP, c)
    vmax = torch.tensor([s[vi].max_abs for s in st], dtype=torch.float64, device="cuda")[None, :, None, None]
    vsc = torch.tensor([s[vi].scale for s in st], dtype=torch.float64, device="cuda")[None, :, None, None]
    cd = Vc.double()
    Vd = torch.where(cd == qmax, vmax.expand_as(cd), torch.where(cd == -qmax, -vmax.expand_as(cd), cd * vsc))
    V = Vd.permute(1, 3, 2, 0).reshape(n, c, TP, 6, 6)
    dx_r, dw_r, db_r = (t.cpu().numpy() for t in _ste_torch(torch.tensor(dy, dtype=torch.float64, device="cuda"),
                                                             U, V, hw, hw, pad))
    assert rel(dx, dx_r) <= TOL
    assert rel(dw, dw_r) <= TOL
    assert rel(db, db_r) <= TOL
