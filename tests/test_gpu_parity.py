"""GPU parity: the sm_100a layer (through the C ABI) against the reference's golden fixtures and the
pinned CPU oracle.  Contract: integer codes of every materialised stage and the StageStat rows are
bit-exact; the fp32 output equals the reference's fp64 output rounded to fp32 (bias = 0)."""

import os

import numpy as np
import pytest

from conftest import golden_cases, load_case

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2004_11077_b200 as W  # noqa: E402
from oracle import oracle as O  # noqa: E402

PLAN = W.build_plan(4, 3, use_legendre=True)


def qc_from_bits(bits):
    return W.QuantConfig(**bits)


def run_gpu(x, w, mode, qc, pad, groups="image", bias=None):
    r = W.QuantWinogradConv(PLAN, mode, qc)
    xt = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32), device="cuda")
    wt = torch.as_tensor(np.ascontiguousarray(w, dtype=np.float32), device="cuda")
    bt = None if bias is None else torch.as_tensor(bias, dtype=torch.float32, device="cuda")
    y = r.forward(xt, wt, bias=bt, padding=pad, scale_groups=groups)
    torch.cuda.synchronize()
    return r, y


def stats_tuples(stats):
    return [(s.stage, s.bits, s.max_abs, s.scale) for s in stats]


@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: os.path.basename(p)[5:-4])
def test_golden_case_bit_exact(path):
    c = load_case(path)
    meta = c["meta"]
    qc = qc_from_bits(meta["bits"])
    pad = meta["pad"]
    x = c["x"][None]
    r, y = run_gpu(x, c["w"], meta["mode"], qc, pad)
    st = r.stats()[0]
    want = list(zip(meta["stages"], c["stat_bits"].tolist(), c["stat_max_abs"].tolist(), c["stat_scale"].tolist()))
    assert stats_tuples(st) == want
    assert np.array_equal(y[0].cpu().numpy(), c["y"].astype(np.float32))
    v = r.debug_views()
    cin, cout = c["w"].shape[1], c["w"].shape[0]
    H, Wd = c["x"].shape[1:]
    ci = c["codes_input"]
    if pad:
        ci = ci[:, pad:pad + H, pad:pad + Wd]
    assert np.array_equal(v["c0"][0].permute(2, 0, 1).cpu().numpy(), ci)
    T = v["V"].shape[1]
    vt = c["codes_input_transform"].reshape(cin, T, 36)
    assert np.array_equal(v["V"].permute(2, 1, 0).cpu().numpy(), vt)
    ht = c["codes_hadamard"].reshape(cout, T, 36)
    assert np.array_equal(v["h"].permute(2, 1, 0).cpu().numpy().astype(np.int32), ht.astype(np.int32))
    wkey = "codes_weight_base_change" if meta["mode"] == "legendre" else "codes_weight_transform"
    if wkey in c:
        assert np.array_equal(v["U"].permute(1, 2, 0).cpu().numpy(), c[wkey].reshape(cout, cin, 36))


def _kaiming(rng, cout, cin):
    return (rng.standard_normal((cout, cin, 3, 3)) * np.sqrt(2.0 / (9 * cin))).astype(np.float32)


def _compare_with_oracle(x, w, mode, qc, pad, groups, sample=None):
    r, y = run_gpu(x, w, mode, qc, pad, groups)
    n = x.shape[0]
    idx = np.arange(n) if sample is None else np.asarray(sample)
    ipg = 1 if groups == "image" else (n if groups == "batch" else int(groups))
    xs = x[idx] if groups == "image" else x
    yo, so, _ = O.quant_conv_batch(xs.astype(np.float64), w.astype(np.float64), mode,
                                   {f: getattr(qc, f) for f in O.BIT_FIELDS}, padding=pad,
                                   images_per_group=ipg)
    yg = y.cpu().numpy()
    yg = yg[idx] if groups == "image" else yg
    assert np.array_equal(yg, yo.astype(np.float32))
    st = r.stats()
    if groups == "image":
        for j, i in enumerate(idx):
            assert stats_tuples(st[i]) == [(s.stage, s.bits, s.max_abs, s.scale) for s in so[j]]
    else:
        for gi in range(n // ipg):
            assert stats_tuples(st[gi]) == [(s.stage, s.bits, s.max_abs, s.scale) for s in so[gi]]
    return r, y


def test_config1_full_batch_both_granularities():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((8, 64, 32, 32)).astype(np.float32)
    w = _kaiming(rng, 64, 64)
    for groups in ("image", "batch"):
        _compare_with_oracle(x, w, "legendre", W.QuantConfig.uniform(8), 1, groups)


@pytest.mark.parametrize("mode", ["legendre", "canonical"])
@pytest.mark.parametrize("qname", ["8b", "8b+9b"])
def test_config2(mode, qname):
    rng = np.random.default_rng(2)
    x = rng.standard_normal((128, 128, 16, 16)).astype(np.float32)
    w = _kaiming(rng, 128, 128)
    _compare_with_oracle(x, w, mode, W.QuantConfig.from_name(qname), 1, "image", sample=range(0, 128, 9))


@pytest.mark.parametrize("c,hw", [(64, 32), (128, 16), (256, 8), (512, 4)])
def test_config3_shapes(c, hw):
    rng = np.random.default_rng(3)
    x = np.maximum(rng.standard_normal((256, c, hw, hw)), 0).astype(np.float32)
    w = _kaiming(rng, c, c)
    _compare_with_oracle(x, w, "legendre", W.QuantConfig.uniform(8), 1, "image", sample=[0, 1, 77, 255])


def test_config4_sampled_images():
    rng = np.random.default_rng(0)
    n = 64  # full config-4 shape per image; per-image scales make sampled parity exact
    x = rng.standard_normal((n, 256, 56, 56)).astype(np.float32)
    w = _kaiming(rng, 256, 256)
    _compare_with_oracle(x, w, "legendre", W.QuantConfig.uniform(8), 1, "image", sample=[0, 31, 63])


@pytest.mark.parametrize("kind", ["relu", "heavy_tail", "small_integers", "sparse"])
def test_config4_shape_adverse_statistics(kind):
    """Config-4 image shape with input statistics that stress the exact paths at scale: ReLU activations,
    heavy tails (one huge value sets the scale, most codes are tiny), small integers (exact ties in every
    stage, fix lists far beyond their capacity -> inline fallbacks) and 95 % zeros."""
    rng = np.random.default_rng(44)
    n = 6
    shape = (n, 256, 56, 56)
    if kind == "relu":
        x = np.maximum(rng.standard_normal(shape), 0)
    elif kind == "heavy_tail":
        x = rng.standard_t(1.5, shape)
    elif kind == "small_integers":
        x = rng.integers(-2, 3, shape).astype(np.float64)
    else:
        x = rng.standard_normal(shape) * (rng.random(shape) < 0.05)
    w = _kaiming(rng, 256, 256) if kind != "small_integers" else np.rint(rng.standard_normal((256, 256, 3, 3))).astype(np.float32)
    _compare_with_oracle(x.astype(np.float32), w, "legendre", W.QuantConfig.uniform(8), 1, "image", sample=[0, n - 1])


@pytest.mark.parametrize("cin,cout,h,w,pad", [(3, 64, 32, 32, 1), (5, 10, 13, 14, 0), (33, 70, 9, 7, 1),
                                               (96, 200, 6, 11, 1), (1, 1, 3, 3, 0)])
@pytest.mark.parametrize("mode", ["legendre", "canonical"])
def test_ragged_shapes(cin, cout, h, w, pad, mode):
    rng = np.random.default_rng(cin * 131 + cout)
    x = rng.standard_normal((3, cin, h, w)).astype(np.float32)
    wt = rng.standard_normal((cout, cin, 3, 3)).astype(np.float32)
    _compare_with_oracle(x, wt, mode, W.QuantConfig.uniform(8, hadamard_bits=9), pad, "image")
    _compare_with_oracle(x, wt, mode, W.QuantConfig.uniform(8), pad, "batch")


@pytest.mark.parametrize("cin,cout,h,w,pad", [(8, 12, 10, 98, 1), (6, 8, 6, 138, 1), (4, 8, 22, 42, 0), (12, 8, 34, 18, 1)])
def test_wide_images_output_item_shapes(cin, cout, h, w, pad):
    """Tile rows of 25, 35, 10 and 5 tiles: every branch of the output pass's item shape (tile-row items in 1, 2
    and 4 passes, 32-tile chunks of rows wider than 32 tiles; csrc/wl_staged.cuh cw_shape), bias included."""
    rng = np.random.default_rng(cin * 7 + w)
    x = rng.standard_normal((2, cin, h, w)).astype(np.float32)
    wt = _kaiming(rng, cout, cin)
    _compare_with_oracle(x, wt, "legendre", W.QuantConfig.uniform(8), pad, "image")
    _compare_with_oracle(x, wt, "legendre", W.QuantConfig.uniform(8), pad, "batch")


@pytest.mark.parametrize("seed", range(int(os.environ.get("WL_RANDOM_SEEDS", "48"))))
def test_random_shapes_modes_widths(seed):
    """Seeded random sweep over shapes, modes, stage widths, padding, scale groups and input statistics
    (Gaussian, ReLU, heavy-tailed, small-integer inputs full of ties): every draw bit-exact against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    cin, cout = int(rng.choice([1, 3, 7, 16, 31, 40, 64, 96])), int(rng.choice([1, 5, 16, 33, 64, 72, 130]))
    h, w_ = int(rng.integers(3, 27)), int(rng.integers(3, 27))
    pad = int(rng.integers(0, 3))
    if h + 2 * pad < 3 or w_ + 2 * pad < 3:
        pad = 1
    n = int(rng.choice([1, 2, 3, 5, 6]))
    mode = str(rng.choice(["legendre", "canonical"]))
    kind = seed % 4
    if kind == 0:
        x = rng.standard_normal((n, cin, h, w_))
    elif kind == 1:
        x = np.maximum(rng.standard_normal((n, cin, h, w_)), 0)
    elif kind == 2:
        x = rng.standard_t(2, (n, cin, h, w_))
    else:
        x = rng.integers(-3, 4, (n, cin, h, w_)).astype(np.float64)
    wt = rng.standard_normal((cout, cin, 3, 3)) * (0.3 if kind != 3 else 1.0)
    if kind == 3:
        wt = np.rint(wt)
    bits = dict(input_bits=int(rng.integers(4, 9)), weight_bits=int(rng.integers(4, 9)),
                weight_transform_bits=int(rng.integers(5, 9)), input_transform_bits=int(rng.integers(5, 9)),
                hadamard_bits=int(rng.integers(6, 10)), output_transform_bits=int(rng.choice([6, 8, 10, 12, 14, 16])),
                base_change_bits=int(rng.integers(5, 9)))
    qc = W.QuantConfig(**bits)
    groups = "image" if seed % 3 else "batch"
    if seed % 5 == 0 and n > 1:
        groups = [d for d in (2, 3, 5) if n % d == 0][0]  # groups of several images
    _compare_with_oracle(x.astype(np.float32), wt.astype(np.float32), mode, qc, pad, groups)


@pytest.mark.parametrize("seed", range(int(os.environ.get("WL_RANDOM_SEEDS_WIDE", "12"))))
def test_random_wide_channels(seed):
    """Seeded draws with up to 512 channels on tiny images (the LD = 512 kernels, multi-block GEMM tiles, one-tile
    scale groups), fp32 tensors and the fp64 numpy entry point."""
    rng = np.random.default_rng(5000 + seed)
    cin, cout = int(rng.choice([130, 256, 300, 512])), int(rng.choice([65, 200, 257, 512]))
    h, w_ = int(rng.integers(3, 9)), int(rng.integers(3, 9))
    pad = int(rng.integers(0, 2))
    if h + 2 * pad < 3 or w_ + 2 * pad < 3:
        pad = 1
    n = int(rng.choice([1, 2, 4]))
    mode = str(rng.choice(["legendre", "canonical"]))
    x = rng.standard_normal((n, cin, h, w_)) if seed % 2 else np.rint(2 * rng.standard_normal((n, cin, h, w_)))
    wt = _kaiming(rng, cout, cin)
    qc = W.QuantConfig(hadamard_bits=int(rng.choice([8, 9])), output_transform_bits=int(rng.choice([8, 12, 16])))
    _compare_with_oracle(x.astype(np.float32), wt, mode, qc, pad, "image" if seed % 3 else "batch")
    if seed % 4 == 0:  # fp64 numpy call on one image: the reference's own signature and dtype
        xd, wd = x[0].astype(np.float64) * np.pi, wt.astype(np.float64) / 3
        if pad:
            xd = np.pad(xd, ((0, 0), (pad, pad), (pad, pad)))
        y, stats = W.conv2d_winograd_quantized(xd, wd, PLAN, mode, qc)
        yo, so, _ = O.quant_conv_batch(xd[None], wd, mode, {f: getattr(qc, f) for f in O.BIT_FIELDS}, padding=0)
        assert np.array_equal(np.asarray(y), yo[0])
        assert stats_tuples(stats) == [(s.stage, s.bits, s.max_abs, s.scale) for s in so[0]]


@pytest.mark.parametrize("n,ipg,c,k,h,w,pad,mode", [(6, 2, 20, 24, 9, 10, 1, "legendre"), (6, 3, 33, 70, 5, 14, 1, "canonical"),
                                                    (8, 4, 64, 64, 16, 16, 1, "legendre"), (4, 2, 256, 256, 8, 8, 1, "legendre"),
                                                    (9, 3, 8, 130, 3, 3, 2, "legendre")])
def test_groups_of_several_images(n, ipg, c, k, h, w, pad, mode):
    """Scale groups of 2-4 consecutive images (the ABI's images_per_group): tile rows of one warp / GEMM tile
    then belong to different groups."""
    rng = np.random.default_rng(n * 31 + c)
    x = (rng.standard_normal((n, c, h, w)) * rng.uniform(0.2, 5.0, (n, 1, 1, 1))).astype(np.float32)
    wt = _kaiming(rng, k, c)
    _compare_with_oracle(x, wt, mode, W.QuantConfig.from_name("8b+9b"), pad, ipg)


def test_unaligned_input_and_output_pointers():
    """x and y at 4-byte (not 16-byte) aligned addresses take the scalar load / store paths and give the same
    bits as the aligned call."""
    rng = np.random.default_rng(21)
    n, c, k, h = 3, 24, 40, 16
    x = torch.as_tensor(rng.standard_normal((n, c, h, h)).astype(np.float32), device="cuda")
    w = torch.as_tensor(_kaiming(rng, k, c), device="cuda")
    for mode in ("legendre", "canonical"):
        r = W.QuantWinogradConv(PLAN, mode, W.QuantConfig.uniform(8))
        y0 = r.forward(x, w, padding=1).clone()
        xb = torch.empty(x.numel() + 1, device="cuda")
        xu = xb[1:].view_as(x)
        xu.copy_(x)
        yb = torch.empty(y0.numel() + 3, device="cuda")
        yu = yb[3:].view_as(y0)
        assert xu.data_ptr() % 16 != 0 and yu.data_ptr() % 16 != 0
        r.forward(xu, w, padding=1, out=yu)
        torch.cuda.synchronize()
        assert torch.equal(yu, y0)


@pytest.mark.parametrize("n,groups,parts", [(6, "image", 2), (7, "image", 3), (8, 2, 2), (8, 2, 3), (12, 4, 8), (5, "image", 1)])
def test_forward_split_equals_forward(n, groups, parts):
    """forward_split (independent parts on forked streams, own workspaces) gives the bits and the StageStats of
    forward(): scale groups never straddle a part.  Also as a captured CUDA graph (the fork/join is capturable)."""
    rng = np.random.default_rng(100 + n)
    c, k, h = 24, 40, 12
    x = torch.as_tensor((rng.standard_normal((n, c, h, h)) * rng.uniform(0.3, 4.0, (n, 1, 1, 1))).astype(np.float32),
                        device="cuda")
    w = torch.as_tensor(_kaiming(rng, k, c), device="cuda")
    b = torch.as_tensor(rng.standard_normal(k).astype(np.float32), device="cuda")
    for mode in ("legendre", "canonical"):
        r = W.QuantWinogradConv(PLAN, mode, W.QuantConfig.from_name("8b+9b"))
        y0 = r.forward(x, w, bias=b, padding=1, scale_groups=groups).clone()
        s0 = r.stats()
        y1 = r.forward_split(x, w, bias=b, padding=1, scale_groups=groups, parts=parts)
        s1 = r.stats()
        torch.cuda.synchronize()
        assert torch.equal(y1, y0)
        assert s1 == s0
        y2 = torch.zeros_like(y0)
        r.forward_split(x, w, bias=b, padding=1, scale_groups=groups, parts=parts, out=y2)  # buffers for the capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            r.forward_split(x, w, bias=b, padding=1, scale_groups=groups, parts=parts, out=y2)
        y2.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(y2, y0)
    with pytest.raises(ValueError):
        r.forward_split(x, w, padding=1, scale_groups="batch")


def test_degenerate_inputs_ties_and_equal_maxima():
    rng = np.random.default_rng(5)
    cases = [np.zeros((2, 8, 8, 8)), np.ones((2, 8, 8, 8)), rng.integers(-2, 3, (2, 8, 8, 8)),
             np.broadcast_to(rng.standard_normal((1, 8, 1, 1)), (2, 8, 8, 8))]
    w = rng.integers(-1, 2, (16, 8, 3, 3)).astype(np.float32)
    for x in cases:
        x = np.ascontiguousarray(x, dtype=np.float32)
        for mode in ("canonical", "legendre"):
            _compare_with_oracle(x, w, mode, W.QuantConfig.uniform(8), 1, "image")


def test_bias_added_after_dequant():
    rng = np.random.default_rng(8)
    x = rng.standard_normal((2, 16, 12, 12)).astype(np.float32)
    w = _kaiming(rng, 24, 16)
    b = rng.standard_normal(24).astype(np.float32)
    _, y0 = run_gpu(x, w, "legendre", W.QuantConfig.uniform(8), 1)
    _, y1 = run_gpu(x, w, "legendre", W.QuantConfig.uniform(8), 1, bias=b)
    assert torch.equal(y1, y0 + torch.as_tensor(b, device="cuda")[None, :, None, None])


def test_reference_shaped_numpy_call():
    c = load_case(golden_cases()[0])
    meta = c["meta"]
    x = c["x"].astype(np.float64)
    if meta["pad"]:
        x = np.pad(x, ((0, 0), (1, 1), (1, 1)))
    y, st = W.conv2d_winograd_quantized(x, c["w"].astype(np.float64), PLAN, meta["mode"],
                                        W.QuantConfig(**meta["bits"]))
    assert y.dtype == np.float64 and y.shape == c["y"].shape
    assert np.array_equal(y, c["y"])  # fp64 in -> the reference's fp64 output, bit for bit
    assert [s.stage for s in st] == meta["stages"]


def test_determinism_bit_identical():
    rng = np.random.default_rng(9)
    x = rng.standard_normal((4, 32, 20, 20)).astype(np.float32)
    w = _kaiming(rng, 48, 32)
    for mode in ("canonical", "legendre"):
        _, a = run_gpu(x, w, mode, W.QuantConfig.uniform(8, hadamard_bits=9), 1)
        _, b = run_gpu(x, w, mode, W.QuantConfig.uniform(8, hadamard_bits=9), 1)
        assert torch.equal(a, b)


def test_identity_free_errors():
    r = W.QuantWinogradConv(PLAN, "legendre", W.QuantConfig.uniform(8))
    x = torch.zeros((1, 4, 8, 8), device="cuda")
    with pytest.raises(W.DimensionError):
        r.forward(x, torch.zeros((2, 3, 3, 3), device="cuda"))
    with pytest.raises(W.DimensionError):
        r.forward(x[0], torch.zeros((2, 4, 3, 3), device="cuda"))
    with pytest.raises(ValueError):
        W.QuantWinogradConv(PLAN, "legendre", W.QuantConfig.uniform(10)).forward(
            x, torch.zeros((2, 4, 3, 3), device="cuda"))
    with pytest.raises(ValueError):
        W.QuantWinogradConv(W.build_plan(4, 3), "legendre", W.QuantConfig.uniform(8))


def test_forward_host_chunked_equals_device_call():
    rng = np.random.default_rng(12)
    x = rng.standard_normal((10, 32, 14, 14)).astype(np.float32)
    w = _kaiming(rng, 48, 32)
    r, y = run_gpu(x, w, "legendre", W.QuantConfig.uniform(8), 1)
    xh = torch.tensor(x).pin_memory()
    yh = torch.empty(tuple(y.shape)).pin_memory()
    r.forward_host(xh, torch.tensor(w, device="cuda"), yh, padding=1, chunks=4)
    torch.cuda.synchronize()
    assert torch.equal(yh, y.cpu())


def test_weight_cache_not_fooled_by_recycled_address():
    """A fresh weight tensor allocated at a freed tensor's address must not hit the weight cache."""
    rng = np.random.default_rng(13)
    x = torch.tensor(rng.standard_normal((2, 8, 10, 10)), dtype=torch.float32, device="cuda")
    r = W.QuantWinogradConv(PLAN, "legendre", W.QuantConfig.uniform(8))
    for t in range(4):
        w64 = torch.tensor(rng.standard_normal((6, 8, 3, 3)), dtype=torch.float64, device="cuda")
        y = r.forward(x, w64.float(), padding=1)   # temporary fp32 weights, freed after the call
        fresh = W.QuantWinogradConv(PLAN, "legendre", W.QuantConfig.uniform(8)).forward(x, w64.float(), padding=1)
        assert torch.equal(y, fresh), t


@pytest.mark.parametrize("mode", ["legendre", "canonical"])
@pytest.mark.parametrize("qname", ["8b", "8b+9b"])
def test_fp64_boundary_bit_exact_arbitrary_doubles(mode, qname):
    """fp64 operands (not fp32-representable): codes, stats and the fp64 output equal the oracle's."""
    rng = np.random.default_rng(21)
    x = rng.standard_normal((3, 7, 13, 14)) * 3.7
    w = rng.standard_normal((5, 7, 3, 3))
    qc = W.QuantConfig.from_name(qname)
    r = W.QuantWinogradConv(PLAN, mode, qc)
    for pad in (0, 1):
        y = r.forward(torch.tensor(x, device="cuda"), torch.tensor(w, device="cuda"), padding=pad)
        assert y.dtype == torch.float64
        yo, so, _ = O.quant_conv_batch(x, w, mode, {f: getattr(qc, f) for f in O.BIT_FIELDS}, padding=pad,
                                       images_per_group=1)
        assert np.array_equal(y.cpu().numpy(), yo)
        for i, st in enumerate(r.stats()):
            assert stats_tuples(st) == [(s.stage, s.bits, s.max_abs, s.scale) for s in so[i]]


def test_fp64_numpy_call_equals_oracle_single_image():
    rng = np.random.default_rng([424242, 3])
    x = rng.standard_normal((3, 13, 14))
    w = rng.standard_normal((2, 3, 3, 3))
    for mode in ("canonical", "legendre"):
        y, st = W.conv2d_winograd_quantized(x, w, PLAN, mode, W.QuantConfig.uniform(8, hadamard_bits=9))
        yo, so = O.conv2d_winograd_quantized(x, w, mode, O.uniform_bits(8, 9))
        assert np.array_equal(y, yo)
        assert stats_tuples(st) == [(s.stage, s.bits, s.max_abs, s.scale) for s in so]


@pytest.mark.parametrize("cap", [1, 7])
@pytest.mark.parametrize("mode", ["legendre", "canonical"])
def test_fix_list_overflow_falls_back_inline(cap, mode):
    """Deferred exact-fix and finalize-candidate lists of capacity 1 / 7 overflow on every stage, so
    the producers' inline fallbacks (exact int64 recompute, fp64 tie replay) run instead of the fixup
    kernels: outputs and stage statistics are unchanged and still equal the oracle."""
    rng = np.random.default_rng(40 + cap)
    ints = rng.integers(-2, 3, (3, 24, 12, 12)).astype(np.float32)   # tie-heavy
    x = rng.standard_normal((3, 40, 13, 14)).astype(np.float32)
    wi = rng.integers(-1, 2, (32, 24, 3, 3)).astype(np.float32)
    w = _kaiming(rng, 36, 40)
    lib = W._lib.lib()
    try:
        lib.wl_debug_set_fix_cap(cap)
        for qc in (W.QuantConfig.uniform(8), W.QuantConfig.uniform(8, hadamard_bits=9)):
            _compare_with_oracle(ints, wi, mode, qc, 1, "image")
            _compare_with_oracle(x, w, mode, qc, 1, "batch")
    finally:
        lib.wl_debug_set_fix_cap(0)


@pytest.mark.parametrize("mode", ["legendre", "canonical"])
def test_batch_scale_groups_config2_shape(mode):
    """One scale per stage over the whole call (scale_groups="batch") at the config-2 shape."""
    rng = np.random.default_rng(22)
    x = rng.standard_normal((128, 128, 16, 16)).astype(np.float32)
    w = _kaiming(rng, 128, 128)
    _compare_with_oracle(x, w, mode, W.QuantConfig.from_name("8b+9b"), 1, "batch")


def test_batch_scale_groups_config3c_shape():
    rng = np.random.default_rng(23)
    x = np.maximum(rng.standard_normal((256, 256, 8, 8)), 0).astype(np.float32)
    w = _kaiming(rng, 256, 256)
    _compare_with_oracle(x, w, "legendre", W.QuantConfig.uniform(8), 1, "batch")


def test_forward_host_back_to_back_calls_do_not_race():
    """Two forward_host calls on different inputs with no synchronisation in between (the pooled
    device buffers are reused): each result equals its own device call."""
    rng = np.random.default_rng(24)
    xa = rng.standard_normal((12, 64, 20, 20)).astype(np.float32)
    xb = rng.standard_normal((12, 64, 20, 20)).astype(np.float32) * 2.5
    w = _kaiming(rng, 64, 64)
    r = W.QuantWinogradConv(PLAN, "legendre", W.QuantConfig.uniform(8))
    wt = torch.tensor(w, device="cuda")
    ya = r.forward(torch.tensor(xa, device="cuda"), wt, padding=1).cpu()
    yb = r.forward(torch.tensor(xb, device="cuda"), wt, padding=1).cpu()
    xha, xhb = torch.tensor(xa).pin_memory(), torch.tensor(xb).pin_memory()
    for chunks in (1, 2, 3):
        yha, yhb = torch.empty_like(ya).pin_memory(), torch.empty_like(yb).pin_memory()
        r.forward_host(xha, wt, yha, padding=1, chunks=chunks)
        r.forward_host(xhb, wt, yhb, padding=1, chunks=chunks)
        r.forward_host(xha, wt, yha, padding=1, chunks=chunks)
        torch.cuda.synchronize()
        assert torch.equal(yha, ya) and torch.equal(yhb, yb), chunks


def test_training_forward_saved_block_equals_forward():
    """wl_forward_train (stage slots + V codes in a separate saved buffer) gives the same output and
    statistics as wl_forward, and backward from the saved block equals backward from the workspace."""
    rng = np.random.default_rng(25)
    x = torch.tensor(np.maximum(rng.standard_normal((6, 40, 12, 12)), 0), dtype=torch.float32, device="cuda")
    w = torch.tensor(_kaiming(rng, 48, 40), device="cuda")
    dy = torch.tensor(rng.standard_normal((6, 48, 12, 12)), dtype=torch.float32, device="cuda")
    for mode in ("legendre", "canonical"):
        r = W.QuantWinogradConv(PLAN, mode, W.QuantConfig.uniform(8))
        y0 = r.forward(x, w, padding=1)
        st0 = r.stats()
        shape, cache, ws, _ = r._last
        g0 = r.backward(dy, shape, cache, ws, True)
        sv_bytes, ws_bytes = r.train_sizes(shape)
        assert ws_bytes < r.workspace_bytes(shape)
        saved = torch.empty(sv_bytes, dtype=torch.uint8, device="cuda")
        y1 = r.forward(x, w, padding=1, saved=saved)
        assert torch.equal(y0, y1)
        assert [stats_tuples(s) for s in r.stats()] == [stats_tuples(s) for s in st0]
        g1 = r.backward(dy, shape, cache, saved, True)
        for a, b in zip(g0, g1):
            assert torch.equal(a, b)
