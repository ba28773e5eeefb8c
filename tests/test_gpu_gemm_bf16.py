"""GPU: the split-bf16 tcgen05 GEMM (gemm_bf16.cuh) behind the STE backward and the float Winograd
path, through its C-ABI test hook, against an fp64 torch matmul of the same fp32 operands.
Operands are split into bf16 planes hi + mid + lo (exact for fp32); quantised-code operands are one
plane.  Tolerance: relative L2 <= 8e-6 per split of <= 4096 (fp32 tensor-core accumulation)."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2004_11077_b200 import _lib  # noqa: E402


def planes(x, p):
    """[batch, rows, Kd] fp32 -> [p, batch, rows, Kd] bf16 with sum == x (p = 3) or bf16(x) (p = 1)."""
    out, r = [], x
    for _ in range(p):
        h = r.to(torch.bfloat16)
        out.append(h)
        r = r - h.float()
    return torch.stack(out).contiguous()


def run(A, PA, B, PB, ks, alpha=1.0):
    batch, M, Kd = A.shape[-3:]
    N = B.shape[-2]
    S = -(-Kd // ks)
    D = torch.full((S, batch, M, N), float("nan"), device="cuda")
    _lib.check(_lib.lib().wl_debug_gemm_bf16(
        ctypes.c_void_p(A.data_ptr()), PA, ctypes.c_void_p(B.data_ptr()), PB, batch, M, N, Kd, ks,
        ctypes.c_void_p(D.data_ptr()), N, alpha, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
        "wl_debug_gemm_bf16")
    torch.cuda.synchronize()
    return D


def rel(a, b):
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


@pytest.mark.parametrize("M,N,Kd,ks,PA,PB", [
    (128, 64, 64, 64, 3, 1), (200, 3, 64, 64, 3, 1), (1000, 256, 256, 256, 3, 1), (333, 512, 128, 128, 3, 1),
    (64, 64, 4096, 1024, 1, 3), (3, 64, 1024, 256, 1, 3), (512, 512, 2048, 512, 1, 3),
    (777, 200, 192, 192, 3, 3), (128, 16, 64, 64, 1, 1)])
def test_split_gemm_matches_fp64(M, N, Kd, ks, PA, PB):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    batch = 36
    a = torch.randn((batch, M, Kd), generator=g, device="cuda")
    b = torch.randn((batch, N, Kd), generator=g, device="cuda")
    if PA == 1:
        a = torch.randint(-127, 128, a.shape, generator=g, device="cuda").float()
    if PB == 1:
        b = torch.randint(-127, 128, b.shape, generator=g, device="cuda").float()
    D = run(planes(a, PA), PA, planes(b, PB), PB, ks, alpha=0.5)
    S = D.shape[0]
    for s in range(S):
        sl = slice(s * ks, min(Kd, (s + 1) * ks))
        ref = 0.5 * torch.einsum("bmk,bnk->bmn", a[..., sl].double(), b[..., sl].double())
        assert not torch.isnan(D[s]).any()
        assert rel(D[s].double(), ref) <= 8e-6, s
