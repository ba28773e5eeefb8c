"""Small driver for ncu captures: forward + STE backward of one layer shape."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_11077_b200 as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--c", type=int, default=64)
ap.add_argument("--hw", type=int, default=32)
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
torch.manual_seed(0)
m = W.WinogradAwareConv2d(a.c, a.c).cuda()
x = torch.randn(a.n, a.c, a.hw, a.hw, device="cuda", requires_grad=True)
for _ in range(a.iters):
    y = m(x)
    y.backward(torch.ones_like(y))
torch.cuda.synchronize()
print("ok")
