"""Small driver for ncu captures: a few forwards of the config-4 layer shape at reduced batch."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_11077_b200 as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--c", type=int, default=256)
ap.add_argument("--hw", type=int, default=56)
ap.add_argument("--mode", default="legendre")
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
torch.manual_seed(0)
x = torch.randn(a.n, a.c, a.hw, a.hw, device="cuda")
w = torch.randn(a.c, a.c, 3, 3, device="cuda") * (2.0 / (9 * a.c)) ** 0.5
r = W.QuantWinogradConv(W.build_plan(4, 3, use_legendre=True), a.mode, W.QuantConfig.uniform(8))
for _ in range(a.iters):
    y = r.forward(x, w, padding=1)
torch.cuda.synchronize()
print("ok", float(y.abs().sum()))
