"""Deferred-unit (fix list) counts of one config-4-shaped forward: python tools/fix_counts.py [N]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2004_11077_b200 as W  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    dev = torch.device("cuda", 0)
    c, hw = 256, 56
    torch.manual_seed(0)
    x = torch.randn((n, c, hw, hw), device=dev)
    w = torch.randn((c, c, 3, 3), device=dev) * float(np.sqrt(2.0 / (9 * c)))
    r = W.QuantWinogradConv(W.build_plan(4, 3, use_legendre=True), "legendre", W.QuantConfig.from_name("8b"), dev)
    r.forward(x, w, padding=1)
    torch.cuda.synchronize()
    shape, cache, ws, whole = r._last
    T = n * 14 * 14
    units = T * c
    cap = max(4096, units // 16)
    size = (64 + 4 * max(cap, 4096) + 255) // 256 * 256
    cnt = ws[ws.numel() - size: ws.numel() - size + 64].view(torch.int32).cpu().numpy()
    print("units", units, "cap", cap, "counters", cnt[:8].tolist(), "fraction", (cnt[:8] / units).round(5).tolist())


if __name__ == "__main__":
    main()
