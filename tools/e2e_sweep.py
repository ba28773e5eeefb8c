"""Config-4 end-to-end (pinned host x -> forward -> pinned host y) time vs chunk count / buffer depth."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_11077_b200 as W  # noqa: E402

dev = torch.device("cuda", 0)
n, c, hw = 1024, 256, 56
w = torch.randn((c, c, 3, 3), device=dev) * float(np.sqrt(2.0 / (9 * c)))
r = W.QuantWinogradConv(W.build_plan(4, 3, use_legendre=True), "legendre", W.QuantConfig.uniform(8), dev)
xh = torch.empty((n, c, hw, hw), dtype=torch.float32, pin_memory=True).normal_()
yh = torch.empty((n, c, hw, hw), dtype=torch.float32, pin_memory=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for chunks in [int(a) for a in sys.argv[1:]] or [8, 16, 32, 64]:
    for depth in (2, 3, 4):
        r.forward_host(xh, w, yh, padding=1, chunks=chunks, depth=depth)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            r.forward_host(xh, w, yh, padding=1, chunks=chunks, depth=depth)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"chunks {chunks:3d} depth {depth}: {ms:7.2f} ms  {n / ms * 1e3:8.0f} img/s", flush=True)
        r._pool = None
        r._pool_key = None
        torch.cuda.empty_cache()
