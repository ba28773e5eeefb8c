"""Run one golden case through the GPU layer (for bisecting with WL_DEBUG_SYNC=1)."""
import sys

import numpy as np
import torch

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import paper_2004_11077_b200 as W  # noqa: E402
from conftest import load_case  # noqa: E402

c = load_case(f"tests/golden/case_{sys.argv[1]}.npz")
meta = c["meta"]
r = W.QuantWinogradConv(W.build_plan(4, 3, use_legendre=True), meta["mode"], W.QuantConfig(**meta["bits"]))
x = torch.tensor(c["x"][None], dtype=torch.float32, device="cuda")
w = torch.tensor(c["w"], dtype=torch.float32, device="cuda")
try:
    y = r.forward(x, w, padding=meta["pad"])
    torch.cuda.synchronize()
    print("ok", np.array_equal(y[0].cpu().numpy(), c["y"].astype(np.float32)))
except Exception as e:  # noqa: BLE001
    print("fail", e)
