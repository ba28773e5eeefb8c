"""Debug helper: compare every materialised GPU stage with the oracle capture for one shape."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2004_11077_b200 as W
from oracle import oracle as O

n, c, hw, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
rng = np.random.default_rng(3)
x = np.maximum(rng.standard_normal((n, c, hw, hw)), 0).astype(np.float32)
w = (rng.standard_normal((c, c, 3, 3)) * np.sqrt(2 / (9 * c))).astype(np.float32)
r = W.QuantWinogradConv(W.build_plan(4, 3, use_legendre=True), mode, W.QuantConfig.uniform(8))
y = r.forward(torch.tensor(x, device="cuda"), torch.tensor(w, device="cuda"), padding=1)
torch.cuda.synchronize()
st = r.stats()
v = r.debug_views()
idx = [0, 1, n - 1]
yo, so, cap = O.quant_conv_batch(x[idx].astype(np.float64), w.astype(np.float64), mode, O.uniform_bits(8), padding=1, capture=True)
T = v["V"].shape[1]; TP = T // n
for j, i in enumerate(idx):
    print("image", i)
    for a, b in zip(st[i], so[j]):
        print("  ", a.stage, a.max_abs == b.max_abs, a.max_abs, b.max_abs)
    Vg = v["V"][:, i * TP:(i + 1) * TP, :].permute(2, 1, 0).cpu().numpy()
    Vo = cap["input_transform"][j].reshape(c, TP, 36)
    print("  V mism", (Vg != Vo).sum())
    hg = v["h"][:, i * TP:(i + 1) * TP, :].permute(2, 1, 0).cpu().numpy().astype(np.int32)
    ho = cap["hadamard"][j].reshape(c, TP, 36)
    print("  h mism", (hg != ho).sum(), "of", ho.size)
    print("  y mism", (y[i].cpu().numpy() != yo[j].astype(np.float32)).sum())
