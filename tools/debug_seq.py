import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2004_11077_b200 as W
from conftest import load_case, golden_cases
names = sys.argv[1].split(",")
for nm in names:
    p = [q for q in golden_cases() if nm in q][0]
    c = load_case(p)
    meta = c["meta"]
    r = W.QuantWinogradConv(W.build_plan(4, 3, use_legendre=True), meta["mode"], W.QuantConfig(**meta["bits"]))
    y = r.forward(torch.tensor(c["x"][None], device="cuda"), torch.tensor(c["w"], device="cuda"), padding=meta["pad"])
    torch.cuda.synchronize()
    print(nm, "ok", np.array_equal(y[0].cpu().numpy(), c["y"].astype(np.float32)), flush=True)
