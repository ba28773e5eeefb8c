"""GPU box: graphed forward time of the launch-bound shapes with the deferred-fix lists on (default) and with a
one-entry list (wl_debug_set_fix_cap(1): every producer fixes its units inline, the fixup kernels find nothing)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_11077_b200 as W  # noqa: E402
from paper_2004_11077_b200 import _lib  # noqa: E402

plan = W.build_plan(4, 3, use_legendre=True)
for n, c, hw in [(8, 64, 32), (128, 128, 16), (256, 64, 32), (256, 128, 16), (256, 256, 8), (256, 512, 4)]:
    for cap in (0, 1):
        _lib.lib().wl_debug_set_fix_cap(cap)
        torch.manual_seed(0)
        x = torch.randn(n, c, hw, hw, device="cuda")
        w = torch.randn(c, c, 3, 3, device="cuda") * (2.0 / (9 * c)) ** 0.5
        r = W.QuantWinogradConv(plan, "legendre", W.QuantConfig.uniform(8))
        y = torch.empty(n, c, hw, hw, device="cuda")
        replay = r.capture(x, w, y, padding=1)
        for _ in range(5):
            replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"n={n} c={c} hw={hw} fix_cap={'auto' if cap == 0 else cap}: {e0.elapsed_time(e1) / 50 * 1000:.1f} us  sum|y|={float(y.abs().sum()):.6e}")
_lib.lib().wl_debug_set_fix_cap(0)
