"""Config-4 forward time vs image-chunk size / concurrent streams / CUDA-graph capture.

With per-image scale groups a batch splits exactly into independent chunks; small chunks keep the
intermediate code tensors (c0, c1, V, h, c4) resident in the 126 MB L2 between passes.

    python tools/chunk_sweep.py [chunk ...]
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2004_11077_b200 as W  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    n, c, hw, pad = 1024, 256, 56, 1
    x = torch.randn((n, c, hw, hw), device=dev)
    w = torch.randn((c, c, 3, 3), device=dev) * float(np.sqrt(2.0 / (9 * c)))
    y = torch.empty((n, c, hw, hw), device=dev)
    r = W.QuantWinogradConv(W.build_plan(4, 3, use_legendre=True), "legendre", W.QuantConfig.from_name("8b"), dev)
    r.forward(x, w, padding=pad, out=y)
    yref = y.clone()
    main_s = torch.cuda.current_stream()
    configs = []
    for ch in [int(a) for a in sys.argv[1:]] or [1024, 128, 64, 32, 16, 8]:
        for ns in ([1] if ch == n else [1, 2, 3, 4]):
            configs.append((ch, ns))
    for ch, ns in configs:
        streams = [torch.cuda.Stream(dev) for _ in range(ns)]
        shape = r._shape(x[:ch], w, pad, "image")
        wsz = r.workspace_bytes(shape)
        wss = [torch.empty(wsz, dtype=torch.uint8, device=dev) for _ in range(ns)]

        def step():
            main_s = torch.cuda.current_stream()
            ev = torch.cuda.Event()
            ev.record(main_s)
            for s in streams:
                s.wait_event(ev)
            for i in range(n // ch):
                s = streams[i % ns]
                with torch.cuda.stream(s):
                    r.forward(x[i * ch:(i + 1) * ch], w, padding=pad, out=y[i * ch:(i + 1) * ch], workspace=wss[i % ns])
            for s in streams:
                e = torch.cuda.Event()
                e.record(s)
                main_s.wait_event(e)

        for graph in ((False, True) if os.environ.get('EAGER') else (True,)):
            try:
                if graph:
                    g = torch.cuda.CUDAGraph()
                    step()
                    torch.cuda.synchronize()
                    with torch.cuda.graph(g):
                        step()
                    fn = g.replay
                else:
                    fn = step
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                y.zero_()
                e0.record(main_s)
                for _ in range(5):
                    fn()
                e1.record(main_s)
                torch.cuda.synchronize()
                ok = torch.equal(y, yref)
                print(f"chunk {ch:5d} streams {ns} graph {int(graph)}: {e0.elapsed_time(e1) / 5:8.3f} ms  exact={ok}",
                      flush=True)
            except Exception as exc:  # report and go on
                print(f"chunk {ch} streams {ns} graph {int(graph)}: FAILED {exc}", flush=True)
                torch.cuda.synchronize()


if __name__ == "__main__":
    main()
