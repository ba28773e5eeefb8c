"""Benchmark of the B200 quantized Legendre-Winograd F(4,3) layer (BASELINE.json metric).

Default workload (BASELINE.json configs[3], the largest single-GPU configuration): per GPU N=1024
images, Cin=Cout=256, 56x56, pad 1, 8-bit Legendre F(4,3) forward, x ~ N(0,1) fp32, Kaiming-normal
weights, bias 0, no collective.  Stage scales are per image ("image" groups: every image is
quantized exactly as one reference call on that image).  A step is one forward over the 1024 images;
the weight transform is cached (computed once before timing, the north star's "amortised" kernel).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload layer|train|bwd|sweep] [--scale-groups image|batch]

--gpus N > 1 without a torchrun environment re-launches itself under torch.distributed.run with N
ranks (one GPU each, NCCL); the batch is sharded (N x 1024 images), no data-path collective,
timing is the max over ranks.  Prints one JSON line on rank 0 (sweep/bwd: one line per config).
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "quantized Legendre-Winograd F(4,3) conv: effective TOPS & images/s"
CFG = dict(n=1024, c=256, hw=56, pad=1, mode="legendre", qconfig="8b")


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def layer_units(n, c, k, hw, pad):
    """SURVEY §8d algorithmic units of one forward call: fp32 x + fp32 y + weights bytes, int8 GEMM
    ops, direct-convolution-equivalent ops, tiles."""
    ho = hw + 2 * pad - 2
    T = n * (-(-ho // 4)) ** 2
    bytes_ = 4 * n * c * hw * hw + 4 * n * k * ho * ho + 36 * c * k + 4 * k
    i8ops = 2 * 36 * T * c * k
    eff_ops = 2 * 9 * n * ho * ho * c * k
    return bytes_, i8ops, eff_ops, T


def bwd_units(n, c, k, hw, pad):
    """SURVEY §8d backward units: dY + dX + re-read x (4 B each per element) + dW bytes; two 36-way
    GEMM sets (dV, dU)."""
    ho = hw + 2 * pad - 2
    T = n * (-(-ho // 4)) ** 2
    bytes_ = 4 * n * k * ho * ho + 4 * n * c * hw * hw * 2 + 4 * 9 * c * k
    ops = 2 * (2 * 36 * T * c * k)
    return bytes_, ops


# Forward kernels behind each wl_profile slot (prof_mark in wl_fwd*.cu), for the DRAM traffic lookup
SLOT_KERNELS = {
    "cast_input": ("cast_input_w64_kernel",),
    "absmax_input": ("absmax_input_kernel",),
    "quant_input": ("quant_input",),
    "input_base_change_max": ("sin_a2_kernel", "finalize_input_kernel<1, 4>", "finalize_input_exec<1, 4>"),
    "input_transform_max": ("sin_b2_kernel", "fixup_ibc_kernel", "finalize_input_kernel<1, 5>",
                            "finalize_input_exec<1, 5>"),
    "input_transform_codes": ("sin_c2_kernel", "fixup_it_kernel"),
    "gemm_hadamard_max": ("gemm_i8_persistent<256, 128, 4, EpiHadMax>", "gemm_i8_bstat<256, 128, 4, EpiHadMax",
                          "finalize_hadamard_kernel"),
    "gemm_hadamard_codes": ("gemm_i8_persistent<256, 128, 3, EpiHadRq", "gemm_i8_bstat<EpiHadRq", "fixup_had_kernel"),
    "output_base_change_max": ("sout_a2_kernel", "finalize_output_kernel<1, 7", "finalize_output_exec<1, 7"),
    "output_max": ("sout_bt2_kernel", "fixup_obct_kernel", "finalize_output_kernel<1, 8", "finalize_output_exec<1, 8"),
    "output_write": ("out_table_kernel", "sout_cw_kernel", "fixup_outt_kernel"),
}
NCU_FULL = os.path.join(ROOT, "profiles", "r02_ncu_full_cfg4_v8.csv")


def ncu_traffic(slot):
    """DRAM bytes (read + write) per launch of a profile slot from the committed `ncu --set full` capture
    of one config-4 forward (profiles/r02_ncu_full_cfg4_v8.csv, tools/ncu_full_cfg4.sh), or None."""
    try:
        with open(NCU_FULL) as fh:
            rows = list(csv.reader(fh))
    except OSError:
        return None
    unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    seen, total = set(), 0.0
    for r in rows[1:]:
        name = r[0]
        if name in seen or not any(name.startswith(p) for p in SLOT_KERNELS.get(slot, ())):
            continue
        seen.add(name)  # first launch of each kernel (the capture holds two forwards)
        for cell in (r[2], r[3]):
            v, u = cell.split()
            total += float(v) * unit[u]
    return total if seen else None


def kernel_units(name, n, c, k, hw, pad, hbytes=1):
    """Algorithmic bytes (what the pass must read and write: its input codes / values and the codes / values it
    produces, each once; c1 = [T][36][Cp] like V, T4E = 17 floats per unit) and int8 ops of one launch of each
    forward slot."""
    ho = hw + 2 * pad - 2
    T = n * (-(-ho // 4)) ** 2
    p2 = lambda v, lo: lo if v <= lo else 1 << (v - 1).bit_length()  # noqa: E731  (wl_internal.h pow2_at_least)
    cp, kp = p2(c, 32), p2(k, 64)
    x, c0, V, U, h, y = 4 * n * c * hw * hw, n * hw * hw * cp, 36 * T * cp, 36 * kp * cp, 36 * T * kp * hbytes, 4 * n * k * ho * ho
    table = {
        "cast_input": (x + c0, 0), "absmax_input": (x, 0), "quant_input": (x + c0, 0),
        "input_base_change_max": (c0, 0), "input_transform_max": (c0 + V, 0), "input_transform_codes": (2 * V, 0),
        "gemm_hadamard_max": (V + U, 2 * 36 * T * cp * kp), "gemm_hadamard_codes": (V + U + h, 2 * 36 * T * cp * kp),
        "output_base_change_max": (h, 0), "output_max": (h + 17 * T * kp * 4, 0), "output_write": (17 * T * kp * 4 + y, 0),
    }
    return table.get(name, (0, 0))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 20 ms during the timed region."""

    def __init__(self, index):
        self.index, self.proc, self.path = index, None, None

    def start(self):
        try:
            self.path = f"/tmp/bench_clocks_{os.getpid()}.csv"
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def physical_cores():
    """Physical cores among the CPUs this process may run on (hyper-thread siblings counted once)."""
    cpus = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else list(range(os.cpu_count() or 1))
    seen = set()
    for cpu in cpus:
        try:
            with open(f"/sys/devices/system/cpu/cpu{cpu}/topology/thread_siblings_list") as fh:
                seen.add(fh.read().strip())
        except OSError:
            seen.add(str(cpu))
    return max(1, len(seen)), len(cpus)


def cpu_baseline_and_parity(x_s, w, y_s, mode, groups):
    """cpu_baseline leg (rank 0, N=1): the CPU port of the reference path (oracle/, pinned bit-identical
    to the reference's numba backend) timed on the host's physical cores over a bounded sample of the
    bench's own images — and, as the checker, those images' GPU outputs compared bit for bit with it."""
    from oracle import oracle as O

    cores, logical = physical_cores()
    bits = O.uniform_bits(8)
    x64, w64 = x_s.astype(np.float64), w.astype(np.float64)
    ipg = 1 if groups == "image" else x_s.shape[0]
    O.quant_conv_batch(x64[:1, :, :8, :8], w64, mode, bits, padding=1, nthreads=1)  # load / warm
    times, yo = [], None
    for _ in range(3):
        t0 = time.perf_counter()
        yo, _, _ = O.quant_conv_batch(x64, w64, mode, bits, padding=1, images_per_group=ipg, nthreads=cores)
        times.append(time.perf_counter() - t0)
        if sum(times) > 20.0:
            break
    best = min(times)
    k = x_s.shape[0]
    base = {"value": k / best, "unit": "images/s", "cores": cores, "logical_cpus": logical, "kind": "port",
            "sample": f"{k} of the bench's config-4 images (256ch 56x56 pad1, Legendre 8b, per-image calls), "
                      f"best of {len(times)} runs, oracle/winoleg_oracle.c fp64 port of the reference path "
                      f"on {cores} physical cores"}
    parity = None
    if groups == "image":
        parity = {"images": int(k), "bit_exact": bool(np.array_equal(y_s, yo.astype(np.float32))),
                  "checker": "oracle/ (pinned to the reference's golden fixtures)", "workload": "N=1024 bench output"}
    return base, parity


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path (C port, bit-identical to the numba backend) on the
    host's physical cores; rank 0 only."""
    if rank != 0:
        return
    from oracle import oracle as O

    cores, logical = physical_cores()
    rng = np.random.default_rng(0)
    k = CFG["c"]
    w = (rng.standard_normal((k, k, 3, 3)) * np.sqrt(2.0 / (9 * k))).astype(np.float32).astype(np.float64)
    x = rng.standard_normal((cores, CFG["c"], CFG["hw"], CFG["hw"])).astype(np.float32).astype(np.float64)
    bits = O.uniform_bits(8)
    for _ in range(args.warmup):
        O.quant_conv_batch(x, w, CFG["mode"], bits, padding=1, images_per_group=1, nthreads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.quant_conv_batch(x, w, CFG["mode"], bits, padding=1, images_per_group=1, nthreads=cores)
    dt = (time.perf_counter() - t0) / args.steps
    _, _, eff, _ = layer_units(cores, CFG["c"], CFG["c"], CFG["hw"], CFG["pad"])
    val = cores / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config4: N=1024/GPU Cin=Cout=256 56x56 pad1 Legendre 8b fwd (sampled)",
                   "sample_images_per_step": cores, "scale_groups": "image"},
        "effective_tops": eff / dt / 1e12,
        "cpu_baseline": {"value": val, "unit": "images/s", "cores": cores, "logical_cpus": logical, "kind": "port",
                         "sample": f"{cores} images per step (one per physical core), per-image reference calls"},
        "e2e": {"value": val, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,  # the reference arm is the CPU path by definition
    }
    print(json.dumps(line), flush=True)


def measure_int8_peak(torch):
    try:
        a = torch.randint(-127, 127, (8192, 8192), dtype=torch.int8, device="cuda")
        b = torch.randint(-127, 127, (8192, 8192), dtype=torch.int8, device="cuda").t()
        for _ in range(3):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(5):
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return 2 * 8192 ** 3 / (best * 1e-3) / 1e12
    except Exception:
        return None


def measure_pcie(torch, nbytes=1 << 30):
    """Pinned-host <-> device copy bandwidth (GB/s, best of 3, CUDA events): H2D alone, D2H alone, and
    both at once on two streams (aggregate GB/s of the bidirectional run)."""
    h, h2 = (torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2))
    d, d2 = (torch.empty(nbytes, dtype=torch.uint8, device="cuda") for _ in range(2))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()

    def both():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    out = {}
    for name, fn, nb in (("h2d_gbs", lambda: d.copy_(h, non_blocking=True), nbytes),
                         ("d2h_gbs", lambda: h.copy_(d, non_blocking=True), nbytes),
                         ("bidir_aggregate_gbs", both, 2 * nbytes)):
        best = 1e9
        for _ in range(3):
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[name] = nb / (best * 1e-3) / 1e9
    del h, h2, d, d2
    return out


def _barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def _max_over_ranks(torch, v, world, dev):
    if world == 1:
        return v
    import torch.distributed as dist

    t = torch.tensor([v], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2004_11077_b200 as W
    from paper_2004_11077_b200 import _lib

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n, c, hw, pad = CFG["n"], CFG["c"], CFG["hw"], CFG["pad"]
    k = c
    groups = args.scale_groups
    qc = W.QuantConfig.from_name(CFG["qconfig"])
    plan = W.build_plan(4, 3, use_legendre=True)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)
    x = torch.randn((n, c, hw, hw), generator=gen, device=dev, dtype=torch.float32)
    gw = torch.Generator(device=dev)
    gw.manual_seed(0)
    w = torch.randn((k, c, 3, 3), generator=gw, device=dev) * float(np.sqrt(2.0 / (9 * c)))
    y = torch.empty((n, k, hw + 2 * pad - 2, hw + 2 * pad - 2), device=dev)
    r = W.QuantWinogradConv(plan, CFG["mode"], qc, dev)
    r.forward(x, w, padding=pad, out=y, scale_groups=groups)  # builds the weight cache + workspace
    torch.cuda.synchronize()
    launches = r.launches()

    # The step: the public forward of the whole batch.  With per-image scale groups the batch is issued as
    # `parts` independent calls on forked streams (QuantWinogradConv.forward_split, bit-identical to one call):
    # one part's kernel tails and helper kernels overlap the other part's passes.  --parts 1 = one stream.
    parts = args.parts if groups == "image" else 1

    def step():
        if parts > 1:
            r.forward_split(x, w, padding=pad, out=y, scale_groups=groups, parts=parts)
        else:
            r.forward(x, w, padding=pad, out=y, scale_groups=groups)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    _barrier(world)
    clocks = ClockSampler(local_rank)
    if rank == 0:
        clocks.start()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    _barrier(world)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    _barrier(world)
    ms_rank = e0.elapsed_time(e1) / args.steps
    # Per-slot kernel times: the same K steps as single-stream calls with the library's event marks on (the
    # marks need one stream), still under the clock sampler.
    _lib.profile_enable(True)
    _lib.profile_read()
    e0.record(stream)
    for _ in range(args.steps):
        r.forward(x, w, padding=pad, out=y, scale_groups=groups)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_single = e0.elapsed_time(e1) / args.steps
    kern, calls = _lib.profile_read()
    _lib.profile_enable(False)
    clk = clocks.stop() if rank == 0 else None
    ms = _max_over_ranks(torch, ms_rank, world, dev)
    per_rank_ms = [ms_rank]
    if world > 1:
        import torch.distributed as dist

        per_rank_ms = [None] * world
        dist.all_gather_object(per_rank_ms, ms_rank)

    # The same step issued as one CUDA-graph replay of two half-batch calls on two streams (per-image scale
    # groups make the halves independent and the result bit-identical): no launch gaps, and the kernels of the
    # two halves fill each other's tails.  Reported next to the eager single-stream headline.
    graph_replay = None
    if groups == "image" and n % 2 == 0 and world == 1:
        try:
            yref = y.clone()
            half = n // 2
            streams = [torch.cuda.Stream(dev) for _ in range(2)]
            wss = [torch.empty(r.workspace_bytes(r._shape(x[:half], w, pad, "image")), dtype=torch.uint8, device=dev)
                   for _ in range(2)]

            def two_stream_step():
                cur = torch.cuda.current_stream()
                ev = torch.cuda.Event()
                ev.record(cur)
                for i, s in enumerate(streams):
                    s.wait_event(ev)
                    with torch.cuda.stream(s):
                        r.forward(x[i * half:(i + 1) * half], w, padding=pad, out=y[i * half:(i + 1) * half],
                                  workspace=wss[i])
                    e = torch.cuda.Event()
                    e.record(s)
                    cur.wait_event(e)

            two_stream_step()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                two_stream_step()
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            y.zero_()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record()
            for _ in range(args.steps):
                g.replay()
            g1.record()
            torch.cuda.synchronize()
            gms = g0.elapsed_time(g1) / args.steps
            graph_replay = {"ms_per_step": gms, "images_per_s": n / (gms * 1e-3), "streams": 2, "calls": 2,
                            "bit_identical_to_single_call": bool(torch.equal(y, yref))}
            del wss, yref, g
        except Exception as exc:  # the headline does not depend on this extra
            graph_replay = {"error": str(exc)[:200]}

    # parity sample (checked in the cpu_baseline leg on rank 0 at N=1)
    # two images per physical core: every host thread of the CPU leg has work (8 images on 16 cores timed half the box)
    ksamp = min(n, max(8, 2 * physical_cores()[0]))
    x_s = x[:ksamp].cpu().numpy() if groups == "image" else x.cpu().numpy()
    y_s = y[:ksamp].cpu().numpy() if groups == "image" else y.cpu().numpy()
    w_s = w.cpu().numpy()

    # end to end through the public API with host buffers: pinned x -> device, forward, y -> pinned host,
    # copies inside the timed region (chunked so copy-in / compute / copy-out overlap; per-image scale
    # groups make the chunks independent, results identical to one call)
    e2e = None
    if not args.no_e2e and groups == "image":
        del x
        torch.cuda.empty_cache()
        xh = torch.empty((n, c, hw, hw), dtype=torch.float32, pin_memory=True)
        xh.normal_(generator=torch.Generator().manual_seed(1000 + rank))
        yh = torch.empty(tuple(y.shape), dtype=torch.float32, pin_memory=True)
        for _ in range(2):
            r.forward_host(xh, w, yh, padding=pad)
        torch.cuda.synchronize()
        _barrier(world)
        ke = max(1, min(args.steps, 5))
        e0.record(stream)
        for _ in range(ke):
            r.forward_host(xh, w, yh, padding=pad)
        e1.record(stream)
        torch.cuda.synchronize()
        me = _max_over_ranks(torch, e0.elapsed_time(e1) / ke, world, dev)
        pcie = measure_pcie(torch)
        hb, db_ = int(xh.numel() * 4), int(yh.numel() * 4)
        bound_ms = max(hb / (pcie["h2d_gbs"] * 1e9), db_ / (pcie["d2h_gbs"] * 1e9),
                       (hb + db_) / (pcie["bidir_aggregate_gbs"] * 1e9)) * 1e3
        e2e = {"value": world * n / (me * 1e-3), "unit": "images/s", "h2d_bytes_per_step": hb,
               "d2h_bytes_per_step": db_, "ms_per_step": me,
               "pcie": dict(pcie, bound_ms=bound_ms, frac=bound_ms / me,
                            note="bound = max(H2D bytes / H2D GB/s, D2H bytes / D2H GB/s, both / measured "
                                 "bidirectional aggregate GB/s): the copies overlap each other and the compute"),
               "path": "QuantWinogradConv.forward_host (C ABI wl_forward per chunk), pinned host x/y, 16 chunks"}
        del xh, yh

    if rank != 0:
        return
    hbm, bf16, peak_kind = _peaks()
    i8_peak = measure_int8_peak(torch)
    bytes_, i8ops, eff, T = layer_units(n, c, k, hw, pad)
    t_roof = max(bytes_ / (hbm * 1e9), i8ops / ((i8_peak or 2 * bf16) * 1e12))
    per_kernel = {name: v / max(calls, 1) for name, v in kern.items()}
    dom = max(per_kernel, key=per_kernel.get)
    kb, kops = kernel_units(dom, n, c, k, hw, pad)
    dom_ms = per_kernel[dom]
    t_hbm, t_tc = kb / (hbm * 1e9), (kops / ((i8_peak or 2 * bf16) * 1e12) if kops else 0.0)
    if t_tc > t_hbm:
        roof = {"kernel": dom, "bound": "tensor", "achieved": kops / (dom_ms * 1e-3) / 1e12,
                "peak": i8_peak or 2 * bf16, "unit": "TOPS(int8)"}
    else:
        roof = {"kernel": dom, "bound": "hbm", "achieved": kb / (dom_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = ncu_traffic(dom)
    roof["traffic_source"] = "profiles/r02_ncu_full_cfg4_v8.csv (ncu --set full, dram__bytes_read+write of the slot's kernels)"
    roof["algorithmic_bytes_per_launch"] = kb
    roof["ms_per_launch"] = dom_ms
    roof["timed_in"] = "single-stream pass of the same K steps with the library's CUDA-event marks, right after the timed region"
    roof["peak_source"] = peak_kind if roof["bound"] == "hbm" else ("torch._int_mm 8192^3 measured live" if i8_peak else "2x bf16 planning")
    # every slot against the same two ceilings; `limiter` is what ncu shows bounds the slot's main kernel
    # (profiles/r02_ncu_full_cfg4_v8.csv): the five transform passes are CUDA-core FMA/ALU-pipe bound, so their
    # HBM fraction is low by construction
    limiter = {"cast_input": "hbm (x read once; the second read of a band hits L2)", "absmax_input": "hbm",
               "quant_input": "issue + hbm", "input_base_change_max": "fma/alu pipes",
               "input_transform_max": "fma/alu pipes", "input_transform_codes": "fma/alu pipes",
               "gemm_hadamard_max": "tmem read (64 B/clk/SM) + hbm", "gemm_hadamard_codes": "epilogue issue + tmem read",
               "output_base_change_max": "fma/alu pipes", "output_max": "fma/alu pipes",
               "output_write": "hbm (NCHW write pattern)"}
    slots = {}
    for name, v in per_kernel.items():
        sb, sops = kernel_units(name, n, c, k, hw, pad)
        t_floor = max(sb / (hbm * 1e9), sops / ((i8_peak or 2 * bf16) * 1e12) if sops else 0.0)
        slots[name] = {"ms": round(v, 4), "algorithmic_gb": round(sb / 1e9, 3),
                       "roof_frac": round(t_floor / (v * 1e-3), 3) if v > 0 else None,
                       "limiter": limiter.get(name)}
    value = world * n / (ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int8", "data": "synthetic (torch.randn on device, seeded per rank)",
        "config": {"workload": "config4: N=1024/GPU Cin=Cout=256 56x56 pad1 Legendre F(4,3) 8b fwd",
                   "scale_groups": groups, "l2": "inputs (3.29 GB) larger than L2", "global_batch": world * n,
                   "call": (f"QuantWinogradConv.forward_split, {parts} parts on forked streams" if parts > 1
                            else "QuantWinogradConv.forward, one stream"),
                   "parallelism": f"batch-sharded x{world}, no collective"},
        "effective_tops": world * eff / (ms * 1e-3) / 1e12,
        "layer_roofline": {"t_roof_ms": t_roof * 1e3, "frac": t_roof / (ms * 1e-3), "hbm_bytes": bytes_,
                           "int8_ops": i8ops, "int8_peak_tops": i8_peak, "hbm_gbs": hbm},
        "roofline": roof,
        "per_rank_ms": per_rank_ms,
        "kernel_ms": {kname: round(v, 4) for kname, v in per_kernel.items()},
        "kernel_roofline": slots,
        "gpu_launches": launches * parts * args.steps,
        "streams": parts, "ms_per_step_single_stream": ms_single,
        "graph_replay": graph_replay,
        "clocks": clk,
        "e2e": e2e,
    }
    if world == 1 and not args.no_cpu:
        base, parity = cpu_baseline_and_parity(x_s, w_s, y_s, CFG["mode"], groups)
        line["cpu_baseline"] = base
        if parity is not None:
            line["parity"] = parity
    print(json.dumps(line), flush=True)


def _time_fn(torch, fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def run_sweep(args, rank, world, local_rank, backward_only=False):
    """One JSON line per BASELINE config (forward, CUDA-graph replay for the launch-bound shapes) and per
    config-3 shape forward + STE backward, each with its SURVEY §8d roofline."""
    import torch

    import paper_2004_11077_b200 as W

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    hbm, bf16, peak_kind = _peaks()
    i8 = measure_int8_peak(torch) or 2 * bf16
    plan = W.build_plan(4, 3, use_legendre=True)
    steps, warm = max(args.steps, 20), max(args.warmup, 3)

    def emit(d):
        if rank == 0:
            print(json.dumps(d), flush=True)

    fwd_cfgs = [("config1", 8, 64, 32, "legendre", "8b", "image")]
    for mode in ("legendre", "canonical"):
        for q in ("8b+9b", "8b"):
            fwd_cfgs.append((f"config2 {mode} {q}", 128, 128, 16, mode, q, "image"))
    for c, hw in ((64, 32), (128, 16), (256, 8), (512, 4)):
        fwd_cfgs.append((f"config3 C={c} {hw}x{hw} fwd", 256, c, hw, "legendre", "8b", "image"))
    fwd_cfgs.append(("config4 batch scale groups", 1024, 256, 56, "legendre", "8b", "batch"))
    if not backward_only:
        for name, n, c, hw, mode, q, groups in fwd_cfgs:
            g = torch.Generator(device=dev)
            g.manual_seed(0)
            x = torch.randn((n, c, hw, hw), generator=g, device=dev)
            if name.startswith("config3"):
                x = x.clamp_min_(0)
            w = torch.randn((c, c, 3, 3), generator=g, device=dev) * float(np.sqrt(2.0 / (9 * c)))
            y = torch.empty((n, c, hw, hw), device=dev)
            r = W.QuantWinogradConv(plan, mode, W.QuantConfig.from_name(q), dev)
            small = n * c * hw * hw * 4 < 512 << 20
            fn = (r.capture(x, w, y, padding=1, scale_groups=groups) if small
                  else (lambda: r.forward(x, w, padding=1, out=y, scale_groups=groups)))
            ms = _time_fn(torch, fn, steps if small else max(3, args.steps), warm)
            bytes_, i8ops, eff, _ = layer_units(n, c, c, hw, 1)
            t_roof = max(bytes_ / (hbm * 1e9), i8ops / (i8 * 1e12))
            emit({"metric": METRIC, "workload": "sweep", "config": name, "n": n, "c": c, "hw": hw, "mode": mode,
                  "qconfig": q, "scale_groups": groups, "ms": ms, "images_per_s": n / (ms * 1e-3),
                  "effective_tops": eff / (ms * 1e-3) / 1e12, "t_roof_us": t_roof * 1e6,
                  "roofline_frac": t_roof / (ms * 1e-3), "cuda_graph": small, "gpu_launches": r.launches(),
                  "peaks": {"hbm_gbs": hbm, "int8_tops": i8, "hbm_source": peak_kind}})
            del x, y, r
            torch.cuda.empty_cache()
    # config 3: forward (training forward, saved block) + STE backward
    for c, hw in ((64, 32), (128, 16), (256, 8), (512, 4)):
        n = 256
        g = torch.Generator(device=dev)
        g.manual_seed(1)
        x = torch.randn((n, c, hw, hw), generator=g, device=dev).clamp_min_(0)
        w = (torch.randn((c, c, 3, 3), generator=g, device=dev) * float(np.sqrt(2.0 / (9 * c)))).requires_grad_()
        dy = torch.randn((n, c, hw, hw), generator=g, device=dev)
        mod = W.WinogradAwareConv2d(c, c).to(dev)
        with torch.no_grad():
            mod.weight.copy_(w)
        xr = x.clone().requires_grad_()

        def fwd_bwd():
            out = mod(xr)
            out.backward(dy)

        ms_fb = _time_fn(torch, fwd_bwd, max(args.steps, 10), warm)
        r = mod._runner(dev)

        def fwd():
            with torch.no_grad():
                mod(x)

        ms_f = _time_fn(torch, fwd, max(args.steps, 10), warm)
        yv = mod(xr)
        shape, cache, saved, _ = r._last

        def bwd():
            r.backward(dy, shape, cache, saved, False)

        ms_b = _time_fn(torch, bwd, max(args.steps, 10), warm)
        bb, bops = bwd_units(n, c, c, hw, 1)
        t_roof_b = max(bb / (hbm * 1e9), bops / (bf16 * 1e12))
        emit({"metric": "config-3 STE backward (dX, dW, db)", "workload": "sweep-bwd", "config": f"config3 C={c} {hw}x{hw}",
              "n": n, "c": c, "hw": hw, "mode": "legendre", "qconfig": "8b", "ms_backward": ms_b,
              "ms_forward_train": ms_f, "ms_forward_plus_backward": ms_fb, "images_per_s_fwd_bwd": n / (ms_fb * 1e-3),
              "t_roof_backward_us": t_roof_b * 1e6, "roofline_frac_backward": t_roof_b / (ms_b * 1e-3),
              "roofline_basis": "SURVEY §8d: bytes dY+dX+x+dW at measured HBM, ops 2x(2*36*T*C*K) at measured bf16 dense"})
        del x, w, dy, mod, xr, yv
        torch.cuda.empty_cache()


def run_train(args, rank, world, local_rank):
    """Config 5: ResNet-18 with every 3x3 stride-1 conv on the Legendre 8b Winograd layer, one
    training step (forward, STE backward, SGD momentum 0.9, lr 0.1) on 256 synthetic 3x32x32 images
    per GPU; data parallel with one NCCL gradient all-reduce per step (DDP) when N > 1."""
    import torch

    from paper_2004_11077_b200 import training as TR

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    torch.manual_seed(0)
    model = TR.ResNet18(TR.winograd_conv_factory("legendre")).to(dev)
    nwino = TR.count_winograd_layers(model)
    net = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local_rank]) if world > 1 else model
    opt = TR.make_optimizer(net, lr=0.1)
    batch = 256
    x, y = TR.synthetic_batch(batch, rank, seed=0, device=dev)
    for _ in range(args.warmup):
        TR.train_step(net, opt, x, y)
    torch.cuda.synchronize()
    _barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        loss = TR.train_step(net, opt, x, y)
    e1.record()
    torch.cuda.synchronize()
    _barrier(world)
    ms_eager = _max_over_ranks(torch, e0.elapsed_time(e1) / args.steps, world, dev)
    ms, graphed = ms_eager, False
    if world == 1 and not args.no_graph:
        # single GPU: the same step as one CUDA graph (the eager step is host-launch-bound at batch 256)
        step = TR.make_graphed_step(net, opt, x, y, warmup=1)
        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            loss = step()
        e1.record()
        torch.cuda.synchronize()
        ms, graphed = e0.elapsed_time(e1) / args.steps, True
        TR.invalidate_weight_caches(model)
    # Phase breakdown on extra steps AFTER the timed region: CUDA events around every Winograd-layer forward
    # (wl_forward_train) and STE backward (wl_backward); the rest is PyTorch (BN, ReLU, stride-2 / 1x1 convs,
    # FC, loss, SGD, DDP all-reduce).
    from paper_2004_11077_b200 import layer as LY
    marks = []

    def _timed(kind, fn):
        def wrapper(self, *a, **k):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            out = fn(self, *a, **k)
            e.record()
            marks.append((kind, s, e))
            return out
        return wrapper

    of, ob = LY.QuantWinogradConv.forward, LY.QuantWinogradConv.backward
    LY.QuantWinogradConv.forward, LY.QuantWinogradConv.backward = _timed("fwd", of), _timed("bwd", ob)
    psteps = 3
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    TR.train_step(net, opt, x, y)  # untimed: rebuilds the weight caches the graphed steps left stale
    marks.clear()
    p0.record()
    for _ in range(psteps):
        TR.train_step(net, opt, x, y)
    p1.record()
    torch.cuda.synchronize()
    LY.QuantWinogradConv.forward, LY.QuantWinogradConv.backward = of, ob
    pf = sum(s.elapsed_time(e) for k, s, e in marks if k == "fwd") / psteps
    pb = sum(s.elapsed_time(e) for k, s, e in marks if k == "bwd") / psteps
    pt = p0.elapsed_time(p1) / psteps
    phases = {"winograd_forward_ms": round(pf, 3), "winograd_backward_ms": round(pb, 3),
              "pytorch_rest_ms": round(pt - pf - pb, 3), "step_ms_with_events": round(pt, 3),
              "note": "3 extra steps after the timed region, CUDA events around each of the %d Winograd layers" % nwino}
    if rank == 0:
        print(json.dumps({
            "metric": "ResNet-18 (Winograd-aware Legendre 8b) training throughput", "value": world * batch / (ms * 1e-3),
            "unit": "images/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8 fwd (tcgen05 kind::i8) / fp32-accurate split-bf16 bwd (tcgen05 kind::f16)",
            "data": "synthetic N(0,1) 3x32x32, uniform labels", "loss": float(loss), "phases": phases,
            "cuda_graph": graphed, "ms_per_step_eager": ms_eager,
            "config": {"workload": "config5: ResNet-18 32x32, %d Winograd layers, batch 256/GPU, SGD m=0.9 lr=0.1"
                       % nwino, "global_batch": world * batch, "parallelism": f"DDP x{world} (NCCL all-reduce)"},
        }), flush=True)


def run_selftest(args, rank, world):
    """CPU check of the launcher and the timing plumbing (gloo): every rank times a fixed numpy step;
    the line's n_gpus is the world size and ms_per_step the max over ranks (tests/test_bench_launcher.py)."""
    import torch
    import torch.distributed as dist

    a = np.random.default_rng(rank).standard_normal((256, 256))
    _barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        a = np.tanh(a @ a.T * 1e-3)
    ms = (time.perf_counter() - t0) / args.steps * 1e3 * (1 + rank)  # rank-dependent: the max must win
    t = torch.tensor([ms], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    per = [None] * world
    if world > 1:
        dist.all_gather_object(per, ms)
    else:
        per = [ms]
    if rank == 0:
        print(json.dumps({"selftest": True, "n_gpus": world, "ms_per_step": float(t.item()), "per_rank_ms": per,
                          "steps": args.steps}), flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="train workload: time the eager step only")
    ap.add_argument("--scale-groups", default="image", choices=["image", "batch"])
    ap.add_argument("--parts", type=int, default=2,
                    help="layer workload: independent calls on forked streams per step (per-image scale groups)")
    ap.add_argument("--workload", default="layer", choices=["layer", "train", "bwd", "sweep"],
                    help="layer: config-4 layer throughput (default); train: config-5 ResNet-18 training step; "
                         "bwd: config-3 forward + STE backward lines; sweep: every forward config + bwd")
    ap.add_argument("--selftest", action="store_true", help="CPU/gloo check of the launcher (no GPU work)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # self-launch: one rank per GPU under torch.distributed.run (the driver's own command line)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.selftest:
        if world > 1:
            import torch.distributed as dist

            dist.init_process_group("gloo")
        run_selftest(args, rank, world)
        if world > 1:
            dist.destroy_process_group()
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.workload == "train":
        run_train(args, rank, world, local_rank)
    elif args.workload in ("sweep", "bwd"):
        run_sweep(args, rank, world, local_rank, backward_only=args.workload == "bwd")
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
