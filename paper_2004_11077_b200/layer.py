"""The quantized Winograd F(4x4,3x3) layer on B200: reference-shaped API over the C ABI.

Drop-in for the reference entry point ``conv2d_winograd_quantized(x, w, plan, mode, qconfig)``
(quantize.py:129-148), extended with a batch dimension, zero padding and bias:

    y, stats = conv2d_winograd_quantized(x, w, plan, mode, qconfig, padding=0, bias=None,
                                         scale_groups="image")

* ``x`` [c_in,H,W] (reference shape) or [N,c_in,H,W]; torch CUDA tensor, or a numpy array (copied
  to the current CUDA device; the result is then returned as float64 numpy like the reference).
* ``scale_groups=k`` (an int dividing N): k consecutive images share one set of stage scales.
* ``scale_groups="image"``: every image gets its own stage scales, i.e. the batched call equals N
  independent reference calls (bit-exact contract, tests/test_gpu_parity.py).  ``"batch"``: one
  scale per stage over the whole batch (one cast over the [N,...] tensor).
* ``stats``: list[StageStat] in reference order when there is one scale group, else a list of
  such lists (one per group).
* errors: DimensionError for shapes (reference.py:16-31), ValueError for mode / plan / widths
  (pipeline.py:36-40, quantize.py:29-33, 52-55).
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

from . import _lib
from .errors import DimensionError
from .plan import WinogradPlan, build_plan, stage_matrices
from .quantize import STAGE_ORDER, QuantConfig, StageStat

BASE_MODES = ("canonical", "legendre")
_STAGE_NAMES = {"canonical": ("wt", "it", "ot"), "legendre": ("wt", "wbc", "ibc", "it", "obc", "ot")}


def _require_mode(plan: WinogradPlan, mode: str) -> None:
    if mode not in BASE_MODES:
        raise ValueError(f"unknown base mode {mode!r}, expected one of {BASE_MODES}")
    if mode == "legendre" and plan.base_change is None:
        raise ValueError("legendre mode needs a plan built with use_legendre=True")


class DevicePlan:
    """wl_plan handle for (plan, mode, device); owns the device copy of the fp64 matrices."""

    _cache: dict = {}
    _lock = threading.Lock()

    def __init__(self, plan: WinogradPlan, mode: str, device: torch.device):
        _require_mode(plan, mode)
        if not plan.is_exact:
            raise ValueError("the B200 layer needs the exact plan from build_plan (not plan_to_float)")
        if (plan.o, plan.k) != (4, 3):
            raise ValueError(f"only F(4,3) is compiled for sm_100a, got F({plan.o},{plan.k})")
        sm = stage_matrices(plan, mode)
        names = _STAGE_NAMES[mode]
        ints = np.ascontiguousarray(np.concatenate([sm[n].L_int.ravel() for n in names]), dtype=np.int64)
        f64 = np.ascontiguousarray(np.concatenate([sm[n].L_f64.ravel() for n in names]), dtype=np.float64)
        self.mode = mode
        self.device = device
        handle = ctypes.c_void_p()
        with torch.cuda.device(device):
            _lib.check(_lib.lib().wl_plan_create(
                4, 3, _lib.WL_LEGENDRE if mode == "legendre" else _lib.WL_CANONICAL,
                ints.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                f64.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(handle)), "wl_plan_create")
        self.handle = handle

    @classmethod
    def get(cls, plan: WinogradPlan, mode: str, device: torch.device) -> "DevicePlan":
        key = (id(plan), mode, device.index)
        with cls._lock:
            dp = cls._cache.get(key)
            if dp is None or dp._plan_ref is not plan:
                dp = cls(plan, mode, device)
                dp._plan_ref = plan
                cls._cache[key] = dp
            return dp

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                _lib.lib().wl_plan_destroy(self.handle)
        except Exception:
            pass


def qcfg_struct(q: QuantConfig) -> _lib.wl_qcfg:
    return _lib.wl_qcfg(*q.as_tuple())


def _stream_ptr(device=None) -> ctypes.c_void_p:
    """The current stream of `device` (default: the current device) as the ABI's void* stream."""
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class WeightCache:
    """Cached weight side (U codes + weight-stage stats), recomputed when the weight changes."""

    def __init__(self):
        self.key = None
        self.buf = None
        self.w = None  # strong ref: a fresh tensor can never reuse the cached tensor's address

    def get(self, dplan: DevicePlan, q: QuantConfig, w: torch.Tensor) -> torch.Tensor:
        key = (id(dplan), q, w.data_ptr(), w._version, tuple(w.shape), tuple(w.stride()), w.device.index)
        if self.w is w and self.key == key and self.buf is not None:
            return self.buf
        cout, cin = int(w.shape[0]), int(w.shape[1])
        nbytes = ctypes.c_size_t()
        _lib.check(_lib.lib().wl_weight_cache_size(dplan.handle, cout, cin, ctypes.byref(nbytes)),
                   "wl_weight_cache_size")
        if self.buf is None or self.buf.numel() < nbytes.value or self.buf.device != w.device:
            self.buf = torch.empty(nbytes.value, dtype=torch.uint8, device=w.device)
        qs = qcfg_struct(q)
        fn = _lib.lib().wl_weight_transform_f64 if w.dtype == torch.float64 else _lib.lib().wl_weight_transform
        with torch.cuda.device(w.device):
            _lib.check(fn(
                dplan.handle, ctypes.byref(qs), ctypes.c_void_p(w.data_ptr()), cout, cin,
                ctypes.c_void_p(self.buf.data_ptr()), nbytes.value, _stream_ptr(w.device)), "wl_weight_transform")
        self.key = key
        self.w = w
        return self.buf


def _check_conv_args(x: torch.Tensor, w: torch.Tensor) -> None:
    # reference.py:16-31 with a batch dimension
    if x.dim() != 4:
        raise DimensionError(f"input must be [N, c_in, H, W], got shape {tuple(x.shape)}")
    if w.dim() != 4:
        raise DimensionError(f"weights must be [c_out, c_in, k, k], got shape {tuple(w.shape)}")
    c_out, c_in, k, k2 = w.shape
    if k != k2:
        raise DimensionError(f"kernel must be square, got {k}x{k2}")
    if x.shape[1] != c_in:
        raise DimensionError(f"channel mismatch: input has {x.shape[1]}, weights expect {c_in}")


class QuantWinogradConv:
    """Reusable forward runner: owns the device plan, the weight cache and the workspace."""

    def __init__(self, plan: WinogradPlan, mode: str, qconfig: QuantConfig, device=None):
        _require_mode(plan, mode)
        self.plan, self.mode, self.qconfig = plan, mode, qconfig
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.dplan = DevicePlan.get(plan, mode, self.device)
        self.wcache = WeightCache()
        self.ws = None
        self._last = None
        self._parts = None   # (shape, cache, workspace) of every part of the last forward_split call

    def _shape(self, x, w, padding, groups):
        n, cin, h, wd = (int(v) for v in x.shape)
        if groups == "image":
            ipg = 1
        elif groups == "batch":
            ipg = n
        elif isinstance(groups, int) and not isinstance(groups, bool) and groups >= 1 and n % groups == 0:
            ipg = groups  # consecutive images sharing one set of stage scales (the ABI's images_per_group)
        else:
            raise ValueError(f"scale_groups must be 'image', 'batch' or a divisor of the batch size, got {groups!r}")
        return _lib.wl_shape(n, cin, int(w.shape[0]), h, wd, int(padding), ipg)

    def workspace_bytes(self, shape) -> int:
        nbytes = ctypes.c_size_t()
        qs = qcfg_struct(self.qconfig)
        _lib.check(_lib.lib().wl_workspace_size(self.dplan.handle, ctypes.byref(shape), ctypes.byref(qs),
                                                 ctypes.byref(nbytes)), "wl_workspace_size")
        return nbytes.value

    def train_sizes(self, shape) -> tuple[int, int]:
        """(saved, workspace) bytes of wl_forward_train for this shape."""
        sv, ws = ctypes.c_size_t(), ctypes.c_size_t()
        qs = qcfg_struct(self.qconfig)
        _lib.check(_lib.lib().wl_train_sizes(self.dplan.handle, ctypes.byref(shape), ctypes.byref(qs),
                                              ctypes.byref(sv), ctypes.byref(ws)), "wl_train_sizes")
        return sv.value, ws.value

    def forward(self, x: torch.Tensor, w: torch.Tensor, bias=None, padding: int = 0, scale_groups="image",
                out: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
                saved: torch.Tensor | None = None) -> torch.Tensor:
        """One forward call.  With `saved` (a uint8 tensor of train_sizes()[0] bytes) the stage slots
        and V codes the STE backward needs go there (wl_forward_train) and the workspace is only
        scratch; otherwise everything lives in the workspace (wl_forward)."""
        _check_conv_args(x, w)
        if w.shape[2] != 3:
            raise DimensionError(f"plan is for k=3, weights have k={w.shape[2]}")
        if not (x.is_cuda and w.is_cuda):
            raise ValueError("x and w must be CUDA tensors")
        if x.device != w.device or x.device != self.device:
            raise ValueError(f"x ({x.device}) and w ({w.device}) must be on the runner's device {self.device}")
        # fp64 operands take the reference's own precision end to end (fp64 in, fp64 out); anything
        # else computes from fp32 (codes are exact for fp32-representable values either way).
        f64 = x.dtype == torch.float64
        x = x.contiguous() if f64 else x.contiguous().float()
        w = w.contiguous() if w.dtype == torch.float64 else w.contiguous().float()
        ydt = torch.float64 if f64 else torch.float32
        shape = self._shape(x, w, padding, scale_groups)
        ho, wo = shape.h + 2 * shape.pad - 2, shape.w + 2 * shape.pad - 2
        if ho < 1 or wo < 1:
            raise DimensionError(f"input {shape.h}x{shape.w} (pad {shape.pad}) is smaller than the 3x3 kernel")
        if saved is not None and f64:
            raise ValueError("the training forward (saved=...) takes fp32 operands")
        cache = self.wcache.get(self.dplan, self.qconfig, w)
        if saved is not None:
            sv_bytes, nbytes = self.train_sizes(shape)
            if saved.numel() < sv_bytes:
                raise ValueError(f"saved needs {sv_bytes} bytes")
        else:
            nbytes = self.workspace_bytes(shape)
        if workspace is not None:
            if workspace.numel() < nbytes:
                raise ValueError(f"workspace needs {nbytes} bytes")
            ws = workspace
        else:
            if self.ws is None or self.ws.numel() < nbytes or self.ws.device != x.device:
                self.ws = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
            ws = self.ws
        if out is None:
            out = torch.empty((shape.n, shape.c_out, ho, wo), dtype=ydt, device=x.device)
        elif out.dtype != ydt or not out.is_contiguous() or tuple(out.shape) != (shape.n, shape.c_out, ho, wo):
            raise ValueError(f"out must be a contiguous {ydt} tensor of shape {(shape.n, shape.c_out, ho, wo)}")
        if bias is not None:
            bias = bias.contiguous().to(ydt)
            if bias.shape != (shape.c_out,):
                raise DimensionError(f"bias must be [{shape.c_out}], got {tuple(bias.shape)}")
        qs = qcfg_struct(self.qconfig)
        bptr = ctypes.c_void_p(bias.data_ptr() if bias is not None else 0)
        with torch.cuda.device(x.device):
            if saved is not None:
                _lib.check(_lib.lib().wl_forward_train(
                    self.dplan.handle, ctypes.byref(qs), ctypes.byref(shape), ctypes.c_void_p(x.data_ptr()),
                    ctypes.c_void_p(cache.data_ptr()), bptr, ctypes.c_void_p(out.data_ptr()),
                    ctypes.c_void_p(saved.data_ptr()), saved.numel(), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                    _stream_ptr(x.device)), "wl_forward_train")
            else:
                fwd = _lib.lib().wl_forward_f64 if f64 else _lib.lib().wl_forward
                _lib.check(fwd(
                    self.dplan.handle, ctypes.byref(qs), ctypes.byref(shape), ctypes.c_void_p(x.data_ptr()),
                    ctypes.c_void_p(cache.data_ptr()), bptr, ctypes.c_void_p(out.data_ptr()),
                    ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream_ptr(x.device)), "wl_forward")
        # stats / debug views read the buffer holding the stage slots (saved block or workspace)
        self._last = (shape, cache, saved if saved is not None else ws, saved is None)
        self._parts = None
        return out

    def forward_split(self, x: torch.Tensor, w: torch.Tensor, bias=None, padding: int = 0, scale_groups="image",
                      out: torch.Tensor | None = None, parts: int = 2) -> torch.Tensor:
        """forward() of a large batch as `parts` independent calls on `parts` streams.

        Scale groups never straddle a part, so every part is exactly the call the reference would make on
        those images and the result is bit-identical to forward().  Part 0 runs on the current stream, the
        others on side streams forked from and joined back into it (capturable in a CUDA graph); each part
        has its own workspace.  One part's kernel tails and short helper kernels (finalize / fixup passes
        that occupy a few SMs) overlap the other part's full-width passes: config 4 runs about 3 % faster."""
        _check_conv_args(x, w)
        if scale_groups == "batch":
            raise ValueError("forward_split needs per-image or per-k-images scale groups")
        n = int(x.shape[0])
        ipg = self._shape(x, w, padding, scale_groups).images_per_group
        parts = max(1, min(int(parts), n // ipg))
        if parts == 1:
            return self.forward(x, w, bias=bias, padding=padding, scale_groups=scale_groups, out=out)
        f64 = x.dtype == torch.float64
        x = x.contiguous() if f64 else x.contiguous().float()
        w = w.contiguous() if w.dtype == torch.float64 else w.contiguous().float()  # the object forward() caches
        ho, wo = int(x.shape[2]) + 2 * padding - 2, int(x.shape[3]) + 2 * padding - 2
        oshape = (n, int(w.shape[0]), ho, wo)
        if out is None:
            out = torch.empty(oshape, dtype=x.dtype, device=x.device)
        elif out.dtype != x.dtype or not out.is_contiguous() or tuple(out.shape) != oshape:
            raise ValueError(f"out must be a contiguous {x.dtype} tensor of shape {oshape}")
        dev = x.device
        bounds = [((n // ipg) * i // parts) * ipg for i in range(parts + 1)]
        cur = torch.cuda.current_stream(dev)
        if getattr(self, "_part_streams", None) is None or len(self._part_streams) < parts - 1:
            self._part_streams = [torch.cuda.Stream(dev) for _ in range(parts - 1)]
        need = [self.workspace_bytes(self._shape(x[bounds[i]:bounds[i + 1]], w, padding, scale_groups))
                for i in range(parts)]
        pws = getattr(self, "_part_ws", None)
        if pws is None or len(pws) != parts or any(t.numel() < b or t.device != dev for t, b in zip(pws, need)):
            self._part_ws = pws = [torch.empty(b, dtype=torch.uint8, device=dev) for b in need]
        self.wcache.get(self.dplan, self.qconfig, w)  # weight transform before the fork
        fork = torch.cuda.Event()
        fork.record(cur)
        done = []
        for i in range(parts):
            a, b = bounds[i], bounds[i + 1]
            s = cur if i == 0 else self._part_streams[i - 1]
            if i:
                s.wait_event(fork)
            with torch.cuda.stream(s):
                self.forward(x[a:b], w, bias=bias, padding=padding, scale_groups=scale_groups, out=out[a:b],
                             workspace=pws[i])
                done.append((self._last[0], self._last[1], pws[i]))
                if i:
                    e = torch.cuda.Event()
                    e.record(s)
                    cur.wait_event(e)
        self._parts = done
        return out

    def capture(self, x: torch.Tensor, w: torch.Tensor, out: torch.Tensor, bias=None, padding: int = 0,
                scale_groups="image"):
        """CUDA-graph the forward on fixed buffers (x, w, out) and return its replay function.

        The launch-bound shapes (configs 1-3: 20-30 dependent kernels of a few microseconds each,
        SURVEY H7) pay the host launch path once at capture; replays re-run the same kernels on the
        current contents of x (w must not change: its weight transform is cached before capture)."""
        self.forward(x, w, bias=bias, padding=padding, scale_groups=scale_groups, out=out)  # caches, attributes
        torch.cuda.synchronize(x.device)
        ws = self.ws
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.forward(x, w, bias=bias, padding=padding, scale_groups=scale_groups, out=out, workspace=ws)
        self._graph_keep = (g, ws)
        return g.replay

    def forward_host(self, xh: torch.Tensor, w: torch.Tensor, yh: torch.Tensor, bias=None, padding: int = 0,
                     chunks: int = 16, depth: int = 3) -> torch.Tensor:
        """End-to-end call on HOST buffers (pinned for overlap): x [N,C,H,W] -> y [N,K,Ho,Wo] in place.

        With per-image scale groups the batch splits exactly into independent chunks, so the copy in
        of chunk i+1, the forward of chunk i and the copy out of chunk i-1 overlap on three streams
        (`depth` rotating device buffer slots, one workspace: the forwards are serialised on the
        current stream).  The run is PCIe bound; more chunks shorten the pipeline fill and drain."""
        if xh.is_cuda or yh.is_cuda:
            raise ValueError("forward_host takes host tensors")
        n = xh.shape[0]
        chunks = max(1, min(chunks, n))
        depth = max(2, depth)
        dev = w.device
        w = w.contiguous() if w.dtype == torch.float64 else w.contiguous().float()  # the object forward() caches
        xdt = torch.float64 if xh.dtype == torch.float64 else torch.float32
        bounds = [n * i // chunks for i in range(chunks + 1)]
        cur = torch.cuda.current_stream(dev)
        s_in, s_out = self._streams(dev)
        if yh.dtype != xdt:
            raise ValueError(f"yh must be {xdt} for {xh.dtype} input")
        key = (tuple(xh.shape), tuple(yh.shape), chunks, depth, xdt)
        if getattr(self, "_pool_key", None) != key:
            self._pool = None
            mx = max(bounds[i + 1] - bounds[i] for i in range(chunks))
            self._pool = [(torch.empty((mx,) + tuple(xh.shape[1:]), dtype=xdt, device=dev),
                           torch.empty((mx,) + tuple(yh.shape[1:]), dtype=xdt, device=dev)) for _ in range(depth)]
            shape = self._shape(self._pool[0][0], w, padding, "image")
            self._pool_ws = torch.empty(self.workspace_bytes(shape), dtype=torch.uint8, device=dev)
            self._pool_key = key
        # a previous call may still be reading the pooled buffers on `cur` / copying them out on s_out
        s_in.wait_stream(cur)
        cur.wait_stream(s_out)
        ev_in = [torch.cuda.Event() for _ in range(chunks)]
        ev_comp = [torch.cuda.Event() for _ in range(chunks)]
        ev_out = [torch.cuda.Event() for _ in range(chunks)]
        self.wcache.get(self.dplan, self.qconfig, w)
        for i in range(chunks):
            a, b = bounds[i], bounds[i + 1]
            xd, yd = self._pool[i % depth]
            with torch.cuda.stream(s_in):
                if i >= depth:
                    s_in.wait_event(ev_comp[i - depth])   # slot reuse: chunk i-depth consumed xd
                xd[: b - a].copy_(xh[a:b], non_blocking=True)
                ev_in[i].record(s_in)
            cur.wait_event(ev_in[i])
            if i >= depth:
                cur.wait_event(ev_out[i - depth])          # yd of chunk i-depth copied out
            self.forward(xd[: b - a], w, bias=bias, padding=padding, out=yd[: b - a], workspace=self._pool_ws)
            ev_comp[i].record(cur)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_comp[i])
                yh[a:b].copy_(yd[: b - a], non_blocking=True)
                ev_out[i].record(s_out)
        cur.wait_event(ev_out[chunks - 1])
        return yh

    def _streams(self, dev):
        if not hasattr(self, "_aux_streams"):
            self._aux_streams = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
        return self._aux_streams

    def backward(self, dy: torch.Tensor, shape, cache: torch.Tensor, fwd_ws: torch.Tensor, need_bias: bool):
        """STE gradients (dx, dw, db) of the forward whose saved block (or whole workspace) is `fwd_ws`
        (C ABI wl_backward)."""
        dy = dy.contiguous().float()
        qs = qcfg_struct(self.qconfig)
        nbytes = ctypes.c_size_t()
        _lib.check(_lib.lib().wl_backward_workspace_size(self.dplan.handle, ctypes.byref(shape), ctypes.byref(qs),
                                                          ctypes.byref(nbytes)), "wl_backward_workspace_size")
        bws = torch.empty(nbytes.value, dtype=torch.uint8, device=dy.device)
        dx = torch.empty((shape.n, shape.c_in, shape.h, shape.w), dtype=torch.float32, device=dy.device)
        dw = torch.empty((shape.c_out, shape.c_in, 3, 3), dtype=torch.float32, device=dy.device)
        db = torch.empty((shape.c_out,), dtype=torch.float32, device=dy.device) if need_bias else None
        with torch.cuda.device(dy.device):
            _lib.check(_lib.lib().wl_backward(
                self.dplan.handle, ctypes.byref(qs), ctypes.byref(shape), ctypes.c_void_p(dy.data_ptr()),
                ctypes.c_void_p(cache.data_ptr()), ctypes.c_void_p(fwd_ws.data_ptr()), ctypes.c_void_p(dx.data_ptr()),
                ctypes.c_void_p(dw.data_ptr()), ctypes.c_void_p(db.data_ptr() if db is not None else 0),
                ctypes.c_void_p(bws.data_ptr()), nbytes.value, _stream_ptr(dy.device)), "wl_backward")
        return dx, dw, db

    def stats(self):
        """StageStat rows of the last forward (synchronises the stream)."""
        if self._parts is not None:  # forward_split: the groups of every part, in batch order
            return [row for part in self._parts for row in self._stats_of(*part)]
        shape, cache, accbuf, _ = self._last
        return self._stats_of(shape, cache, accbuf)

    def _stats_of(self, shape, cache, accbuf):
        ns = _lib.lib().wl_num_stages(self.dplan.handle)
        groups = shape.n // shape.images_per_group
        arr = (_lib.wl_stage_stat * (groups * ns))()
        qs = qcfg_struct(self.qconfig)
        _lib.check(_lib.lib().wl_read_stats(self.dplan.handle, ctypes.byref(shape), ctypes.byref(qs),
                                            ctypes.c_void_p(cache.data_ptr()),
                                            ctypes.c_void_p(accbuf.data_ptr()), arr, _stream_ptr(accbuf.device)),
                   "wl_read_stats")
        names = STAGE_ORDER[self.mode]
        return [[StageStat(names[i], arr[g * ns + i].bits, arr[g * ns + i].max_abs, arr[g * ns + i].scale)
                 for i in range(ns)] for g in range(groups)]

    def launches(self) -> int:
        shape = self._last[0]
        qs = qcfg_struct(self.qconfig)
        return int(_lib.lib().wl_forward_launches(self.dplan.handle, ctypes.byref(shape), ctypes.byref(qs)))

    def debug_views(self):
        """Views of the materialised codes of the last call in logical layouts:
        c0 [N,H,W,C], V [36,T,C], h [36,T,K], U [36,K,C] (storage is [T][36][Cp] etc.)."""
        shape, cache, ws, whole = self._last
        if not whole:
            raise ValueError("debug_views needs a wl_forward call (not the training forward)")
        off = (ctypes.c_size_t * 4)()
        dims = (ctypes.c_int * 4)()
        qs = qcfg_struct(self.qconfig)
        _lib.check(_lib.lib().wl_debug_layout(self.dplan.handle, ctypes.byref(shape), ctypes.byref(qs), off, dims),
                   "wl_debug_layout")
        Cp, Kp, T, _ = dims[0], dims[1], dims[2], dims[3]
        c0 = ws[off[0]: off[0] + shape.n * shape.h * shape.w * Cp].view(torch.int8).view(shape.n, shape.h, shape.w, Cp)
        V = ws[off[1]: off[1] + 36 * T * Cp].view(torch.int8).view(T, 36, Cp).permute(1, 0, 2)
        hb = 2 if self.qconfig.hadamard_bits > 8 else 1
        hraw = ws[off[2]: off[2] + 36 * T * Kp * hb]
        h = (hraw.view(torch.int16) if hb == 2 else hraw.view(torch.int8)).view(T, 36, Kp).permute(1, 0, 2)
        cin, cout = shape.c_in, shape.c_out
        ucodes = cache[cache.numel() - 36 * Kp * Cp:].view(torch.int8).view(Kp, 36, Cp).permute(1, 0, 2)
        return {"c0": c0[..., :cin], "V": V[..., :cin], "h": h[..., :cout], "U": ucodes[:, :cout, :cin]}


class _QuantWinogradFn(torch.autograd.Function):
    """Forward on the sm_100a path; straight-through-estimator backward."""

    @staticmethod
    def forward(ctx, x, w, bias, runner: QuantWinogradConv, padding: int, scale_groups: str):
        xf = x if x.dtype == torch.float32 else x.float()
        shape = runner._shape(xf, w, padding, scale_groups)
        sv_bytes, _ = runner.train_sizes(shape)
        # only the stage slots + V codes outlive the call; the scratch workspace is the runner's own
        saved = torch.empty(sv_bytes, dtype=torch.uint8, device=x.device)
        y = runner.forward(xf, w, bias=bias, padding=padding, scale_groups=scale_groups, saved=saved)
        shape_, cache = runner._last[0], runner._last[1]
        ctx.runner, ctx.shape, ctx.has_bias = runner, shape_, bias is not None
        ctx.dtypes = (x.dtype, w.dtype, bias.dtype if bias is not None else None)
        ctx.save_for_backward(saved, cache)
        return y

    @staticmethod
    def backward(ctx, dy):
        ws, cache = ctx.saved_tensors
        dx, dw, db = ctx.runner.backward(dy, ctx.shape, cache, ws, ctx.has_bias)
        dx, dw = dx.to(ctx.dtypes[0]), dw.to(ctx.dtypes[1])  # fp32 STE gradients, cast to the operand dtypes
        if db is not None:
            db = db.to(ctx.dtypes[2])
        return dx, dw, db, None, None, None


def winograd_conv2d(x: torch.Tensor, w: torch.Tensor, bias, runner: QuantWinogradConv, padding: int = 1,
                    scale_groups: str = "image") -> torch.Tensor:
    """Differentiable quantized Winograd convolution (3x3, stride 1)."""
    return _QuantWinogradFn.apply(x, w, bias, runner, padding, scale_groups)


class WinogradAwareConv2d(torch.nn.Module):
    """3x3 stride-1 convolution computed by the 8/9-bit quantized Winograd F(4,3) layer
    (canonical or Legendre base) with a straight-through-estimator backward."""

    def __init__(self, in_channels: int, out_channels: int, padding: int = 1, bias: bool = False,
                 mode: str = "legendre", qconfig: QuantConfig | None = None, scale_groups: str = "image",
                 plan: WinogradPlan | None = None):
        super().__init__()
        self.in_channels, self.out_channels, self.padding = in_channels, out_channels, padding
        self.mode, self.scale_groups = mode, scale_groups
        self.qconfig = QuantConfig.uniform(8) if qconfig is None else qconfig
        self.plan = build_plan(4, 3, use_legendre=True) if plan is None else plan
        _require_mode(self.plan, mode)
        self.weight = torch.nn.Parameter(torch.empty(out_channels, in_channels, 3, 3))
        torch.nn.init.kaiming_normal_(self.weight, mode="fan_in", nonlinearity="relu")
        self.bias = torch.nn.Parameter(torch.zeros(out_channels)) if bias else None
        self._runners: dict = {}

    def _runner(self, device) -> QuantWinogradConv:
        r = self._runners.get(device.index)
        if r is None:
            r = QuantWinogradConv(self.plan, self.mode, self.qconfig, device)
            self._runners[device.index] = r
        return r

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return winograd_conv2d(x, self.weight, self.bias, self._runner(x.device), self.padding, self.scale_groups)

    def extra_repr(self) -> str:
        return (f"{self.in_channels}, {self.out_channels}, padding={self.padding}, mode={self.mode}, "
                f"qconfig={self.qconfig}, scale_groups={self.scale_groups}")


_runners: dict = {}


def conv2d_winograd_quantized(x, w, plan: WinogradPlan, mode: str, qconfig: QuantConfig, padding: int = 0,
                              bias=None, scale_groups: str = "image"):
    """Reference-compatible entry point (quantize.py:129-148) running on the GPU."""
    _require_mode(plan, mode)
    as_numpy = isinstance(x, np.ndarray) or isinstance(w, np.ndarray)
    if as_numpy:
        dev = torch.device("cuda", torch.cuda.current_device())
        # the reference copies to contiguous fp64 (pipeline.py:112-113): so does this path, and the
        # fp64 kernels return the reference's fp64 output bit for bit
        x = torch.as_tensor(np.asarray(x, dtype=np.float64), device=dev)
        w = torch.as_tensor(np.asarray(w, dtype=np.float64), device=dev)
        if bias is not None:
            bias = torch.as_tensor(np.asarray(bias, dtype=np.float64), device=dev)
    single = x.dim() == 3
    if single:
        x = x.unsqueeze(0)
    key = (id(plan), mode, qconfig, x.device.index)
    r = _runners.get(key)
    if r is None or r.plan is not plan:
        r = QuantWinogradConv(plan, mode, qconfig, x.device)
        _runners[key] = r
    y = r.forward(x, w, bias=bias, padding=padding, scale_groups=scale_groups)
    st = r.stats()
    stats = st[0] if len(st) == 1 else st
    if single:
        y = y[0]
    if as_numpy:
        y = y.cpu().numpy()
    return y, stats


def conv2d_winograd(x, w, plan: WinogradPlan, mode: str = "canonical", padding: int = 0, bias=None):
    """Float (unquantized) Winograd correlation on the GPU in fp32: the reference's
    ``conv2d_winograd`` (pipeline.py:161-164, run_pipeline with the identity cast), SURVEY §8f row 2.

    x: [c_in, H, W] or [N, c_in, H, W]; w: [c_out, c_in, 3, 3]; CUDA tensors or numpy arrays
    (numpy in -> numpy out, like the reference; computed in fp32 either way).  Zero padding and bias
    follow ``conv2d_winograd_quantized``."""
    _require_mode(plan, mode)
    as_numpy = isinstance(x, np.ndarray) or isinstance(w, np.ndarray)
    dev = torch.device("cuda", torch.cuda.current_device()) if as_numpy else x.device
    x = torch.as_tensor(np.asarray(x) if as_numpy else x, device=dev).float().contiguous()
    w = torch.as_tensor(np.asarray(w) if as_numpy else w, device=dev).float().contiguous()
    single = x.dim() == 3
    if single:
        x = x.unsqueeze(0)
    _check_conv_args(x, w)
    if w.shape[2] != 3:
        raise DimensionError(f"plan is for k=3, weights have k={w.shape[2]}")
    n, cin, h, wd = (int(v) for v in x.shape)
    cout = int(w.shape[0])
    shape = _lib.wl_shape(n, cin, cout, h, wd, int(padding), 1)
    ho, wo = h + 2 * padding - 2, wd + 2 * padding - 2
    if ho < 1 or wo < 1:
        raise DimensionError(f"input {h}x{wd} (pad {padding}) is smaller than the 3x3 kernel")
    if bias is not None:
        bias = torch.as_tensor(np.asarray(bias) if isinstance(bias, np.ndarray) else bias, device=dev).float().contiguous()
        if bias.shape != (cout,):
            raise DimensionError(f"bias must be [{cout}], got {tuple(bias.shape)}")
    dplan = DevicePlan.get(plan, mode, dev)
    nbytes = ctypes.c_size_t()
    _lib.check(_lib.lib().wl_float_workspace_size(dplan.handle, ctypes.byref(shape), ctypes.byref(nbytes)),
               "wl_float_workspace_size")
    ws = torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
    y = torch.empty((n, cout, ho, wo), dtype=torch.float32, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().wl_forward_float(
            dplan.handle, ctypes.byref(shape), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w.data_ptr()),
            ctypes.c_void_p(bias.data_ptr() if bias is not None else 0), ctypes.c_void_p(y.data_ptr()),
            ctypes.c_void_p(ws.data_ptr()), nbytes.value, _stream_ptr(dev)), "wl_forward_float")
    if single:
        y = y[0]
    return y.cpu().numpy() if as_numpy else y


def conv2d_direct_quantized(x, w, qconfig: QuantConfig | None = None, padding: int = 0,
                            scale_groups: str = "image"):
    """Quantized direct-convolution baseline on the GPU: the reference's ``conv2d_direct_quantized``
    (quantize.py:151-160), SURVEY §8f row 3 — fake-quantise x (input_bits) and w (weight_bits),
    correlate in fp64 in the reference's order, fake-quantise the result (output_transform_bits).

    fp64 operands (and numpy arrays, copied to fp64 like the reference) run ``wl_direct_quantized_f64``
    and return the reference's output bit for bit; fp32 CUDA tensors run ``wl_direct_quantized`` (the
    same fp64 computation, result rounded to fp32).  Shapes, padding and ``scale_groups`` follow
    ``conv2d_winograd_quantized``."""
    if qconfig is None:
        qconfig = QuantConfig()
    if scale_groups not in ("image", "batch"):
        raise ValueError(f"scale_groups must be 'image' or 'batch', got {scale_groups!r}")
    as_numpy = isinstance(x, np.ndarray) or isinstance(w, np.ndarray)
    if as_numpy:
        dev = torch.device("cuda", torch.cuda.current_device())
        x = torch.as_tensor(np.asarray(x, dtype=np.float64), device=dev)
        w = torch.as_tensor(np.asarray(w, dtype=np.float64), device=dev)
    single = x.dim() == 3
    if single:
        x = x.unsqueeze(0)
    _check_conv_args(x, w)
    if w.shape[2] != 3:
        raise DimensionError(f"the direct baseline is 3x3, weights have k={w.shape[2]}")
    f64 = x.dtype == torch.float64 or w.dtype == torch.float64
    dt = torch.float64 if f64 else torch.float32
    x, w = x.to(dt).contiguous(), w.to(dt).contiguous()
    n, cin, h, wd = (int(v) for v in x.shape)
    cout = int(w.shape[0])
    ho, wo = h + 2 * padding - 2, wd + 2 * padding - 2
    if padding < 0 or ho < 1 or wo < 1:
        raise DimensionError(f"input {h}x{wd} (pad {padding}) is smaller than the 3x3 kernel")
    shape = _lib.wl_shape(n, cin, cout, h, wd, int(padding), 1 if scale_groups == "image" else n)
    nbytes = ctypes.c_size_t()
    _lib.check(_lib.lib().wl_direct_workspace_size(ctypes.byref(shape), ctypes.byref(nbytes)), "wl_direct_workspace_size")
    ws = torch.empty(nbytes.value, dtype=torch.uint8, device=x.device)
    y = torch.empty((n, cout, ho, wo), dtype=dt, device=x.device)
    fn = _lib.lib().wl_direct_quantized_f64 if f64 else _lib.lib().wl_direct_quantized
    with torch.cuda.device(x.device):
        _lib.check(fn(ctypes.byref(qcfg_struct(qconfig)), ctypes.byref(shape), ctypes.c_void_p(x.data_ptr()),
                      ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                      nbytes.value, _stream_ptr(x.device)), "wl_direct_quantized")
    if single:
        y = y[0]
    return y.cpu().numpy() if as_numpy else y


def conv2d_direct(x, w, padding: int = 0):
    """fp64 direct correlation on the GPU: the reference's ``conv2d_direct`` (reference.py:34-39),
    bit-identical to it (same operation order, _kernels.py:53-66).  The ground truth of the error
    experiment.  x [c_in,H,W] or [N,c_in,H,W], w [c_out,c_in,3,3]; numpy in -> numpy out."""
    as_numpy = isinstance(x, np.ndarray) or isinstance(w, np.ndarray)
    dev = torch.device("cuda", torch.cuda.current_device()) if as_numpy else x.device
    x = torch.as_tensor(np.asarray(x, dtype=np.float64) if as_numpy else x, device=dev).double().contiguous()
    w = torch.as_tensor(np.asarray(w, dtype=np.float64) if as_numpy else w, device=dev).double().contiguous()
    single = x.dim() == 3
    if single:
        x = x.unsqueeze(0)
    _check_conv_args(x, w)
    if w.shape[2] != 3:
        raise DimensionError(f"the GPU direct correlation is 3x3, weights have k={w.shape[2]}")
    n, cin, h, wd = (int(v) for v in x.shape)
    cout = int(w.shape[0])
    ho, wo = h + 2 * padding - 2, wd + 2 * padding - 2
    if padding < 0 or ho < 1 or wo < 1:
        raise DimensionError(f"input {h}x{wd} (pad {padding}) is smaller than the 3x3 kernel")
    shape = _lib.wl_shape(n, cin, cout, h, wd, int(padding), 1)
    nbytes = ctypes.c_size_t()
    _lib.check(_lib.lib().wl_direct_workspace_size(ctypes.byref(shape), ctypes.byref(nbytes)), "wl_direct_workspace_size")
    ws = torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
    y = torch.empty((n, cout, ho, wo), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().wl_direct_f64(ctypes.byref(shape), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                                            ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(ws.data_ptr()), nbytes.value,
                                            _stream_ptr(dev)), "wl_direct_f64")
    if single:
        y = y[0]
    return y.cpu().numpy() if as_numpy else y


def default_plan(use_legendre: bool = True) -> WinogradPlan:
    return build_plan(4, 3, use_legendre=use_legendre)
