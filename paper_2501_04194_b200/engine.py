"""Device execution of compiled formulas and the reference-facing API.

``trace`` is the batched path (the B200 equivalent of ``masking.trace_var``
with leading batch axes, masking.py:308-343, plus ``tape.backward``,
tape.py:114-134): channels are CUDA fp32 tensors ``[B, T]``, the result is a
``[B, T]`` trace whose autograd backward calls ``stlg_backward``.

``robustness_trace`` / ``robustness`` / ``value_and_grad`` /
``eventually_trace`` / ``always_trace`` / ``until_trace`` keep the reference
signatures (masking.py:350-401, autodiff.py:64-107) over host ``NamedSignals``.

The only compute path is libstlg.so on the GPU.  Without a CUDA device (or
without the built library) every entry point raises; nothing falls back to
the CPU.
"""

from __future__ import annotations

import ctypes
import threading
from collections import OrderedDict
from ctypes import byref, c_int32, c_size_t, c_void_p
from dataclasses import dataclass, replace
from typing import Mapping, Optional

import numpy as np
import torch

from . import _lib
from .core import (EmptyWindowError, NamedSignals, SemanticsConfig, ShapeError, SmoothInterval,
                   StepInterval, ValidationError)
from .formula import (Always, Eventually, Pred, Until, smooth_intervals, validate_against,
                      variables)
from .lower import (cfg_key, cfg_struct, check_smooth_nonempty, lower, node_array)

__all__ = ["Compiled", "compile_formula", "trace", "robustness_trace", "robustness",
           "value_and_grad", "Gradients", "eventually_trace", "always_trace", "until_trace"]


# ---------------------------------------------------------------------------
# compiled plans
# ---------------------------------------------------------------------------

class Compiled:
    """A formula compiled for a fixed channel order and config (one stlg_plan)."""

    def __init__(self, f, channel_names, cfg):
        self.lib = _lib.load()
        self.low = lower(f, channel_names)
        self.cfg = cfg
        self.channel_names = tuple(channel_names)
        arr = node_array(self.low)
        cs = cfg_struct(cfg)
        plan = c_void_p()
        _lib.check(self.lib.stlg_compile(arr, len(self.low.nodes), len(channel_names),
                                         len(self.low.smooth), byref(cs), byref(plan)))
        self.plan = plan
        nt, ns, rt = c_int32(), c_int32(), c_int32()
        self.lib.stlg_plan_info(plan, byref(nt), byref(ns), byref(rt))
        self.n_temporal, self.n_slots, self.root_temporal = nt.value, ns.value, rt.value

    def __del__(self):
        plan = getattr(self, "plan", None)
        if plan is not None and plan.value:
            try:
                self.lib.stlg_free(plan)
            except Exception:  # interpreter teardown
                pass

    @property
    def n_smooth(self):
        return len(self.low.smooth)

    def workspace_bytes(self, B, T):
        fb, bb = c_size_t(), c_size_t()
        _lib.check(self.lib.stlg_workspace_bytes(self.plan, B, T, byref(fb), byref(bb)))
        return fb.value, bb.value

    def smooth_params(self, binding=None, eps_override=None):
        out = []
        for iv in self.low.smooth:
            eps = float(iv.eps) if eps_override is None else float(eps_override)
            if binding is None:
                out.append((float(iv.a), float(iv.b), float(iv.c), eps))
            else:
                a, b, c = binding
                out.append((float(a), float(b), float(c), eps))
        return out

    @staticmethod
    def _channel_table(chans):
        tab = (_lib.StlgChannel * max(len(chans), 1))()
        for i, t in enumerate(chans):
            tab[i].ptr = t.data_ptr()
            tab[i].row_stride = t.stride(0)
            tab[i].elem_stride = t.stride(1)
        return tab

    @staticmethod
    def _smooth_table(params):
        tab = (_lib.StlgSmooth * max(len(params), 1))()
        for i, (a, b, c, eps) in enumerate(params):
            tab[i].a, tab[i].b, tab[i].c, tab[i].eps = a, b, c, eps
        return tab

    def forward(self, chans, params, out, fws, stream):
        B, T = out.shape
        _lib.check(self.lib.stlg_forward(self.plan, self._channel_table(chans), B, T,
                                         self._smooth_table(params), out.data_ptr(),
                                         fws.data_ptr(), fws.numel(), stream))

    def backward(self, chans, params, trace, cot, dchans, d_smooth, fws, bws, stream):
        B, T = trace.shape
        gt = (_lib.StlgGrad * max(len(dchans), 1))()
        for i, d in enumerate(dchans):
            if d is None:
                gt[i].ptr = None
            else:
                gt[i].ptr = d.data_ptr()
                gt[i].row_stride = d.stride(0)
                gt[i].elem_stride = d.stride(1)
                gt[i].accumulate = 0  # the library writes every element
        _lib.check(self.lib.stlg_backward(
            self.plan, self._channel_table(chans), B, T, self._smooth_table(params),
            trace.data_ptr(), cot.data_ptr(), gt,
            d_smooth.data_ptr() if d_smooth is not None else None,
            fws.data_ptr(), fws.numel(), bws.data_ptr(), bws.numel(), stream))


# compiled plans, least recently used first; a plan is freed (stlg_free) when it is
# evicted and no live autograd graph still holds it
_PLANS: "OrderedDict" = OrderedDict()
PLAN_CACHE_SIZE = 256
_PLANS_LOCK = threading.Lock()


def compile_formula(f, channel_names, cfg) -> Compiled:
    names = tuple(channel_names)
    try:
        key = (f, names, cfg_key(cfg))
        hash(key)
    except TypeError:  # unhashable duck-typed AST: lower to get a structural key
        key = (lower(f, names).key, names, cfg_key(cfg))
    with _PLANS_LOCK:
        hit = _PLANS.get(key)
        if hit is not None:
            _PLANS.move_to_end(key)
            return hit
    hit = Compiled(f, names, cfg)
    with _PLANS_LOCK:
        _PLANS[key] = hit
        while len(_PLANS) > PLAN_CACHE_SIZE:
            _PLANS.popitem(last=False)
    return hit


# ---------------------------------------------------------------------------
# autograd
# ---------------------------------------------------------------------------

def _stream(dev):
    """The current stream of the tensors' device (the library launches on the current
    device, so callers hold `torch.cuda.device(dev)` around the call)."""
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


# rows per library call: the kernels index rows on grid.y (stlg_forward rejects
# B > 65535); larger batches run as row chunks (rows are independent).
MAX_ROWS_PER_CALL = 65535


def _row_chunks(B):
    return [(r, min(r + MAX_ROWS_PER_CALL, B)) for r in range(0, B, MAX_ROWS_PER_CALL)]


class _TraceFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, comp, params, abc, *chans):
        B, T = chans[0].shape
        dev = chans[0].device
        out = torch.empty((B, T), dtype=torch.float32, device=dev)
        fws_list = []
        bb_list = []
        with torch.cuda.device(dev):
            for r0, r1 in _row_chunks(B):
                fb, bb = comp.workspace_bytes(r1 - r0, T)
                fws = torch.empty(fb, dtype=torch.uint8, device=dev)
                comp.forward([c[r0:r1] for c in chans], params, out[r0:r1], fws, _stream(dev))
                fws_list.append(fws)
                bb_list.append(bb)
        ctx.comp = comp
        ctx.params = params
        ctx.bwd_bytes = bb_list
        ctx.save_for_backward(out, *fws_list, *chans)
        ctx.n_chunks = len(fws_list)
        return out

    @staticmethod
    def backward(ctx, g):
        saved = ctx.saved_tensors
        out = saved[0]
        fws_list = saved[1:1 + ctx.n_chunks]
        chans = saved[1 + ctx.n_chunks:]
        comp = ctx.comp
        B, T = out.shape
        dev = out.device
        g = g.to(torch.float32).contiguous()
        dch = [torch.empty((B, T), dtype=torch.float32, device=dev)
               if ctx.needs_input_grad[3 + i] else None for i in range(len(chans))]
        d_total = None
        with torch.cuda.device(dev):
            for (r0, r1), fws, bb in zip(_row_chunks(B), fws_list, ctx.bwd_bytes):
                d_smooth = None
                # the d/dw pass runs only when a bound (a, b, c) tensor asks for its gradient
                if comp.n_smooth and ctx.needs_input_grad[2]:
                    d_smooth = torch.zeros(3 * comp.n_smooth, dtype=torch.float64, device=dev)
                bws = torch.empty(bb, dtype=torch.uint8, device=dev)
                comp.backward([c[r0:r1] for c in chans], ctx.params, out[r0:r1], g[r0:r1],
                              [d[r0:r1] if d is not None else None for d in dch], d_smooth, fws, bws,
                              _stream(dev))
                if d_smooth is not None:
                    d_total = d_smooth if d_total is None else d_total + d_smooth
        dabc = None
        if ctx.needs_input_grad[2] and d_total is not None:
            dabc = d_total.view(-1, 3).sum(0)
        return (None, None, dabc, *dch)


def _as_rows(t, name):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"channel {name!r} must be a torch tensor")
    if not t.is_cuda:
        raise RuntimeError(f"channel {name!r} must live on a CUDA device (no CPU path)")
    if t.dtype != torch.float32:
        t = t.float()
    if t.dim() == 1:
        t = t.unsqueeze(0)
    if t.dim() != 2:
        raise ShapeError(f"channel {name!r} must be [B, T] or [T], got {tuple(t.shape)}")
    return t


def trace(f, channels: Mapping[str, torch.Tensor], cfg: SemanticsConfig = SemanticsConfig(),
          smooth_binding=None) -> torch.Tensor:
    """Robustness trace ``[B, T]`` of ``f`` over CUDA fp32 channels (differentiable).

    ``smooth_binding=(a, b, c)`` (floats or tensors) rebinds every smooth-interval
    node's parameters (masking.py:313-315); tensor entries receive gradients.
    """
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2501_04194_b200 requires a CUDA device; there is no CPU path")
    missing = validate_against(f, list(channels))
    if missing:
        raise ValidationError(missing)
    names = sorted(variables(f))
    if not names:  # formula without predicates (TRUE): still needs a shape
        names = [next(iter(channels))]
    chans = [_as_rows(channels[n], n) for n in names]
    shape = chans[0].shape
    if any(c.shape != shape for c in chans):
        raise ShapeError(f"channel shapes differ: {[tuple(c.shape) for c in chans]}")
    if shape[1] == 0 or shape[0] == 0:
        raise ShapeError("signals must be non-empty")
    comp = compile_formula(f, names, cfg)
    abc = None
    binding_vals = None
    if smooth_binding is not None and comp.n_smooth:
        vals = []
        tensors = []
        for v in smooth_binding:
            if isinstance(v, torch.Tensor):
                tensors.append(v)
                vals.append(float(v.detach().double().cpu().item()))
            else:
                vals.append(float(v))
        binding_vals = tuple(vals)
        if tensors and any(t.requires_grad for t in tensors):
            abc = torch.stack([torch.as_tensor(v, dtype=torch.float64, device=chans[0].device)
                               if not isinstance(v, torch.Tensor) else v.to(torch.float64).reshape(())
                               for v in smooth_binding])
    params = comp.smooth_params(binding_vals)
    check_smooth_nonempty(params, shape[1])
    if abc is None:
        return _TraceFn.apply(comp, params, None, *chans)
    return _TraceFn.apply(comp, params, abc, *chans)


# ---------------------------------------------------------------------------
# reference-shaped host API
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Gradients:
    """Robustness value with its gradients (autodiff.py:26-38)."""

    value: float
    d_signal: dict
    d_a: Optional[float] = None
    d_b: Optional[float] = None
    d_c: Optional[float] = None


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2501_04194_b200 requires a CUDA device; there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def _upload(signals: NamedSignals, names):
    dev = _device()
    return {n: torch.as_tensor(np.asarray(signals[n].values, dtype=np.float32), device=dev)[None, :]
            for n in names}


def robustness_trace(f, signals: NamedSignals, cfg: SemanticsConfig = SemanticsConfig()) -> np.ndarray:
    """Robustness of every suffix (masking.py:350-357); float64 array of fp32 values."""
    missing = validate_against(f, signals)
    if missing:
        raise ValidationError(missing)
    names = sorted(variables(f)) or [signals.names()[0]]
    with torch.no_grad():
        out = trace(f, _upload(signals, names), cfg)
    return out[0].double().cpu().numpy()


def robustness(f, signals: NamedSignals, cfg: SemanticsConfig = SemanticsConfig()) -> float:
    """Entry 0 of the trace (masking.py:360-363)."""
    return float(robustness_trace(f, signals, cfg)[0])


def _rebind(f, si):
    k = type(f).__name__
    if k in ("Eventually", "Always"):
        iv = si if type(f.interval).__name__ == "SmoothInterval" else f.interval
        return replace(f, arg=_rebind(f.arg, si), interval=iv)
    if k == "Not":
        return replace(f, arg=_rebind(f.arg, si))
    if k in ("And", "Or", "Until"):
        return replace(f, left=_rebind(f.left, si), right=_rebind(f.right, si))
    return f


def value_and_grad(f, signals: NamedSignals, cfg: SemanticsConfig = SemanticsConfig(),
                   si: Optional[SmoothInterval] = None) -> Gradients:
    """Robustness (entry 0) and its gradients (autodiff.py:64-107)."""
    missing = validate_against(f, signals)
    if missing:
        raise ValidationError(missing)
    sis = smooth_intervals(f)
    if si is not None:
        if not sis:
            raise ValueError("formula has no smooth-interval node to bind")
        f = _rebind(f, si)
        target = si
    elif sis:
        if len(set(sis)) > 1:
            raise ValueError("multiple distinct smooth intervals; pass si= to bind them")
        target = sis[0]
    else:
        target = None
    dev = _device()
    names = signals.names()
    used = sorted(variables(f))
    chans = {n: torch.as_tensor(np.asarray(signals[n].values, dtype=np.float32), device=dev)[None, :]
             .requires_grad_(True) for n in used}
    binding = None
    abc = None
    if target is not None:
        abc = [torch.tensor(float(v), dtype=torch.float64, device=dev, requires_grad=True)
               for v in (target.a, target.b, target.c)]
        binding = tuple(abc)
    if not used:
        feed = {names[0]: torch.zeros((1, signals.length), device=dev)}
    else:
        feed = chans
    out = trace(f, feed, cfg, smooth_binding=binding)
    value = out[0, 0]
    leaves = list(chans.values()) + (abc or [])
    grads = torch.autograd.grad(value, leaves, allow_unused=True) if leaves and value.requires_grad \
        else [None] * len(leaves)
    d_signal = {}
    for n in names:
        if n in chans:
            g = grads[used.index(n)]
            d_signal[n] = (g[0].double().cpu().numpy() if g is not None
                           else np.zeros(signals.length))
        else:
            d_signal[n] = np.zeros(signals.length)
    res = Gradients(value=float(value.detach().cpu()), d_signal=d_signal)
    if abc is not None:
        ga = grads[len(chans):]
        res = replace(res, d_a=float(ga[0]) if ga[0] is not None else 0.0,
                      d_b=float(ga[1]) if ga[1] is not None else 0.0,
                      d_c=float(ga[2]) if ga[2] is not None else 0.0)
    return res


def _as_trace(values, name):
    arr = np.asarray(values, dtype=np.float64).reshape(-1)
    if arr.size == 0:
        raise ShapeError(f"{name} trace must be non-empty")
    return arr


def _trace_op(node, arrays, cfg):
    dev = _device()
    feed = {k: torch.as_tensor(v.astype(np.float32), device=dev)[None, :] for k, v in arrays.items()}
    with torch.no_grad():
        return trace(node, feed, cfg)[0].double().cpu().numpy()


def eventually_trace(inner, iv, cfg: SemanticsConfig = SemanticsConfig()) -> np.ndarray:
    """Windowed max over a trace (masking.py:377-382).  ``x > 0.0`` is the identity."""
    arr = _as_trace(inner, "inner")
    return _trace_op(Eventually(Pred("u_", ">", 0.0), iv), {"u_": arr}, cfg)


def always_trace(inner, iv, cfg: SemanticsConfig = SemanticsConfig()) -> np.ndarray:
    """Windowed min over a trace (masking.py:385-390)."""
    arr = _as_trace(inner, "inner")
    return _trace_op(Always(Pred("u_", ">", 0.0), iv), {"u_": arr}, cfg)


def until_trace(left, right, iv, cfg: SemanticsConfig = SemanticsConfig()) -> np.ndarray:
    """Until over two traces (masking.py:393-401)."""
    l_arr = _as_trace(left, "left")
    r_arr = _as_trace(right, "right")
    if l_arr.size != r_arr.size:
        raise ShapeError(f"trace lengths differ: {l_arr.size} vs {r_arr.size}")
    if iv is not None and type(iv).__name__ == "SmoothInterval":
        raise TypeError("until does not support smooth intervals")
    return _trace_op(Until(Pred("l_", ">", 0.0), Pred("r_", ">", 0.0), iv),
                     {"l_": l_arr, "r_": r_arr}, cfg)
