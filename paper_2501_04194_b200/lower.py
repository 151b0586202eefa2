"""Lower a formula AST to the flat node program of ``stlg_compile``.

Mirrors the recursion of ``masking.trace_var`` (masking.py:308-343) once per
formula instead of once per call.  Structurally equal sub-formulas are
merged (hash-consing), so a shared temporal sub-formula is evaluated once;
values are unchanged and gradients are summed, as the reference tape does.

Node classes are matched by *name* and fields, so ASTs built with the
reference package (``stlmask.formula``) lower exactly like this package's.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import EmptyWindowError

_OPS = {"TrueFormula": _lib.OP_TRUE, "Pred": _lib.OP_PRED, "Not": _lib.OP_NOT,
        "And": _lib.OP_AND, "Or": _lib.OP_OR, "Eventually": _lib.OP_EV, "Always": _lib.OP_AL,
        "Until": _lib.OP_UNTIL, "NormPred": _lib.OP_NORM}


@dataclass
class Lowered:
    nodes: list            # list of dicts (field values of StlgNode)
    channels: tuple        # channel names, in program index order
    smooth: list           # distinct SmoothInterval objects, by slot
    key: tuple             # structural key (plan cache)


def _kind(f):
    return type(f).__name__


def _iv_key(iv):
    if iv is None:
        return None
    k = _kind(iv)
    if k == "StepInterval":
        return ("step", int(iv.a), int(iv.b))
    if k == "SmoothInterval":
        return ("smooth", float(iv.a), float(iv.b), float(iv.c), float(iv.eps))
    raise TypeError(f"unsupported interval: {iv!r}")


def lower(f, channel_names) -> Lowered:
    """Flatten ``f`` (children first).  ``channel_names`` fixes channel indices."""
    chan_index = {n: i for i, n in enumerate(channel_names)}
    nodes: list = []
    memo: dict = {}
    smooth: list = []
    smooth_idx: dict = {}

    def visit(g):
        k = _kind(g)
        if k not in _OPS:
            raise TypeError(f"not a Formula node: {g!r}")
        nd = dict(op=_OPS[k], left=-1, right=-1, chan=-1, chan2=-1, cmp=0, threshold=0.0,
                  center0=0.0, center1=0.0, itv_kind=_lib.ITV_NONE, a=0, b=0, smooth_slot=-1)
        if k == "Pred":
            nd.update(chan=chan_index[g.var], cmp=0 if g.cmp in (">", ">=") else 1,
                      threshold=float(g.threshold))
            key = ("P", nd["chan"], nd["cmp"], nd["threshold"])
        elif k == "NormPred":
            nd.update(chan=chan_index[g.vars[0]], chan2=chan_index[g.vars[1]],
                      cmp=0 if g.cmp in (">", ">=") else 1, threshold=float(g.threshold),
                      center0=float(g.center[0]), center1=float(g.center[1]))
            key = ("N", nd["chan"], nd["chan2"], nd["cmp"], nd["threshold"], nd["center0"],
                   nd["center1"])
        elif k == "TrueFormula":
            key = ("T",)
        elif k == "Not":
            nd["left"] = visit(g.arg)
            key = ("~", nd["left"])
        elif k in ("And", "Or", "Until"):
            nd["left"] = visit(g.left)
            nd["right"] = visit(g.right)
            ivk = None
            if k == "Until":
                ivk = _iv_key(g.interval)
                if ivk is not None and ivk[0] == "smooth":
                    raise TypeError("until does not support smooth intervals")
                if ivk is not None:
                    nd.update(itv_kind=_lib.ITV_STEP, a=ivk[1], b=ivk[2])
            key = (k, nd["left"], nd["right"], ivk)
        else:  # Eventually / Always
            nd["left"] = visit(g.arg)
            ivk = _iv_key(g.interval)
            if ivk is not None:
                if ivk[0] == "step":
                    nd.update(itv_kind=_lib.ITV_STEP, a=ivk[1], b=ivk[2])
                else:
                    if ivk not in smooth_idx:
                        smooth_idx[ivk] = len(smooth)
                        smooth.append(g.interval)
                    nd.update(itv_kind=_lib.ITV_SMOOTH, smooth_slot=smooth_idx[ivk])
            key = (k, nd["left"], ivk)
        if key in memo:
            return memo[key]
        nodes.append(nd)
        memo[key] = len(nodes) - 1
        return len(nodes) - 1

    root = visit(f)
    if root != len(nodes) - 1:  # root merged with an earlier node: re-append it as the last node
        nodes.append(dict(nodes[root]))
    key = tuple(tuple(sorted(n.items())) for n in nodes)
    return Lowered(nodes, tuple(channel_names), smooth, key)


def node_array(low: Lowered):
    arr = (_lib.StlgNode * len(low.nodes))()
    for i, nd in enumerate(low.nodes):
        for k, v in nd.items():
            setattr(arr[i], k, v)
    return arr


def cfg_struct(cfg) -> _lib.StlgCfg:
    m = _kind(cfg.mode)
    mode = {"Hard": _lib.MODE_HARD, "SoftMax": _lib.MODE_SOFTMAX, "LogSumExp": _lib.MODE_LSE}.get(m)
    if mode is None:
        raise TypeError(f"unsupported mode: {cfg.mode!r}")
    s = _lib.StlgCfg()
    s.mode = mode
    s.temp = float(getattr(cfg.mode, "temp", 1.0))
    s.pad_last = 1 if cfg.padding.kind == "last" else 0
    s.pad_value = float(cfg.padding.value)
    s.top_value = float(cfg.top_value)
    s.sentinel = float(cfg.sentinel)
    s.masked_fill = 1 if cfg.masked_fill else 0
    return s


def cfg_key(cfg) -> tuple:
    return (_kind(cfg.mode), float(getattr(cfg.mode, "temp", 1.0)), cfg.padding.kind,
            float(cfg.padding.value), float(cfg.top_value), float(cfg.sentinel),
            bool(cfg.masked_fill))


# ---------------------------------------------------------------------------
# smooth-interval weights (host, fp64) — only for the empty-window check and
# the kept range; the device recomputes the table itself
# ---------------------------------------------------------------------------

def _sigmoid(z):
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


def smooth_weights_np(a, b, c, eps, length):
    """``relu(sigmoid(c (i - a L)) - sigmoid(c (i - b L)) - eps)`` (smoothing.py:85-97)."""
    i = np.arange(length, dtype=np.float64)
    pre = _sigmoid((i - a * float(length)) * c) - _sigmoid((i - b * float(length)) * c) - eps
    return np.where(pre > 0, pre, 0.0)


def check_smooth_nonempty(params, length):
    for a, b, c, eps in params:
        if not np.any(smooth_weights_np(a, b, c, eps, length) > 0):
            raise EmptyWindowError("smooth interval produced an all-zero weight vector")
