"""CPU oracle for the masked-STL robustness path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
(``cpu_baseline`` / ``--impl reference``) may import this module, and only
as the checker or the timed CPU baseline.  The product path
(``paper_2501_04194_b200``) never imports it and fails loudly when the CUDA
library is missing.

What it is: a float64 numpy restatement of the reference's masking engine
and its reverse-mode gradients, written from the semantics, not copied:

* predicate / negation / And / Or           masking.py:316-330, tape.py:338-391
* timed F/G + padding + overrun rule        masking.py:155-192, 229-235
* untimed F/G (suffix scans, softmax L x L) masking.py:217-227, tape.py:475-535
* smooth-interval F/G (sigmoid weights)     masking.py:207-215, 300-305; smoothing.py:85-109
* Until, timed and untimed                  masking.py:238-293
* masked_fill compatibility                 masking.py:195-202, 94-148
* value_and_grad                            autodiff.py:64-107

It carries its own small tape (``_Tape``): each primitive records the VJP
closures that route a cotangent to its inputs; ``backward`` replays them
in reverse creation order.  Reductions follow the reference exactly: hard
max selects the FIRST maximal entry (ties to the lower index), smooth
reductions shift by the detached hard max over kept entries.

Parity pin: ``tests/golden/`` holds vectors produced by the reference
itself (``tests/golden/make_golden.py``); ``tests/test_oracle_golden.py``
checks this module against them (hard mode value-exact, smooth 1e-12).

The ``NormPred`` extension node is evaluated as ``sqrt(dx*dx + dy*dy)``
with no epsilon, matching SURVEY §8(d) C2.
"""

from __future__ import annotations

import math

import numpy as np

__all__ = ["trace", "trace_and_grad", "value_and_grad", "smooth_weights"]


# ---------------------------------------------------------------------------
# configuration access (duck-typed: works for this package's and stlmask's types)
# ---------------------------------------------------------------------------

def _mode(cfg):
    name = type(cfg.mode).__name__
    if name == "Hard":
        return "hard", None
    if name == "LogSumExp":
        return "lse", float(cfg.mode.temp)
    if name == "SoftMax":
        return "softmax", float(cfg.mode.temp)
    raise TypeError(f"unsupported mode: {cfg.mode!r}")


def _kind(obj):
    return type(obj).__name__


# ---------------------------------------------------------------------------
# a minimal reverse-mode tape
# ---------------------------------------------------------------------------

class _Node:
    __slots__ = ("val", "grad", "leaf")

    def __init__(self, val, leaf=False):
        self.val = np.asarray(val, dtype=np.float64)
        self.grad = None
        self.leaf = leaf


class _Tape:
    def __init__(self):
        self.entries = []  # (out_node, [(parent_node, vjp)])

    def record(self, out, links):
        links = [(p, fn) for p, fn in links if p is not None and not _is_const(p)]
        if links:
            self.entries.append((out, links))
        return out

    def backward(self, out, seed):
        out.grad = np.asarray(seed, dtype=np.float64).copy()
        for node, links in reversed(self.entries):
            if node.grad is None:
                continue
            g = node.grad
            for parent, fn in links:
                contrib = fn(g)
                parent.grad = contrib if parent.grad is None else parent.grad + contrib


def _const(val):
    n = _Node(val)
    n.leaf = "const"
    return n


def _is_const(n):
    return n.leaf == "const"


# ---------------------------------------------------------------------------
# primitives
# ---------------------------------------------------------------------------

def _add_scalar(T, x, c):
    return T.record(_Node(x.val + c), [(x, lambda g: g)])


def _neg(T, x):
    return T.record(_Node(-x.val), [(x, lambda g: -g)])


def _add(T, x, y):
    return T.record(_Node(x.val + y.val), [(x, lambda g: g), (y, lambda g: g)])


def _norm(T, x, y, cx, cy):
    dx = x.val - cx
    dy = y.val - cy
    d = np.sqrt(dx * dx + dy * dy)
    with np.errstate(divide="ignore", invalid="ignore"):
        ux = np.where(d > 0, dx / d, 0.0)
        uy = np.where(d > 0, dy / d, 0.0)
    return T.record(_Node(d), [(x, lambda g: g * ux), (y, lambda g: g * uy)])


def _stack(T, xs):
    out = _Node(np.stack([x.val for x in xs], axis=-1))
    links = [(x, (lambda i: (lambda g: g[..., i]))(i)) for i, x in enumerate(xs)]
    return T.record(out, links)


def _concat(T, xs):
    out = _Node(np.concatenate([x.val for x in xs], axis=-1))
    bounds = np.cumsum([0] + [x.val.shape[-1] for x in xs])
    links = [(x, (lambda lo, hi: (lambda g: g[..., lo:hi]))(bounds[i], bounds[i + 1]))
             for i, x in enumerate(xs)]
    return T.record(out, links)


def _index(T, x, i):
    """x[..., i] for a fixed integer i."""
    width = x.val.shape[-1]

    def vjp(g):
        acc = np.zeros(g.shape + (width,))
        acc[..., i] = g
        return acc
    return T.record(_Node(x.val[..., i]), [(x, vjp)])


def _gather(T, x, idx):
    """x[..., idx] for an integer index array of any shape."""
    idx = np.asarray(idx, dtype=np.intp)
    width = x.val.shape[-1]
    lead = x.val.shape[:-1]

    def vjp(g):
        rows = int(np.prod(lead, dtype=np.intp)) if lead else 1
        gf = g.reshape(rows, idx.size)
        acc = np.zeros((rows, width))
        flat = idx.ravel()
        _scatter_rows(acc, flat, gf)
        return acc.reshape(lead + (width,))
    return T.record(_Node(np.take(x.val, idx, axis=-1)), [(x, vjp)])


def _scatter_rows(acc, flat, gf):
    # sum columns that share a destination, then add once per destination
    order = np.argsort(flat, kind="stable")
    dst = flat[order]
    sums = np.add.reduceat(gf[:, order], np.flatnonzero(np.r_[True, dst[1:] != dst[:-1]]), axis=1)
    uniq = dst[np.r_[True, dst[1:] != dst[:-1]]]
    acc[:, uniq] += sums


def _window(T, x, a, K):
    """Sliding windows: out[..., t, k] = x[..., t + a + k], t = 0..n-a-K."""
    n = x.val.shape[-1]
    count = n - a - K + 1
    view = np.lib.stride_tricks.sliding_window_view(x.val[..., a:], K, axis=-1)[..., :count, :]

    def vjp(g):
        acc = np.zeros(x.val.shape)
        for k in range(K):
            acc[..., a + k:a + k + count] += g[..., :, k]
        return acc
    return T.record(_Node(np.array(view)), [(x, vjp)])


def _mask_fill(T, x, keep, fill):
    keep = np.asarray(keep, dtype=bool)
    out = _Node(np.where(keep, x.val, fill))
    return T.record(out, [(x, lambda g: _unbroadcast(g * keep, x.val.shape))])


def _unbroadcast(g, shape):
    if g.shape == tuple(shape):
        return g
    extra = g.ndim - len(shape)
    if extra:
        g = g.sum(axis=tuple(range(extra)))
    axes = tuple(i for i, n in enumerate(shape) if n == 1 and g.shape[i] != 1)
    return g.sum(axis=axes, keepdims=True) if axes else g


def _broadcast_last(T, x, length):
    """x[..., None] * ones(length) (masking.py:189)."""
    out = _Node(x.val[..., None] * np.ones(length))
    return T.record(out, [(x, lambda g: g.sum(axis=-1))])


# ---------------------------------------------------------------------------
# reductions along the last axis (tape.py:338-391 semantics)
# ---------------------------------------------------------------------------

def _reduce_max(T, x, mode, tau, w=None, wnode=None):
    """Max-type reduction; w (last-axis weights) selects kept entries (w > 0)."""
    xv = x.val
    if w is not None:
        kept = np.broadcast_to(w > 0, xv.shape)
        masked = np.where(kept, xv, -np.inf)
    else:
        kept = None
        masked = xv
    sel = np.argmax(masked, axis=-1)
    m = np.take_along_axis(masked, sel[..., None], axis=-1)[..., 0]
    if not np.all(np.isfinite(m)):
        raise _empty("hard reduction over a window with no kept entries")
    if mode == "hard":
        def vjp_h(g):
            acc = np.zeros(xv.shape)
            np.put_along_axis(acc, sel[..., None], g[..., None], axis=-1)
            return acc
        return T.record(_Node(m), [(x, vjp_h)])
    z = (xv - m[..., None]) * tau
    if kept is not None:
        z = np.where(kept, z, -np.inf)
    ez = np.exp(z)
    e = ez * w if w is not None else ez
    s = e.sum(axis=-1)
    if not np.all(s > 0):
        raise _empty(f"{mode} reduction over an all-zero-weight window")
    if mode == "lse":
        out = np.log(s) * (1.0 / tau) + m
        p = e / s[..., None]                      # d out / d x

        def vjp_x(g):
            return g[..., None] * p

        def vjp_w(g):
            return _unbroadcast(g[..., None] * ez / (tau * s[..., None]), wnode.val.shape)
    else:
        num = (xv * e).sum(axis=-1)
        out = num / s
        dev = xv - out[..., None]
        p = e / s[..., None] * (1.0 + tau * dev)

        def vjp_x(g):
            return g[..., None] * p

        def vjp_w(g):
            return _unbroadcast(g[..., None] * ez * dev / s[..., None], wnode.val.shape)
    links = [(x, vjp_x)]
    if wnode is not None:
        links.append((wnode, vjp_w))
    return T.record(_Node(out), links)


def _reduce(T, x, kind, mode, tau, w=None, wnode=None):
    if kind == "max":
        return _reduce_max(T, x, mode, tau, w, wnode)
    # min = -max(-x); weight gradients flip sign through the outer negation
    return _neg(T, _reduce_max(T, _neg(T, x), mode, tau, w, wnode))


def _empty(msg):
    try:
        from paper_2501_04194_b200.core import EmptyWindowError
    except Exception:  # pragma: no cover
        EmptyWindowError = RuntimeError
    return EmptyWindowError(msg)


# ---------------------------------------------------------------------------
# smooth interval weights (masking.py:300-305, smoothing.py:85-109)
# ---------------------------------------------------------------------------

def _sigmoid(z):
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


def smooth_weights(a, b, c, eps, length):
    """Weights and their partials: w, dw/da, dw/db, dw/dc (all float64, shape (L,))."""
    i = np.arange(length, dtype=np.float64)
    lo = _sigmoid((i - a * float(length)) * c)
    hi = _sigmoid((i - b * float(length)) * c)
    pre = lo - hi - eps
    w = np.where(pre > 0, pre, 0.0)
    on = pre > 0
    slo = lo * (1.0 - lo)
    shi = hi * (1.0 - hi)
    dwa = np.where(on, -slo * c * length, 0.0)
    dwb = np.where(on, shi * c * length, 0.0)
    dwc = np.where(on, slo * (i - a * length) - shi * (i - b * length), 0.0)
    return w, dwa, dwb, dwc


# ---------------------------------------------------------------------------
# evaluator
# ---------------------------------------------------------------------------

class _Ctx:
    def __init__(self, channels, length, cfg, binding):
        self.T = _Tape()
        self.ch = channels
        self.L = length
        self.cfg = cfg
        self.mode, self.tau = _mode(cfg)
        self.binding = binding          # (a, b, c) floats or None
        self.eps_override = None        # si.eps when value_and_grad rebinds
        self.wnodes = []                # (node, eps) of bound smooth weights
        lead = next(iter(channels.values())).val.shape[:-1] if channels else ()
        self.lead = lead


def _pad(ctx, x, count):
    """Append ``count`` virtual samples (masking.py:155-161)."""
    if count == 0:
        return x
    if ctx.cfg.padding.kind == "last":
        tail = _gather(ctx.T, x, np.full(count, ctx.L - 1, dtype=np.intp))
        return _concat(ctx.T, [x, tail])
    fill = _const(np.full(x.val.shape[:-1] + (count,), float(ctx.cfg.padding.value)))
    return _concat(ctx.T, [x, fill])


def _pad_value(ctx, x):
    if ctx.cfg.padding.kind == "last":
        return _index(ctx.T, x, ctx.L - 1)
    return _const(np.full(x.val.shape[:-1], float(ctx.cfg.padding.value)))


def _overrun(ctx, out, upper, pv):
    """Entries with t + upper > L - 1 become the pad value (masking.py:180-192)."""
    if upper == 0:
        return out
    L = ctx.L
    keep = np.arange(L) < L - upper
    repl = _broadcast_last(ctx.T, pv, L)
    if not keep.any():
        return repl
    return _add(ctx.T, _mask_fill(ctx.T, out, keep, 0.0), _mask_fill(ctx.T, repl, ~keep, 0.0))


def _fill_columns(ctx, padded, keep, kind):
    """masked_fill: reduce full sentinel-filled columns (masking.py:195-202)."""
    rows = padded.val.shape[-1]
    idx = np.broadcast_to(np.arange(rows), (keep.shape[1], rows))
    cols = _gather(ctx.T, padded, idx)
    fill = -ctx.cfg.sentinel if kind == "max" else ctx.cfg.sentinel
    return _reduce(ctx.T, _mask_fill(ctx.T, cols, keep.T, fill), kind, ctx.mode, ctx.tau)


def _sub_mask(length, rows):
    return np.arange(rows)[:, None] >= np.arange(length)[None, :]


def _time_mask(length, a, b):
    r = np.arange(length + b)[:, None]
    t = np.arange(length)[None, :]
    return (r >= t + a) & (r <= t + b)


def _smooth_weights_node(ctx, iv):
    L = ctx.L
    if ctx.binding is not None:
        a, b, c = ctx.binding
        eps = iv.eps if ctx.eps_override is None else ctx.eps_override
        w = smooth_weights(a, b, c, eps, L)[0]
        node = _Node(w, leaf=True)
        ctx.wnodes.append((node, eps))
        return w, node
    w = smooth_weights(iv.a, iv.b, iv.c, iv.eps, L)[0]
    return w, None


def _ev_al(ctx, child, iv, kind):
    T, L = ctx.T, ctx.L
    ivk = _kind(iv) if iv is not None else None
    if ivk == "SmoothInterval":
        padded = _pad(ctx, child, L - 1)
        win = _window(T, padded, 0, L)
        w, wnode = _smooth_weights_node(ctx, iv)
        if not np.any(w > 0):
            raise _empty("smooth interval produced an all-zero weight vector")
        return _reduce(T, win, kind, ctx.mode, ctx.tau, w=w, wnode=wnode)
    if iv is None:
        if ctx.cfg.masked_fill:
            return _fill_columns(ctx, child, _sub_mask(L, L), kind)
        if ctx.mode == "softmax":
            pos = np.arange(L)[:, None] + np.arange(L)[None, :]
            win = _gather(T, child, np.minimum(pos, L - 1))
            return _reduce(T, win, kind, ctx.mode, ctx.tau, w=(pos <= L - 1).astype(np.float64))
        return _suffix(ctx, child, kind)
    a, b = iv.a, iv.b
    padded = _pad(ctx, child, b)
    if ctx.cfg.masked_fill:
        keep = _sub_mask(L, L + b) & _time_mask(L, a, b)
        return _fill_columns(ctx, padded, keep, kind)
    win = _window(T, padded, a, b - a + 1)          # (..., L, K)
    out = _reduce(T, win, kind, ctx.mode, ctx.tau)
    return _overrun(ctx, out, b, _pad_value(ctx, child))


def _suffix(ctx, child, kind):
    """Untimed hard / LSE F,G as suffix scans (tape.py:475-535)."""
    T = ctx.T
    x = child if kind == "max" else _neg(T, child)
    xv = x.val
    L = xv.shape[-1]
    if ctx.mode == "hard":
        sel = np.empty(xv.shape, dtype=np.intp)
        best = xv[..., -1].copy()
        bidx = np.full(xv.shape[:-1], L - 1, dtype=np.intp)
        sel[..., -1] = L - 1
        for t in range(L - 2, -1, -1):
            upd = xv[..., t] >= best
            best = np.where(upd, xv[..., t], best)
            bidx = np.where(upd, t, bidx)
            sel[..., t] = bidx
        val = np.take_along_axis(xv, sel, axis=-1)

        def vjp(g):
            lead = xv.shape[:-1]
            rows = int(np.prod(lead, dtype=np.intp)) if lead else 1
            acc = np.zeros((rows, L))
            np.add.at(acc, (np.arange(rows)[:, None], sel.reshape(rows, L)), g.reshape(rows, L))
            return acc.reshape(xv.shape)
        out = T.record(_Node(val), [(x, vjp)])
    else:
        tau = ctx.tau
        data = np.flip(np.logaddexp.accumulate(np.flip(tau * xv, axis=-1), axis=-1), axis=-1) / tau

        def vjp(g):
            grad = np.empty_like(xv)
            acc = g[..., 0].copy()
            grad[..., 0] = np.exp(tau * (xv[..., 0] - data[..., 0])) * acc
            for j in range(1, L):
                acc = g[..., j] + np.exp(tau * (data[..., j] - data[..., j - 1])) * acc
                grad[..., j] = np.exp(tau * (xv[..., j] - data[..., j])) * acc
            return grad
        out = T.record(_Node(data), [(x, vjp)])
    return out if kind == "max" else _neg(T, out)


def _hard_min_pair(ctx, x, y):
    T = ctx.T
    return _neg(T, _reduce_max(T, _stack(T, [_neg(T, x), _neg(T, y)]), "hard", None))


def _until(ctx, left, right, iv):
    T, L, mode, tau = ctx.T, ctx.L, ctx.mode, ctx.tau
    if iv is not None and _kind(iv) == "SmoothInterval":
        raise TypeError("until does not support smooth intervals")
    if iv is None:
        a, count = 0, L
        outer_keep = (np.arange(L)[:, None] + np.arange(count)[None, :]) <= L - 1
        lp, rp = left, right
    else:
        a, count = iv.a, iv.b - iv.a + 1
        outer_keep = None
        lp = _pad(ctx, left, iv.b)
        rp = _pad(ctx, right, iv.b)
    t = np.arange(L)
    last = lp.val.shape[-1] - 1
    if ctx.cfg.masked_fill:
        keep_l, keep_r = _until_masks(L, iv)
        terms = []
        for k in range(count):
            pm = _fill_columns(ctx, lp, keep_l[:, :, k], "min")
            rv = _fill_columns(ctx, rp, keep_r[:, :, k], "min")
            terms.append(_reduce(T, _stack(T, [pm, rv]), "min", mode, tau))
        st = _stack(T, terms)
        if outer_keep is not None:
            st = _mask_fill(T, st, outer_keep, -ctx.cfg.sentinel)
        return _reduce(T, st, "max", mode, tau)
    terms = []
    pm = None
    for k in range(count):
        end = np.minimum(t + a + k, last)
        if mode != "softmax":
            lv = _gather(T, lp, end)
            if pm is None:
                if a == 0:
                    pm = lv
                else:
                    idx = np.minimum(t[:, None] + np.arange(a + 1)[None, :], last)
                    pm = _reduce(T, _gather(T, lp, idx), "min", mode, tau)
            else:
                pm = _reduce(T, _stack(T, [pm, lv]), "min", mode, tau)
        else:
            idx = np.minimum(t[:, None] + np.arange(a + k + 1)[None, :], last)
            pm = _reduce(T, _gather(T, lp, idx), "min", mode, tau)
        rv = _gather(T, rp, end)
        terms.append(_reduce(T, _stack(T, [pm, rv]), "min", mode, tau))
    st = _stack(T, terms)
    w = outer_keep.astype(np.float64) if outer_keep is not None else None
    out = _reduce(T, st, "max", mode, tau, w=w)
    if iv is None:
        return out
    pv = _hard_min_pair(ctx, _pad_value(ctx, left), _pad_value(ctx, right))
    return _overrun(ctx, out, iv.b, pv)


def _until_masks(length, iv):
    if iv is None:
        a, count, rows = 0, length, length
    else:
        a, count, rows = iv.a, iv.b - iv.a + 1, length + iv.b
    r = np.arange(rows)[:, None, None]
    t = np.arange(length)[None, :, None]
    k = np.arange(count)[None, None, :]
    end = t + a + k
    valid = end <= rows - 1
    return (r >= t) & (r <= end) & valid, (r == end) & valid


def _eval(ctx, f):
    T = ctx.T
    k = _kind(f)
    if k == "TrueFormula":
        return _const(np.full(ctx.lead + (ctx.L,), float(ctx.cfg.top_value)))
    if k == "Pred":
        x = ctx.ch[f.var]
        if f.cmp in (">", ">="):
            return _add_scalar(T, x, -float(f.threshold))
        return _add_scalar(T, _neg(T, x), float(f.threshold))
    if k == "NormPred":
        d = _norm(T, ctx.ch[f.vars[0]], ctx.ch[f.vars[1]], f.center[0], f.center[1])
        if f.cmp in (">", ">="):
            return _add_scalar(T, d, -float(f.threshold))
        return _add_scalar(T, _neg(T, d), float(f.threshold))
    if k == "Not":
        return _neg(T, _eval(ctx, f.arg))
    if k in ("And", "Or"):
        l = _eval(ctx, f.left)
        r = _eval(ctx, f.right)
        return _reduce(T, _stack(T, [l, r]), "min" if k == "And" else "max", ctx.mode, ctx.tau)
    if k in ("Eventually", "Always"):
        child = _eval(ctx, f.arg)
        return _ev_al(ctx, child, f.interval, "max" if k == "Eventually" else "min")
    if k == "Until":
        l = _eval(ctx, f.left)
        r = _eval(ctx, f.right)
        return _until(ctx, l, r, f.interval)
    raise TypeError(f"not a Formula node: {f!r}")


# ---------------------------------------------------------------------------
# public oracle entry points
# ---------------------------------------------------------------------------

def trace(f, channels, cfg, smooth_binding=None):
    """Robustness trace; channels: name -> array (..., L). Returns float64 (..., L)."""
    out, _ = _run(f, channels, cfg, smooth_binding)
    return out.val.copy()


def _run(f, channels, cfg, smooth_binding, eps_override=None):
    leaves = {k: _Node(np.asarray(v, dtype=np.float64), leaf=True) for k, v in channels.items()}
    L = next(iter(leaves.values())).val.shape[-1]
    ctx = _Ctx(leaves, L, cfg, smooth_binding)
    ctx.eps_override = eps_override
    out = _eval(ctx, f)
    return out, (ctx, leaves)


def trace_and_grad(f, channels, cfg, cotangent=None, smooth_binding=None, eps_override=None):
    """Trace plus the VJP of the full trace with ``cotangent`` (ones by default).

    Returns (trace, {name: d_channel}, (d_a, d_b, d_c) or None).
    """
    out, (ctx, leaves) = _run(f, channels, cfg, smooth_binding, eps_override)
    seed = np.ones_like(out.val) if cotangent is None else np.asarray(cotangent, dtype=np.float64)
    if out.leaf != "const":
        ctx.T.backward(out, seed)
    grads = {k: (n.grad.copy() if n.grad is not None else np.zeros_like(n.val))
             for k, n in leaves.items()}
    dabc = None
    if smooth_binding is not None:
        a, b, c = smooth_binding
        da = db = dc = 0.0
        for node, eps in ctx.wnodes:
            if node.grad is None:
                continue
            gw = node.grad
            _, dwa, dwb, dwc = smooth_weights(a, b, c, eps, ctx.L)
            da += float(np.sum(gw * dwa))
            db += float(np.sum(gw * dwb))
            dc += float(np.sum(gw * dwc))
        dabc = (da, db, dc)
    return out.val.copy(), grads, dabc


def value_and_grad(f, arrays, cfg, si=None):
    """Entry-0 robustness and its gradients (autodiff.py:64-107), 1-D signals."""
    from paper_2501_04194_b200.formula import smooth_intervals
    sis = smooth_intervals(f)
    binding = None
    if si is not None:
        binding = (si.a, si.b, si.c)
    elif sis:
        if len(set(sis)) > 1:
            raise ValueError("multiple distinct smooth intervals; pass si= to bind them")
        binding = (sis[0].a, sis[0].b, sis[0].c)
    L = len(next(iter(arrays.values())))
    cot = np.zeros(L)
    cot[0] = 1.0
    tr, grads, dabc = trace_and_grad(f, arrays, cfg, cot, smooth_binding=binding,
                                     eps_override=None if si is None else si.eps)
    return float(tr[0]), grads, dabc


# ---------------------------------------------------------------------------
# O(L)-memory restatements for long signals (same semantics, checked against the
# tape oracle above at small L by tests/test_oracle_long.py)
# ---------------------------------------------------------------------------

def until_untimed_hard(left, right, cot):
    """Hard untimed Until over child traces (rows, L), masking.py:238-293 with iv=None.

    Per output t the reference stacks, for k = 0..L-1-t, pm_k = min(l[t..t+k]) built
    incrementally (a tie keeps pm_{k-1}, i.e. the earliest arg-min) and
    term_k = min(pm_k, r[t+k]) (a tie keeps pm, the first stacked operand), then takes
    the first arg-max over k (tape.py:338-357 one-hot rule); min is -max(-x), so every
    value is a selected input, signed zeros included.  Entries with t+k > L-1 carry
    weight 0 and never win.  Returns (trace, d_left, d_right) for cotangent ``cot``;
    O(L) memory and O(L^2) time per row.
    """
    left = np.atleast_2d(np.asarray(left, dtype=np.float64))
    right = np.atleast_2d(np.asarray(right, dtype=np.float64))
    cot = np.atleast_2d(np.asarray(cot, dtype=np.float64))
    R, L = left.shape
    out = np.empty((R, L))
    dl = np.zeros((R, L))
    dr = np.zeros((R, L))
    ar = np.arange(L)
    for t in range(L):
        ls = left[:, t:]
        rs = right[:, t:]
        n = L - t
        # earliest arg-min prefix: a new minimum only on a strict decrease
        pmv = np.minimum.accumulate(ls, axis=1)
        new = np.ones((R, n), dtype=bool)
        new[:, 1:] = ls[:, 1:] < pmv[:, :-1]
        pidx = np.maximum.accumulate(np.where(new, ar[None, :n], 0), axis=1)
        pm = np.take_along_axis(ls, pidx, axis=1)
        take_pm = pm <= rs
        term = np.where(take_pm, pm, rs)
        k = np.argmax(term, axis=1)
        rows = np.arange(R)
        out[:, t] = term[rows, k]
        via_pm = take_pm[rows, k]
        src_l = t + pidx[rows, k]
        src_r = t + k
        np.add.at(dl, (rows[via_pm], src_l[via_pm]), cot[rows[via_pm], t])
        np.add.at(dr, (rows[~via_pm], src_r[~via_pm]), cot[rows[~via_pm], t])
    return out, dl, dr


def suffix_hard(x, cot, kind="max"):
    """Untimed hard F (kind='max') / G ('min') over (rows, L), tape.py:475-491: reverse
    running extremum, the gradient of out[t] routed to the FIRST extremum at or after t.
    Vectorised form of ``_suffix`` (O(L) numpy passes)."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    cot = np.atleast_2d(np.asarray(cot, dtype=np.float64))
    v = x if kind == "max" else -x
    R, L = v.shape
    rv = v[:, ::-1]
    best = np.maximum.accumulate(rv, axis=1)
    # scanning from the end, a later-in-time (earlier-in-scan) index is replaced on >=
    new = np.ones((R, L), dtype=bool)
    new[:, 1:] = rv[:, 1:] >= best[:, :-1]
    ridx = np.maximum.accumulate(np.where(new, np.arange(L)[None, :], 0), axis=1)
    sel = (L - 1 - ridx)[:, ::-1]
    val = np.take_along_axis(v, sel, axis=1)
    g = np.zeros((R, L))
    np.add.at(g, (np.repeat(np.arange(R), L), sel.ravel()), cot.ravel())
    if kind == "max":
        return val, g
    return -val, g
