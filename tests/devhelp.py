"""Helpers for the GPU parity tests: run the device path through the public API."""

import json

import numpy as np


def has_op(f, names):
    k = type(f).__name__
    if k in names:
        return True
    for attr in ("arg", "left", "right"):
        if hasattr(f, attr) and has_op(getattr(f, attr), names):
            return True
    return False


def has_smooth(f):
    from paper_2501_04194_b200 import smooth_intervals
    return bool(smooth_intervals(f))


def device_supports(f, cfg):
    """Operators implemented on the device in this build."""
    import paper_2501_04194_b200 as P
    try:
        names = sorted(P.variables(f)) or ["x"]
        P.compile_formula(f, names, cfg)
    except TypeError:
        return False
    return True


def run_device(f, arrays, cfg, cot=None, binding=None):
    """trace [B, L] + VJP with `cot` through paper_2501_04194_b200.trace (CUDA)."""
    import torch
    import paper_2501_04194_b200 as P
    dev = torch.device("cuda", 0)
    chans = {k: torch.tensor(np.asarray(v, dtype=np.float32), device=dev).reshape(
        np.asarray(v).shape[0] if np.asarray(v).ndim == 2 else 1, -1).requires_grad_(True)
        for k, v in arrays.items()}
    abc = None
    if binding is not None:
        abc = tuple(torch.tensor(float(v), dtype=torch.float64, device=dev, requires_grad=True)
                    for v in binding)
    out = P.trace(f, chans, cfg, smooth_binding=abc)
    tr = out.detach().double().cpu().numpy()
    if cot is None:
        cot = np.ones_like(tr)
    leaves = list(chans.values()) + (list(abc) if abc else [])
    if out.requires_grad:
        grads = torch.autograd.grad(out, leaves, torch.tensor(np.asarray(cot, dtype=np.float32),
                                                              device=dev), allow_unused=True)
    else:
        grads = [None] * len(leaves)
    g = {}
    for i, k in enumerate(chans):
        gi = grads[i]
        g[k] = np.zeros(tr.shape) if gi is None else gi.detach().double().cpu().numpy()
    dabc = None
    if abc:
        dabc = np.array([0.0 if x is None else float(x) for x in grads[len(chans):]])
    return tr, g, dabc


def rel_err(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if got.size == 0:
        return 0.0
    return float(np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref))))


def assert_hard_equal(got, ref32):
    """Bit-exact: the fp32 rounding of the f64 reference, including the sign of zero."""
    got = np.asarray(got, dtype=np.float32)
    ref32 = np.asarray(ref32, dtype=np.float32)
    bad = np.flatnonzero(got.view(np.uint32) != ref32.view(np.uint32))
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:5]}: got {got.ravel()[bad[:5]]} ref {ref32.ravel()[bad[:5]]}"
