"""masked_fill (compat mode) Until on the device vs the oracle (SURVEY §8(a) a8 + a9).

In masked_fill mode the reference builds every pm_k and right operand as a reduction
over a FULL sentinel-filled column (`_fill_reduce_columns`, masking.py:195-202, 261-270),
the untimed outer max sees -sentinel for the slices past the end (masking.py:271-273)
and there is no overrun replacement.  A small sentinel makes the filled entries
numerically active in the smooth modes (the reference's documented hazard,
core.py:260-265), so the sweep checks the sentinel algebra, not just its underflow.
"""

import zlib

import numpy as np
import pytest

from devhelp import assert_hard_equal, rel_err, run_device

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2501_04194_b200 as P
    P._lib.load()
    return P


def _oracle():
    import os
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.join(here, "..", "oracle"))
    import stl_oracle
    return stl_oracle


@pytest.mark.parametrize("mode", ["hard", "lse", "soft"])
@pytest.mark.parametrize("iv", [None, (0, 3), (2, 9)], ids=["untimed", "a0b3", "a2b9"])
@pytest.mark.parametrize("pad", ["last", "const"])
@pytest.mark.parametrize("sent", [1e5, 4.0])
@pytest.mark.parametrize("L", [30, 150])
def test_masked_fill_until_vs_oracle(cuda, mode, iv, pad, sent, L):
    P = cuda
    orc = _oracle()
    # str hash() is salted per process (PYTHONHASHSEED): derive a stable seed instead
    rng = np.random.default_rng(zlib.crc32(repr((mode, iv, pad, sent, L)).encode()))
    x = np.asarray(rng.normal(0, 1.5, (2, L)), dtype=np.float32).astype(np.float64)
    y = np.asarray(rng.normal(0.2, 1.5, (2, L)), dtype=np.float32).astype(np.float64)
    if mode == "hard":  # ties for the first-index rules
        x, y = np.round(x), np.round(y)
    m = {"hard": P.Hard(), "lse": P.LogSumExp(2.0), "soft": P.SoftMax(2.0)}[mode]
    padding = P.PaddingPolicy.last_value() if pad == "last" else P.PaddingPolicy.constant(-0.75)
    cfg = P.SemanticsConfig(mode=m, padding=padding, masked_fill=True, sentinel=sent)
    interval = None if iv is None else P.StepInterval(*iv)
    f = P.Until(P.Pred("x", ">", 0.25), P.Pred("y", "<", 0.5), interval)
    cot = rng.normal(0, 1, (2, L))
    tr, g, _ = run_device(f, {"x": x, "y": y}, cfg, cot=cot)
    ref_tr, ref_g, _ = orc.trace_and_grad(f, {"x": x, "y": y}, cfg, cot)
    if mode == "hard":
        assert_hard_equal(tr, np.asarray(ref_tr, dtype=np.float32))
        tol = 1e-5
    else:
        tol = 1e-5
        assert rel_err(tr, ref_tr) <= tol
    for k in ("x", "y"):
        assert rel_err(g[k], ref_g[k]) <= tol, k


def test_untimed_lse_until_long_signal(cuda):
    """Untimed LSE Until at T=6000: the backward's checkpoints live in the persistent
    kernel's global slab (the shared-memory design stopped near T=5000)."""
    P = cuda
    orc = _oracle()
    T = 6000
    rng = np.random.default_rng(6000)
    x = np.asarray(rng.normal(0, 1, (1, T)), dtype=np.float32).astype(np.float64)
    y = np.asarray(rng.normal(0, 1, (1, T)), dtype=np.float32).astype(np.float64)
    f = P.Until(P.Pred("x", ">", 0.0), P.Pred("y", ">", 0.0))
    cfg = P.SemanticsConfig(mode=P.LogSumExp(10.0))
    cot = rng.normal(0, 1, (1, T))
    tr, g, _ = run_device(f, {"x": x, "y": y}, cfg, cot=cot)
    ref_tr, ref_g, _ = orc.trace_and_grad(f, {"x": x, "y": y}, cfg, cot)
    assert rel_err(tr, ref_tr) <= 1e-5
    for k in ("x", "y"):
        assert rel_err(g[k], ref_g[k]) <= 1e-5, k


@pytest.mark.parametrize("T", [1, 2, 31, 32, 33, 127, 128, 129, 161, 300, 513])
@pytest.mark.parametrize("tau", [1.0, 10.0])
def test_untimed_lse_until_ragged(cuda, T, tau):
    """Untimed LSE Until (reciprocal-form kernels, csrc/until.cu) at lengths around the
    32-column chunks and 128-output tiles, AR(1) and iid rows, signed cotangents."""
    P = cuda
    orc = _oracle()
    rng = np.random.default_rng(T * 7 + int(tau))
    B = 3
    x = rng.normal(0, 1, (B, T))
    x[1] = np.cumsum(0.3 * rng.normal(0, 1, T))
    y = rng.normal(0, 1, (B, T))
    x = np.asarray(x, dtype=np.float32).astype(np.float64)
    y = np.asarray(y, dtype=np.float32).astype(np.float64)
    f = P.Until(P.Pred("x", ">", 0.2), P.Pred("y", "<", 0.5))
    cfg = P.SemanticsConfig(mode=P.LogSumExp(tau))
    cot = rng.normal(0, 1, (B, T))
    tr, g, _ = run_device(f, {"x": x, "y": y}, cfg, cot=cot)
    ref_tr, ref_g, _ = orc.trace_and_grad(f, {"x": x, "y": y}, cfg, cot)
    assert rel_err(tr, ref_tr) <= 1e-5
    for k in ("x", "y"):
        assert rel_err(g[k], ref_g[k]) <= 1e-5, k


def test_untimed_lse_until_wide_range_rows(cuda):
    """Rows whose values span more than the reciprocal form's 400 log2 units take the
    per-pair path inside the same launch; mixed with narrow rows and with tiles whose
    cotangent is zero (skipped)."""
    P = cuda
    orc = _oracle()
    T = 700
    rng = np.random.default_rng(77)
    x = rng.normal(0, 1, (4, T))
    y = rng.normal(0, 1, (4, T))
    x[1] = np.cumsum(0.2 * x[1])
    y[2] = np.linspace(-30, 30, T)  # tau2 * range ~ 870 log2 units > 400: per-pair path
    x = np.asarray(x, dtype=np.float32).astype(np.float64)
    y = np.asarray(y, dtype=np.float32).astype(np.float64)
    f = P.Until(P.Pred("x", ">", 0.0), P.Pred("y", ">", 0.0))
    cfg = P.SemanticsConfig(mode=P.LogSumExp(10.0))
    cot = rng.normal(0, 1, (4, T))
    cot[3, 128:384] = 0.0
    cot[0, :] = 0.0
    cot[0, 5] = 1.0
    tr, g, _ = run_device(f, {"x": x, "y": y}, cfg, cot=cot)
    ref_tr, ref_g, _ = orc.trace_and_grad(f, {"x": x, "y": y}, cfg, cot)
    assert rel_err(tr, ref_tr) <= 1e-5
    for k in ("x", "y"):
        assert rel_err(g[k], ref_g[k]) <= 1e-5, k


@pytest.mark.parametrize("mode", ["hard", "lse", "soft"])
@pytest.mark.parametrize("iv", [(0, 0), (0, 1), (1, 3), (4, 5)], ids=["a0b0", "a0b1", "a1b3", "a4b5"])
@pytest.mark.parametrize("pad", ["last", "const"])
@pytest.mark.parametrize("fill", [False, True], ids=["plain", "fill"])
def test_short_window_gather_backward_vs_oracle(cuda, mode, iv, pad, fill):
    """Windows of K < 4 samples that miss the register-blocked kernels (masked_fill) run
    the gather-form backward (fg.cu k_fg_timed_bwd_gather): tie-heavy values, a random
    cotangent, both paddings, L-1 collecting the padded samples."""
    P = cuda
    orc = _oracle()
    rng = np.random.default_rng(zlib.crc32(repr((mode, iv, pad, fill)).encode()))
    L = 77
    x = np.round(rng.normal(0, 1.5, (3, L)) * 2) / 2
    m = {"hard": P.Hard(), "lse": P.LogSumExp(2.0), "soft": P.SoftMax(2.0)}[mode]
    padding = P.PaddingPolicy.last_value() if pad == "last" else P.PaddingPolicy.constant(-0.75)
    cfg = P.SemanticsConfig(mode=m, padding=padding, masked_fill=fill, sentinel=4.0)
    f = P.Eventually(P.Pred("x", ">", 0.25), P.StepInterval(*iv))
    cot = rng.normal(0, 1, (3, L))
    tr, g, _ = run_device(f, {"x": x}, cfg, cot=cot)
    ref_tr, ref_g, _ = orc.trace_and_grad(f, {"x": x}, cfg, cot)
    if mode == "hard":
        assert_hard_equal(tr, np.asarray(ref_tr, dtype=np.float32))
    else:
        assert rel_err(tr, ref_tr) <= 1e-5
    assert rel_err(g["x"], ref_g["x"]) <= 1e-5
