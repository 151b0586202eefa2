"""BASELINE configurations at their stated sizes and the multi-tile paths, on the device,
against the oracle (VERDICT r1 "check every BASELINE config and every multi-tile path").

* C1 exactly as BASELINE configs[0] states it (Always[0,50](x > 0.5), Hard, T=1000);
* C3 at B=256, T=4000 (Hard bit-exact on sampled rows; LSE(10) on one row);
* untimed F/G past the 4096-sample tiles of csrc/fg_unt.cu (T = 4097, 8193, 100000),
  tie-heavy data so the first-arg-max rule crosses tile carries;
* hard untimed Until past its 2048-sample tile (csrc/until.cu), tie-heavy;
* C5 corners: timed F/G[0,100] at T=100k, U[0,100] and untimed U at T=30k.

Rows are independent, so full-size batches run on the device and sampled rows go to the
oracle; at lengths where the tape oracle's O(L^2) Until / suffix windows do not fit, the
O(L)-memory restatements (stl_oracle.until_untimed_hard / suffix_hard, pinned to the tape
oracle by tests/test_oracle_long.py) check them.  Tolerances as test_gpu_parity.py.
"""

import numpy as np
import pytest

import stl_oracle
from devhelp import assert_hard_equal, rel_err

import paper_2501_04194_b200 as P

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _run(f, arrays, cfg, cot=None):
    """Full-batch device trace + VJP; returns host float64 arrays."""
    import torch
    dev = torch.device("cuda", 0)
    chans = {k: torch.tensor(np.asarray(v, dtype=np.float32), device=dev).requires_grad_(True)
             for k, v in arrays.items()}
    out = P.trace(f, chans, cfg)
    c = torch.ones_like(out) if cot is None else torch.tensor(np.asarray(cot, dtype=np.float32), device=dev)
    grads = torch.autograd.grad(out, list(chans.values()), c, allow_unused=True)
    g = {k: (np.zeros(out.shape) if gi is None else gi.double().cpu().numpy())
         for k, gi in zip(chans, grads)}
    return out.detach().double().cpu().numpy(), g


def _ties(rng, shape, levels=2):
    v = rng.integers(-levels, levels + 1, shape).astype(np.float32)
    v[rng.random(shape) < 0.05] = -0.0
    return v


def test_c1_exact_baseline_config(cuda):
    """BASELINE configs[0]: Always[0,50](x > 0.5), hard, 1-D, batch 1, T=1000, last pad."""
    x = np.asarray(np.random.default_rng(0).normal(0, 1, (1, 1000)), dtype=np.float32)
    f = P.Always(P.Pred("x", ">", 0.5), P.StepInterval(0, 50))
    cfg = P.SemanticsConfig(mode=P.Hard())
    tr, g = _run(f, {"x": x}, cfg)
    ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, {"x": x.astype(np.float64)}, cfg)
    assert_hard_equal(tr, ref_tr.astype(np.float32))
    np.testing.assert_array_equal(g["x"], ref_g["x"])
    # robustness mode (value_and_grad, autodiff.py:64) on the same case
    vg = P.value_and_grad(f, P.NamedSignals.from_arrays({"x": x[0]}), cfg)
    rv, rg, _ = stl_oracle.value_and_grad(f, {"x": x[0].astype(np.float64)}, cfg)
    assert np.float32(vg.value) == np.float32(rv)
    np.testing.assert_array_equal(vg.d_signal["x"], rg["x"][0] if rg["x"].ndim == 2 else rg["x"])


def _c3_data():
    rng = np.random.default_rng(2)
    return {k: np.asarray(rng.normal(0, 1, (256, 4000)), dtype=np.float32) for k in ("x", "y", "z")}


C3 = P.And(P.Always(P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(0, 200))),
           P.Until(P.Pred("y", "<", 1.0), P.Pred("z", ">", 0.0)))


def test_c3_full_size_hard_rows_bit_exact(cuda):
    data = _c3_data()
    cfg = P.SemanticsConfig(mode=P.Hard())
    tr, g = _run(C3, data, cfg)
    for r in (0, 131, 255):
        rows = {k: v[r:r + 1].astype(np.float64) for k, v in data.items()}
        ref_tr, ref_g, _ = stl_oracle.trace_and_grad(C3, rows, cfg)
        assert_hard_equal(tr[r:r + 1], ref_tr.astype(np.float32))
        for k in data:
            np.testing.assert_array_equal(g[k][r:r + 1], ref_g[k])
    # size-independent: every output routes its unit cotangent to exactly one sample, and
    # each channel's predicate has one sign (x > 0, z > 0: +1; y < 1: -1)
    total = sum(np.abs(g[k]).sum(axis=1) for k in data)
    assert np.all(total == 4000)
    assert np.all(g["x"] >= 0) and np.all(g["z"] >= 0) and np.all(g["y"] <= 0)


def test_c3_full_size_lse_row(cuda):
    data = _c3_data()
    cfg = P.SemanticsConfig(mode=P.LogSumExp(10.0))
    tr, g = _run(C3, data, cfg)
    r = 77
    rows = {k: v[r:r + 1].astype(np.float64) for k, v in data.items()}
    ref_tr, ref_g, _ = stl_oracle.trace_and_grad(C3, rows, cfg)
    assert rel_err(tr[r:r + 1], ref_tr) <= TOL
    for k in data:
        assert rel_err(g[k][r:r + 1], ref_g[k]) <= TOL, k


@pytest.mark.parametrize("T", [4097, 8193, 100_000])
@pytest.mark.parametrize("op", ["F", "G"])
@pytest.mark.parametrize("ties", [False, True], ids=["noise", "ties"])
def test_untimed_hard_fg_across_tiles(cuda, T, op, ties):
    rng = np.random.default_rng(T + (op == "G") + 2 * ties)
    x = _ties(rng, (3, T)) if ties else np.asarray(rng.normal(0, 1, (3, T)), dtype=np.float32)
    cot = np.asarray(rng.normal(0, 1, (3, T)), dtype=np.float32)
    node = P.Eventually if op == "F" else P.Always
    f = node(P.Pred("x", ">", 0.0))
    cfg = P.SemanticsConfig()
    tr, g = _run(f, {"x": x}, cfg)
    ref, rg = stl_oracle.suffix_hard(x.astype(np.float64) - 0.0, np.ones((3, T)), "max" if op == "F" else "min")
    assert_hard_equal(tr, ref.astype(np.float32))
    np.testing.assert_array_equal(g["x"], rg)
    tr2, g2 = _run(f, {"x": x}, cfg, cot)
    _, rg2 = stl_oracle.suffix_hard(x.astype(np.float64), cot.astype(np.float64), "max" if op == "F" else "min")
    assert rel_err(g2["x"], rg2) <= 1e-6


@pytest.mark.parametrize("T", [4097, 8193, 100_000])
@pytest.mark.parametrize("op", ["F", "G"])
def test_untimed_lse_fg_across_tiles(cuda, T, op):
    rng = np.random.default_rng(7 * T + (op == "G"))
    # the suffix LSE changes scale along the signal: N(0,1) (C5's inputs) plus a slow drift
    # of amplitude 6 (tau |u| <~ 100: the fp32 regime where DESIGN §6's 1e-5 bound holds)
    drift = 6.0 * np.sin(np.arange(T) * (2 * np.pi / min(T, 20000)))
    x = np.asarray(rng.normal(0, 1, (2, T)) + drift, dtype=np.float32)
    cot = np.asarray(rng.uniform(0.5, 1.5, (2, T)), dtype=np.float32)
    node = P.Eventually if op == "F" else P.Always
    f = node(P.Pred("x", ">", 0.25))
    cfg = P.SemanticsConfig(mode=P.LogSumExp(10.0))
    tr, g = _run(f, {"x": x}, cfg, cot)
    ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, {"x": x.astype(np.float64)}, cfg, cot.astype(np.float64))
    assert rel_err(tr, ref_tr) <= TOL
    assert rel_err(g["x"], ref_g["x"]) <= TOL


def test_untimed_softmax_fg_across_tiles(cuda):
    rng = np.random.default_rng(41)
    T = 4097
    x = np.asarray(rng.normal(0, 1, (1, T)), dtype=np.float32)
    f = P.Eventually(P.Pred("x", ">", 0.0))
    cfg = P.SemanticsConfig(mode=P.SoftMax(2.0))
    tr, g = _run(f, {"x": x}, cfg)
    ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, {"x": x.astype(np.float64)}, cfg)
    assert rel_err(tr, ref_tr) <= TOL
    assert rel_err(g["x"], ref_g["x"]) <= TOL


@pytest.mark.parametrize("T", [2049, 4000, 10_000])
def test_hard_untimed_until_across_tiles(cuda, T):
    rng = np.random.default_rng(T)
    x, y = _ties(rng, (2, T), 3), _ties(rng, (2, T), 3)
    f = P.Until(P.Pred("x", ">", 0.0), P.Pred("y", "<", 0.0))
    cfg = P.SemanticsConfig()
    tr, g = _run(f, {"x": x, "y": y}, cfg)
    ref, dl, dr = stl_oracle.until_untimed_hard(x.astype(np.float64) - 0.0, -y.astype(np.float64) + 0.0,
                                                np.ones((2, T)))
    assert_hard_equal(tr, ref.astype(np.float32))
    np.testing.assert_array_equal(g["x"], dl)
    np.testing.assert_array_equal(g["y"], -dr)
    cot = np.asarray(rng.normal(0, 1, (2, T)), dtype=np.float32)
    _, g2 = _run(f, {"x": x, "y": y}, cfg, cot)
    _, dl2, dr2 = stl_oracle.until_untimed_hard(x.astype(np.float64), -y.astype(np.float64),
                                                cot.astype(np.float64))
    assert rel_err(g2["x"], dl2) <= 1e-6
    assert rel_err(g2["y"], -dr2) <= 1e-6


@pytest.mark.parametrize("mode", [P.Hard(), P.LogSumExp(10.0)], ids=["hard", "lse"])
@pytest.mark.parametrize("op", ["F", "G"])
def test_c5_timed_window_T100k(cuda, mode, op):
    rng = np.random.default_rng(100 + (op == "G"))
    B, T = 64, 100_000
    x = np.asarray(rng.normal(0, 1, (B, T)), dtype=np.float32)
    node = P.Eventually if op == "F" else P.Always
    f = node(P.Pred("x", ">", 0.0), P.StepInterval(0, 100))
    cfg = P.SemanticsConfig(mode=mode)
    tr, g = _run(f, {"x": x}, cfg)
    for r in (0, 63):
        ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, {"x": x[r:r + 1].astype(np.float64)}, cfg)
        if type(mode).__name__ == "Hard":
            assert_hard_equal(tr[r:r + 1], ref_tr.astype(np.float32))
            np.testing.assert_array_equal(g["x"][r:r + 1], ref_g["x"])
        else:
            assert rel_err(tr[r:r + 1], ref_tr) <= TOL
            assert rel_err(g["x"][r:r + 1], ref_g["x"]) <= TOL


@pytest.mark.parametrize("mode", [P.Hard(), P.LogSumExp(10.0)], ids=["hard", "lse"])
def test_c5_timed_until_T30k(cuda, mode):
    rng = np.random.default_rng(30)
    B, T = 64, 30_000
    x = np.asarray(rng.normal(0, 1, (B, T)), dtype=np.float32)
    y = np.asarray(rng.normal(0, 1, (B, T)), dtype=np.float32)
    f = P.Until(P.Pred("x", ">", 0.0), P.Pred("y", ">", 0.0), P.StepInterval(0, 100))
    cfg = P.SemanticsConfig(mode=mode)
    tr, g = _run(f, {"x": x, "y": y}, cfg)
    r = 40
    ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, {"x": x[r:r + 1].astype(np.float64),
                                                     "y": y[r:r + 1].astype(np.float64)}, cfg)
    if type(mode).__name__ == "Hard":
        assert_hard_equal(tr[r:r + 1], ref_tr.astype(np.float32))
        for k in ("x", "y"):
            np.testing.assert_array_equal(g[k][r:r + 1], ref_g[k])
    else:
        assert rel_err(tr[r:r + 1], ref_tr) <= TOL
        for k in ("x", "y"):
            assert rel_err(g[k][r:r + 1], ref_g[k]) <= TOL


def test_c5_untimed_until_T30k_hard(cuda):
    rng = np.random.default_rng(31)
    B, T = 64, 30_000
    x = np.asarray(rng.normal(0, 1, (B, T)), dtype=np.float32)
    y = np.asarray(rng.normal(0, 1, (B, T)), dtype=np.float32)
    f = P.Until(P.Pred("x", ">", 0.0), P.Pred("y", ">", 0.0))
    tr, g = _run(f, {"x": x, "y": y}, P.SemanticsConfig())
    r = 17
    ref, dl, dr = stl_oracle.until_untimed_hard(x[r:r + 1].astype(np.float64), y[r:r + 1].astype(np.float64),
                                                np.ones((1, T)))
    assert_hard_equal(tr[r:r + 1], ref.astype(np.float32))
    np.testing.assert_array_equal(g["x"][r:r + 1], dl)
    np.testing.assert_array_equal(g["y"][r:r + 1], dr)


@pytest.mark.parametrize("pad", ["last", "const"])
@pytest.mark.parametrize("a,K,L", [(0, 1, 50), (0, 2, 300), (1, 5, 300), (3, 64, 1500), (0, 101, 1500),
                                   (17, 101, 2500), (2, 300, 5000), (40, 7, 900), (0, 1100, 2600),
                                   (0, 65, 1400), (65, 65, 2100), (70, 129, 3000), (64, 200, 1900)])
def test_hard_timed_until_sweep(cuda, a, K, L, pad):
    """O(T) hard timed Until (csrc/until_ht.cu) vs the oracle: tie-heavy inputs (integers
    and signed zeros), left- and right-sourced outputs, overrun tails, both paddings,
    values bit-exact and gradients exact (ones) / 1e-6 (random cotangent)."""
    rng = np.random.default_rng(a * 1000 + K + L + (pad == "last"))
    x, y = _ties(rng, (2, L), 3), _ties(rng, (2, L), 3)
    f = P.Until(P.Pred("x", ">", 0.0), P.Pred("y", "<", 0.5), P.StepInterval(a, a + K - 1))
    padding = P.PaddingPolicy.last_value() if pad == "last" else P.PaddingPolicy.constant(-0.75)
    cfg = P.SemanticsConfig(padding=padding)
    arrays = {"x": x.astype(np.float64), "y": y.astype(np.float64)}
    tr, g = _run(f, {"x": x, "y": y}, cfg)
    ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, arrays, cfg)
    assert_hard_equal(tr, ref_tr.astype(np.float32))
    for k in ("x", "y"):
        np.testing.assert_array_equal(g[k], ref_g[k])
    cot = np.asarray(rng.normal(0, 1, (2, L)), dtype=np.float32)
    _, g2 = _run(f, {"x": x, "y": y}, cfg, cot)
    _, ref_g2, _ = stl_oracle.trace_and_grad(f, arrays, cfg, cot.astype(np.float64))
    for k in ("x", "y"):
        assert rel_err(g2[k], ref_g2[k]) <= 1e-6, k


@pytest.mark.parametrize("case", ["F_hard", "G_lse", "U_hard"])
def test_untimed_sequential_shape_large_batch(cuda, case):
    """Untimed scans at >= 296 rows take the one-CTA-per-row shape (fg_unt.cu / until.cu,
    LB = false) with its register carry across 4096- / 2048-sample tiles; rows checked
    against the oracle (the look-back shape is covered by the small-batch tests above)."""
    rng = np.random.default_rng(300 + len(case))
    B, T = 300, 9000
    x = np.asarray(rng.normal(0, 1, (B, T)), dtype=np.float32)
    y = np.asarray(rng.normal(0, 1, (B, T)), dtype=np.float32)
    cot = np.asarray(rng.uniform(0.5, 1.5, (B, T)), dtype=np.float32)
    if case == "F_hard":
        f, cfg, data = P.Eventually(P.Pred("x", ">", 0.0)), P.SemanticsConfig(), {"x": np.round(2 * x)}
    elif case == "G_lse":
        f, cfg, data = P.Always(P.Pred("x", ">", 0.0)), P.SemanticsConfig(mode=P.LogSumExp(10.0)), {"x": x}
    else:
        f = P.Until(P.Pred("x", ">", 0.0), P.Pred("y", ">", 0.0))
        cfg, data = P.SemanticsConfig(), {"x": np.round(2 * x), "y": np.round(2 * y)}
    tr, g = _run(f, data, cfg, cot)
    for r in (0, 151, 299):
        c64 = cot[r:r + 1].astype(np.float64)
        if case == "G_lse":
            ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, {"x": x[r:r + 1].astype(np.float64)}, cfg, c64)
            assert rel_err(tr[r:r + 1], ref_tr) <= TOL
            assert rel_err(g["x"][r:r + 1], ref_g["x"]) <= TOL
        elif case == "F_hard":
            xr = data["x"][r:r + 1].astype(np.float64)
            ref, _ = stl_oracle.suffix_hard(xr, np.ones((1, T)), "max")
            _, rg = stl_oracle.suffix_hard(xr, c64, "max")
            assert_hard_equal(tr[r:r + 1], ref.astype(np.float32))
            assert rel_err(g["x"][r:r + 1], rg) <= 1e-6
        else:
            xr, yr = data["x"][r:r + 1].astype(np.float64), data["y"][r:r + 1].astype(np.float64)
            ref, _, _ = stl_oracle.until_untimed_hard(xr, yr, np.ones((1, T)))
            _, dl, dr = stl_oracle.until_untimed_hard(xr, yr, c64)
            assert_hard_equal(tr[r:r + 1], ref.astype(np.float32))
            assert rel_err(g["x"][r:r + 1], dl) <= 1e-6
            assert rel_err(g["y"][r:r + 1], dr) <= 1e-6


@pytest.mark.parametrize("pad", ["last", "const"])
@pytest.mark.parametrize("a,K,L", [(0, 16, 300), (0, 101, 1500), (3, 20, 700), (17, 101, 2500),
                                   (2, 300, 1100), (70, 129, 3000), (0, 600, 700), (5, 40, 30)])
def test_lse_timed_until_reciprocal_sweep(cuda, a, K, L, pad):
    """Timed LSE Until forward in reciprocal form (until.cu k_until_rcp_lse_fwd<true>,
    K >= 16): one rcp per (t, s) pair over the window [t + a, t + b], the pm sum from t;
    overrun outputs, both paddings, a-prefixes, windows longer than the 128-output tile
    and than the row; values and gradients vs the oracle at 1e-5 under a random cotangent."""
    rng = np.random.default_rng(a * 7919 + K * 31 + L + (pad == "last"))
    x = np.asarray(rng.normal(0, 1, (2, L)), dtype=np.float32)
    y = np.asarray(rng.normal(0, 1, (2, L)), dtype=np.float32)
    f = P.Until(P.Pred("x", ">", 0.0), P.Pred("y", "<", 0.5), P.StepInterval(a, a + K - 1))
    padding = P.PaddingPolicy.last_value() if pad == "last" else P.PaddingPolicy.constant(-0.75)
    cfg = P.SemanticsConfig(mode=P.LogSumExp(3.0), padding=padding)
    cot = np.asarray(rng.normal(0, 1, (2, L)), dtype=np.float32)
    tr, g = _run(f, {"x": x, "y": y}, cfg, cot)
    arrays = {"x": x.astype(np.float64), "y": y.astype(np.float64)}
    ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, arrays, cfg, cot.astype(np.float64))
    assert rel_err(tr, ref_tr) <= TOL
    for k in ("x", "y"):
        assert rel_err(g[k], ref_g[k]) <= TOL, k


@pytest.mark.parametrize("mode", [P.Hard(), P.LogSumExp(5.0)], ids=["hard", "lse"])
@pytest.mark.parametrize("child", ["norm_pair", "compound"])
def test_untimed_lookback_child_kinds(cuda, mode, child):
    """The look-back shape (small batch, long rows) with the other child evaluators: a
    NormPred over an interleaved [B, T, 2] tensor (EK_PAIR) and a compound child (an And of
    predicates, materialised by its own pointwise entry); sampled rows vs the oracle."""
    import torch
    rng = np.random.default_rng(90 + (child == "compound"))
    B, T = 6, 9000
    dev = torch.device("cuda", 0)
    if child == "norm_pair":
        pxy = np.asarray(np.cumsum(rng.normal(0, 0.05, (B, T, 2)), axis=1), dtype=np.float32)
        t = torch.tensor(pxy, device=dev).requires_grad_(True)
        chans = {"px": t[..., 0], "py": t[..., 1]}
        f = P.Eventually(P.NormPred(("px", "py"), "<", 0.5))
        arrays = {"px": pxy[..., 0], "py": pxy[..., 1]}
        leaves = [t]
    else:
        x = np.asarray(rng.normal(0, 1, (B, T)), dtype=np.float32)
        y = np.asarray(rng.normal(0, 1, (B, T)), dtype=np.float32)
        tx = torch.tensor(x, device=dev).requires_grad_(True)
        ty = torch.tensor(y, device=dev).requires_grad_(True)
        chans = {"x": tx, "y": ty}
        f = P.Always(P.And(P.Pred("x", ">", -0.5), P.Pred("y", "<", 0.8)))
        arrays = {"x": x, "y": y}
        leaves = [tx, ty]
    cfg = P.SemanticsConfig(mode=mode)
    out = P.trace(f, chans, cfg)
    cot = torch.tensor(np.asarray(rng.uniform(0.5, 1.5, (B, T)), dtype=np.float32), device=dev)
    grads = torch.autograd.grad(out, leaves, cot)
    tr = out.detach().double().cpu().numpy()
    if child == "norm_pair":
        g = grads[0].double().cpu().numpy()
        gk = {"px": g[..., 0], "py": g[..., 1]}
    else:
        gk = {"x": grads[0].double().cpu().numpy(), "y": grads[1].double().cpu().numpy()}
    for r in (0, 5):
        rows = {k: v[r:r + 1].astype(np.float64) for k, v in arrays.items()}
        ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, rows, cfg, cot[r:r + 1].double().cpu().numpy())
        assert rel_err(tr[r:r + 1], ref_tr) <= TOL
        for k in arrays:
            assert rel_err(gk[k][r:r + 1], ref_g[k]) <= TOL, k
