"""Bitwise reproducibility of the backward under a general (random) cotangent
(SURVEY §7.6): two runs on the same inputs must give identical
gradients and d(a, b, c) — no float atomics whose order varies between runs on any
path a general cotangent flows through.  The multi-GPU all-reduce sums these
per-rank partials, so they must be reproducible first."""

import numpy as np
import pytest

import paper_2501_04194_b200 as P

pytestmark = pytest.mark.gpu

SI = P.SmoothInterval(0.3, 0.65, 9.0)
CASES = [
    ("F_untimed_hard", P.Eventually(P.Pred("x", ">", 0.0)), P.Hard()),
    ("G_untimed_lse", P.Always(P.Pred("x", ">", 0.0)), P.LogSumExp(5.0)),
    ("F_timed_hard", P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(3, 60)), P.Hard()),
    ("G_timed_lse", P.Always(P.Pred("x", ">", 0.0), P.StepInterval(0, 40)), P.LogSumExp(5.0)),
    ("F_timed_soft", P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(2, 30)), P.SoftMax(2.0)),
    ("U_untimed_hard", P.Until(P.Pred("x", ">", 0.0), P.Pred("y", ">", 0.0)), P.Hard()),
    ("U_timed_hard", P.Until(P.Pred("x", ">", 0.0), P.Pred("y", ">", 0.0), P.StepInterval(0, 20)), P.Hard()),
    ("U_timed_lse", P.Until(P.Pred("x", ">", 0.0), P.Pred("y", ">", 0.0), P.StepInterval(1, 20)), P.LogSumExp(3.0)),
    ("U_untimed_lse", P.Until(P.Pred("x", ">", 0.0), P.Pred("y", ">", 0.0)), P.LogSumExp(3.0)),
    ("G_smooth_lse", P.Always(P.Pred("x", ">", 0.0), SI), P.LogSumExp(5.0)),
    ("F_smooth_soft", P.Eventually(P.Pred("x", ">", 0.0), SI), P.SoftMax(2.0)),
    ("nested_hard", P.And(P.Always(P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(0, 30))),
                          P.Until(P.Pred("y", "<", 1.0), P.Pred("x", ">", 0.0))), P.Hard()),
    # independent operands (no shared channel): the executor runs them on two streams
    ("lanes_hard", P.And(P.Always(P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(0, 30))),
                         P.Until(P.Pred("y", "<", 1.0), P.Pred("z", ">", 0.0))), P.Hard()),
    ("lanes_lse", P.Or(P.Or(P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(2, 50)),
                            P.Always(P.Pred("y", "<", 1.0))),
                       P.Eventually(P.Pred("z", ">", 0.5))), P.LogSumExp(4.0)),
]


@pytest.mark.parametrize("name,f,mode", CASES, ids=[c[0] for c in CASES])
def test_backward_bitwise_reproducible(cuda, name, f, mode):
    import torch
    g = torch.Generator(device="cuda").manual_seed(5)
    B, T = 64, 1500
    x = torch.randn(B, T, device="cuda", generator=g)
    y = torch.randn(B, T, device="cuda", generator=g)
    z = torch.randn(B, T, device="cuda", generator=g)
    if "hard" in name:  # ties, so the first-arg-max runs are long and cross tiles
        x, y, z = torch.round(x * 2), torch.round(y * 2), torch.round(z * 2)
    cot = torch.randn(B, T, device="cuda", generator=g)
    names = sorted(P.variables(f))
    runs = []
    for _ in range(2):
        chans = {"x": x.clone().requires_grad_(True), "y": y.clone().requires_grad_(True),
                 "z": z.clone().requires_grad_(True)}
        chans = {k: chans[k] for k in names}
        smooth = "smooth" in name
        abc = tuple(torch.tensor(v, dtype=torch.float64, device="cuda", requires_grad=True)
                    for v in (SI.a, SI.b, SI.c)) if smooth else None
        out = P.trace(f, chans, P.SemanticsConfig(mode=mode), smooth_binding=abc)
        leaves = list(chans.values()) + (list(abc) if abc else [])
        grads = torch.autograd.grad(out, leaves, cot)
        runs.append([np.atleast_1d(t.detach().cpu().numpy()) for t in (out, *grads)])
    for a, b in zip(*runs):
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), name


@pytest.mark.parametrize("name,f,mode", [c for c in CASES if "untimed" in c[0]], ids=[c[0] for c in CASES if "untimed" in c[0]])
def test_lookback_shape_bitwise_reproducible(cuda, name, f, mode):
    """Small batch, long rows: the untimed scans run one CTA per 1024-sample tile with
    look-back carries (lookback.cuh) — the fixed fold order keeps the bits independent of
    which tiles finish first."""
    import torch
    if "lse" in name and "U_" in name:
        pytest.skip("untimed LSE Until is O(T^2): covered at T=1500 above")
    g = torch.Generator(device="cuda").manual_seed(9)
    B, T = 6, 20_000
    x = torch.round(torch.randn(B, T, device="cuda", generator=g) * 2)
    y = torch.round(torch.randn(B, T, device="cuda", generator=g) * 2)
    cot = torch.randn(B, T, device="cuda", generator=g)
    names = sorted(P.variables(f))
    runs = []
    for _ in range(3):
        chans = {k: {"x": x, "y": y}[k].clone().requires_grad_(True) for k in names}
        out = P.trace(f, chans, P.SemanticsConfig(mode=mode))
        grads = torch.autograd.grad(out, list(chans.values()), cot)
        runs.append([t.detach().cpu().numpy() for t in (out, *grads)])
    for other in runs[1:]:
        for a, b in zip(runs[0], other):
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), name


MORE = [
    ("F_timed_hard_K9", P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(2, 10)), P.SemanticsConfig()),
    ("G_timed_hard_K3", P.Always(P.Pred("x", ">", 0.0), P.StepInterval(0, 2)), P.SemanticsConfig()),
    ("F_smooth_lse_last", P.Eventually(P.Pred("x", ">", 0.0), SI),
     P.SemanticsConfig(mode=P.LogSumExp(5.0), padding=P.PaddingPolicy.last_value())),
    ("F_timed_hard_fill", P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(1, 30)),
     P.SemanticsConfig(masked_fill=True, sentinel=4.0)),
    ("G_untimed_hard_fill", P.Always(P.Pred("x", ">", 0.0)), P.SemanticsConfig(masked_fill=True, sentinel=4.0)),
    ("F_timed_lse_fill", P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(1, 30)),
     P.SemanticsConfig(mode=P.LogSumExp(3.0), masked_fill=True, sentinel=4.0)),
    ("F_timed_hard_fill_K2", P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(0, 1)),
     P.SemanticsConfig(masked_fill=True, sentinel=4.0, padding=P.PaddingPolicy.last_value())),
    ("G_timed_lse_fill_K3", P.Always(P.Pred("x", ">", 0.0), P.StepInterval(1, 3)),
     P.SemanticsConfig(mode=P.LogSumExp(3.0), masked_fill=True, sentinel=4.0)),
]


@pytest.mark.parametrize("name,f,cfg", MORE, ids=[c[0] for c in MORE])
def test_more_paths_bitwise_reproducible(cuda, name, f, cfg):
    """Short windows (register-blocked K <= 16 kernels), 'last' padding of a smooth
    interval, and masked_fill: same bits on every run under a random cotangent."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(11)
    B, T = 64, 1500
    x = torch.round(torch.randn(B, T, device="cuda", generator=g) * 2)
    cot = torch.randn(B, T, device="cuda", generator=g)
    runs = []
    for _ in range(3):
        xs = x.clone().requires_grad_(True)
        smooth = "smooth" in name
        abc = tuple(torch.tensor(v, dtype=torch.float64, device="cuda", requires_grad=True)
                    for v in (SI.a, SI.b, SI.c)) if smooth else None
        out = P.trace(f, {"x": xs}, cfg, smooth_binding=abc)
        leaves = [xs] + (list(abc) if abc else [])
        grads = torch.autograd.grad(out, leaves, cot)
        runs.append([np.atleast_1d(t.detach().cpu().numpy()) for t in (out, *grads)])
    for other in runs[1:]:
        for a, b in zip(runs[0], other):
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), name
