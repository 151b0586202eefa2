"""Interval mining on the device vs the reference.

Golden vectors come from the reference's own `apps` module
(tests/golden/make_mining_golden.py): `mining_objective` in Hard / LSE / softmax,
`grid_eval` over a 13 x 13 grid, and a 300-step `mine_interval` run.  The device
computes in fp32 over fp32-rounded data (the reference in f64), so values agree to
the smooth tolerance; the descent trajectory to 1e-4.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "mining.npz"))


@pytest.fixture(scope="module")
def P():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2501_04194_b200 as P
    P._lib.load()
    return P


def _rel(got, ref):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    return float(np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref))))


def test_mining_objective_matches_reference(P):
    data = GOLD["data"]
    modes = [P.Hard(), P.LogSumExp(5.0), P.SoftMax(4.0)]
    for (a, b, gamma, sharp), row in zip(GOLD["obj_points"], GOLD["obj_values"]):
        for m, ref in zip(modes, row):
            got = P.mining_objective(a, b, data, gamma, sharp, P.SemanticsConfig(mode=m))
            assert _rel(got, ref) <= 1e-5, (a, b, m, got, ref)


def test_grid_eval_matches_reference(P):
    g = GOLD["grid"]
    got = P.grid_eval_mining(g, g, GOLD["data"], 0.15, 9.0, P.SemanticsConfig(mode=P.LogSumExp(5.0)))
    ref = GOLD["grid_values"]
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    ok = ~np.isnan(ref)
    assert _rel(got[ok], ref[ok]) <= 1e-5


def test_mine_interval_matches_reference(P):
    res = P.mine_interval(GOLD["data"], P.MiningConfig(steps=300, lr=5e-2))
    assert _rel(res["loss_history"], GOLD["mine_history"]) <= 1e-4
    assert np.max(np.abs(np.array(res["interval"]) - GOLD["mine_interval"])) <= 1e-4


def test_large_grid_one_launch(P):
    """The paper's 90k-interval sweep shape: a 300 x 300 grid in one call."""
    rng = np.random.default_rng(0)
    data = (rng.normal(0, 0.05, (64, 200)) + (np.arange(200) > 50)).astype(np.float64)
    g = np.linspace(0.0, 1.0, 300)
    out = P.grid_eval_mining(g, g, data, 0.15, 9.0, P.SemanticsConfig(mode=P.LogSumExp(5.0)))
    assert np.isnan(out).sum() == 300 * 301 // 2
    assert np.isfinite(out[np.triu_indices(300, 1)]).all()
    # spot-check against the single-pair entry point
    for (i, j) in [(3, 250), (120, 121), (0, 299)]:
        v = P.mining_objective(g[i], g[j], data, 0.15, 9.0, P.SemanticsConfig(mode=P.LogSumExp(5.0)))
        assert abs(v - out[i, j]) <= 1e-12 * max(1.0, abs(v))
