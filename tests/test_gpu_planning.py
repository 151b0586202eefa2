"""Trajectory planning on the device vs the reference.

Golden vectors from the reference's `apps` (tests/golden/make_planning_golden.py):
`planning_objective` at random controls / window bounds / (temp, sharp), and a
40-step `plan_trajectory`.  The robustness and its gradients run in fp32 on the
device (the reference in f64), so objective values agree to 1e-5 and the descent
trajectory to 1e-4.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "planning.npz"))


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


def test_planning_objective_matches_reference(P):
    from paper_2501_04194_b200 import planning
    cfg = planning.PlannerConfig()
    for u, (a_raw, b_raw, temp, sharp), ref in zip(GOLD["controls"], GOLD["points"], GOLD["values"]):
        got = planning.planning_objective(u, a_raw, b_raw, cfg, temp=temp, sharp=sharp)
        assert _rel(got, ref) <= 1e-5, (got, ref)


def test_plan_trajectory_matches_reference(P):
    from paper_2501_04194_b200 import planning
    res = planning.plan_trajectory(planning.PlannerConfig(steps=40), seed=2)
    assert _rel(res["objective_history"], GOLD["hist"]) <= 1e-4
    assert _rel(res["controls"], GOLD["final_controls"]) <= 1e-4
    assert np.max(np.abs(np.array(res["interval"]) - GOLD["interval"])) <= 1e-5
    assert abs(res["final_robustness"] - float(GOLD["final_robustness"])) <= 1e-4
