"""Golden vectors for trajectory planning, generated from the REFERENCE (dev container only).

Imports the reference's `stlmask.apps` (/root/reference/pkg/src) and records
`planning_objective` at random controls / bounds / (temp, sharp), and a 40-step
`plan_trajectory` (objective history, final controls, interval).  Writes
tests/golden/planning.npz.  Run: python tests/golden/make_planning_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from stlmask import apps  # noqa: E402  (reference)

cfg = apps.PlannerConfig()
rng = np.random.default_rng(11)
pts, vals, ctrls = [], [], []
for k in range(6):
    u = rng.normal(0.0, 0.6, (cfg.horizon, 2)) + np.array([0.4, 0.4])
    a_raw, b_raw = rng.normal(-1.5, 0.5), rng.normal(1.2, 0.5)
    temp, sharp = [(3.0, 0.1), (10.0, 5.0), (100.0, 35.0)][k % 3]
    ctrls.append(u)
    pts.append((a_raw, b_raw, temp, sharp))
    vals.append(apps.planning_objective(u, a_raw, b_raw, cfg, temp=temp, sharp=sharp))
run_cfg = apps.PlannerConfig(steps=40)
res = apps.plan_trajectory(run_cfg, seed=2)
np.savez_compressed(os.path.join(HERE, "planning.npz"), controls=np.array(ctrls), points=np.array(pts),
                    values=np.array(vals), hist=np.array(res["objective_history"]),
                    final_controls=res["controls"], interval=np.array(res["interval"]),
                    final_robustness=np.array(res["final_robustness"]))
print("ok", vals, res["interval"], res["objective_history"][:3], res["objective_history"][-1])
