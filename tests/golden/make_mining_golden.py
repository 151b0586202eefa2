"""Golden vectors for interval mining, generated from the REFERENCE (dev container only).

Imports the reference's `stlmask.apps` (/root/reference/pkg/src) and records, for
datasets from its own `synth_step_dataset` (apps.py:252-269):
  * `mining_objective` at several (a, b, gamma, sharp) in Hard / LSE / softmax,
  * `grid_eval` of the LSE objective over a 13 x 13 (a, b) grid,
  * `mine_interval` (300 steps) final interval and loss history.
Writes tests/golden/mining.npz.  Run: python tests/golden/make_mining_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from stlmask import apps  # noqa: E402  (reference)
from stlmask.core import Hard, LogSumExp, SemanticsConfig, SoftMax  # noqa: E402

out = {}
data = apps.synth_step_dataset(seed=3, n=64, length=40)
out["data"] = data
modes = {"hard": Hard(), "lse": LogSumExp(5.0), "soft": SoftMax(4.0)}
pts = [(0.2, 0.6, 0.15, 9.0), (0.05, 0.95, 0.0, 4.0), (0.3, 0.5, 0.3, 20.0), (0.22, 0.61, 0.15, 2.0)]
vals = []
for (a, b, gamma, sharp) in pts:
    row = [apps.mining_objective(a, b, data, gamma, sharp, SemanticsConfig(mode=m)) for m in modes.values()]
    vals.append(row)
out["obj_points"] = np.array(pts)
out["obj_values"] = np.array(vals)  # [points, (hard, lse, soft)]
grid = np.linspace(0.0, 1.0, 13)
cfg = SemanticsConfig(mode=LogSumExp(5.0))
out["grid"] = grid
out["grid_values"] = apps.grid_eval(grid, grid, lambda a, b: apps.mining_objective(a, b, data, 0.15, 9.0, cfg))
mc = apps.MiningConfig(steps=300, lr=5e-2)
res = apps.mine_interval(data, mc)
out["mine_interval"] = np.array(res["interval"])
out["mine_history"] = np.array(res["loss_history"])
np.savez_compressed(os.path.join(HERE, "mining.npz"), **out)
print("wrote", os.path.join(HERE, "mining.npz"), {k: np.shape(v) for k, v in out.items()})
