"""Trajectory planning with a learnable smooth window on the GPU (
reference apps.py:81-226).

The reference descends on controls u (horizon x 2) and the pre-sigmoid window bounds
(alpha, beta) of `And(Always_[a,b]^smooth(in target box), Eventually(in goal box))`
over the single-integrator rollout, with `tape` gradients.  Here one descent step is
torch autograd around `paper_2501_04194_b200.trace` (the robustness trace and its
gradients to the rolled-out signals and to (a, b) come from the device kernels,
csrc/smooth.cu and csrc/fg*.cu); the control costs and the rollout are torch ops on the
GPU.  Ties in `_ordered_bounds` route the gradient to the first operand, as the
reference's hard max does (apps.py:69-74).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .core import DivergedError, Hard, LogSumExp, NamedSignals, SemanticsConfig, SmoothInterval, StepInterval
from .formula import Always, And, Eventually, Formula, Pred
from .mining import _logit, _schedule


@dataclass(frozen=True)
class PlannerConfig:
    """Weights, geometry and descent settings (apps.py:81-115)."""

    gamma1: float = 1.1
    gamma2: float = 0.05
    gamma3: float = 2.0
    gamma4: float = 0.5
    interval_nominal: float = 0.2
    control_limit: float = 2.0
    dt: float = 0.1
    horizon: int = 51
    target_box: tuple = (0.8, 1.2, 0.8, 1.2)
    goal_box: tuple = (1.8, 2.2, 1.8, 2.2)
    start: tuple = (0.0, 0.0)
    init_interval: tuple = (0.14, 0.82)
    control_init_scale: float = 0.05
    lr: float = 0.06
    steps: int = 4000
    temp_anneal: tuple = ("sigmoid", 3.0, 100.0)
    sharp_anneal: tuple = ("linear", 0.1, 35.0)

    def __post_init__(self):
        if min(self.gamma1, self.gamma2, self.gamma3, self.gamma4) < 0:
            raise ValueError("objective weights must be nonnegative")
        if not self.control_limit > 0:
            raise ValueError("control limit must be positive")
        if not 0 < self.interval_nominal < 1:
            raise ValueError("nominal interval size must lie in (0, 1)")
        if self.horizon < 2:
            raise ValueError("horizon must be at least 2")


def rollout_single_integrator(x0, controls, dt: float) -> np.ndarray:
    """States under x_{t+1} = x_t + dt u_t (apps.py:118-123)."""
    controls = np.asarray(controls, dtype=np.float64)
    x0 = np.asarray(x0, dtype=np.float64)
    return np.concatenate([x0[None, :], x0 + dt * np.cumsum(controls, axis=0)])


def box_formula(box, xname: str = "x", yname: str = "y") -> Formula:
    """Inside-box membership: the conjunction of the four signed margins (apps.py:126-130)."""
    xl, xh, yl, yh = box
    return And(And(Pred(xname, ">", xl), Pred(xname, "<", xh)),
               And(Pred(yname, ">", yl), Pred(yname, "<", yh)))


def planning_formula(cfg: PlannerConfig, si: SmoothInterval) -> Formula:
    return And(Always(box_formula(cfg.target_box), si), Eventually(box_formula(cfg.goal_box)))


def _ordered_bounds(alpha, beta):
    import torch
    sa, sb = torch.sigmoid(alpha), torch.sigmoid(beta)
    hi = torch.where(sa >= sb, sa, sb)  # first argmax of (sa, sb)
    lo = torch.where(sa <= sb, sa, sb)  # first argmax of (-sa, -sb)
    return lo, hi


def _planning_terms(u, alpha, beta, cfg: PlannerConfig, temp: float, sharp: float):
    """Objective terms (apps.py:136-161); u [horizon, 2], alpha / beta 0-d, all float64."""
    import torch
    from .engine import trace
    a, b = _ordered_bounds(alpha, beta)
    start = torch.tensor(cfg.start, dtype=torch.float64, device=u.device)
    pos = torch.cat([start[None, :], torch.cumsum(u, dim=0) * cfg.dt + start])  # [horizon + 1, 2]
    phi = planning_formula(cfg, SmoothInterval(0.25, 0.75, sharp))  # rebound below
    sem = SemanticsConfig(mode=LogSumExp(temp))
    tr = trace(phi, {"x": pos[:, 0].float()[None, :], "y": pos[:, 1].float()[None, :]}, sem,
               smooth_binding=(a, b, sharp))
    rho = tr[0, 0].double()
    sumsq = (u * u).sum(dim=-1)
    norms = torch.sqrt(sumsq + 1e-12)
    j_stl = torch.relu(-rho)
    j_int = torch.exp((a - b + cfg.interval_nominal) * 2.0)
    j_lim = torch.relu(norms - cfg.control_limit).sum() * (1.0 / cfg.horizon)
    j_eff = sumsq.sum() * (1.0 / cfg.horizon)
    total = j_stl * cfg.gamma1 + j_int * cfg.gamma2 + j_lim * cfg.gamma3 + j_eff * cfg.gamma4
    return total, a, b, rho


def planning_objective(controls, a_raw: float, b_raw: float, cfg: PlannerConfig,
                       temp: Optional[float] = None, sharp: Optional[float] = None) -> float:
    """Objective value at given controls and pre-sigmoid bounds (apps.py:164-177)."""
    import torch
    u = torch.tensor(np.asarray(controls, dtype=np.float64), device="cuda")
    if tuple(u.shape) != (cfg.horizon, 2):
        raise ValueError(f"controls must have shape ({cfg.horizon}, 2), got {tuple(u.shape)}")
    temp = cfg.temp_anneal[2] if temp is None else temp
    sharp = cfg.sharp_anneal[2] if sharp is None else sharp
    al = torch.tensor(float(a_raw), dtype=torch.float64, device="cuda")
    be = torch.tensor(float(b_raw), dtype=torch.float64, device="cuda")
    total, _, _, _ = _planning_terms(u, al, be, cfg, temp, sharp)
    return float(total.item())


def _hard_interval(a: float, b: float, length: int) -> StepInterval:
    lo = int(math.ceil(a * length))
    hi = max(lo, int(math.floor(b * length)))
    return StepInterval(lo, hi)


def plan_trajectory(cfg: PlannerConfig = PlannerConfig(), seed: int = 0) -> dict:
    """Descend on controls and window bounds (apps.py:186-226); returns the same
    artifacts.  `final_robustness` is the hard robustness of the optimised
    specification with the window rounded to [ceil(aL), floor(bL)]."""
    import torch
    from .engine import robustness
    rng = np.random.default_rng(seed)
    u = torch.tensor(rng.normal(0.0, cfg.control_init_scale, (cfg.horizon, 2)), device="cuda")
    alpha = torch.tensor(_logit(cfg.init_interval[0]), dtype=torch.float64, device="cuda")
    beta = torch.tensor(_logit(cfg.init_interval[1]), dtype=torch.float64, device="cuda")
    temp_sched = _schedule(cfg.temp_anneal, cfg.steps)
    sharp_sched = _schedule(cfg.sharp_anneal, cfg.steps)
    history = []
    for step in range(cfg.steps):
        uv = u.detach().requires_grad_(True)
        av = alpha.detach().requires_grad_(True)
        bv = beta.detach().requires_grad_(True)
        total, a_var, b_var, _ = _planning_terms(uv, av, bv, cfg, temp_sched.value(step), sharp_sched.value(step))
        value = float(total.item())
        if not math.isfinite(value):
            raise DivergedError(f"planning objective became {value} at step {step}")
        assert 0.0 <= float(a_var.detach()) < float(b_var.detach()) <= 1.0, \
            "interval reparameterization escaped 0 <= a < b <= 1"
        history.append(value)
        gu, ga, gb = torch.autograd.grad(total, [uv, av, bv])
        u = u - cfg.lr * gu
        alpha = alpha - cfg.lr * ga
        beta = beta - cfg.lr * gb
    a = float(torch.sigmoid(alpha))
    b = float(torch.sigmoid(beta))
    a, b = min(a, b), max(a, b)
    controls = u.cpu().numpy()
    states = rollout_single_integrator(cfg.start, controls, cfg.dt)
    length = cfg.horizon + 1
    signals = NamedSignals.from_arrays({"x": states[:, 0], "y": states[:, 1]}, dt=cfg.dt)
    hard_phi = And(Always(box_formula(cfg.target_box), _hard_interval(a, b, length)),
                   Eventually(box_formula(cfg.goal_box)))
    rho_final = robustness(hard_phi, signals, SemanticsConfig(mode=Hard()))
    return {"controls": controls, "states": states, "interval": (a, b),
            "objective_history": history, "final_robustness": rho_final}
