"""Interval mining on the GPU (reference apps.py:234-335).

The reference mines the widest window [a, b] over which a dataset stays positive by
gradient descent on `_mining_loss_var` (apps.py:272-280), and `grid_eval`
(apps.py:326-335) maps the objective over an (a, b) grid one pair per call — the
paper's 90k-interval sweep.  Here the objective of every pair runs in one launch of
`stlg_mining_grid` (csrc/mining.cu): fp64 window weights, per-row weighted smooth
min, hinge mean, and (for the descent) d loss / d(a, b).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import DivergedError, EmptyWindowError, Hard, LogSumExp, SemanticsConfig, SoftMax

Schedule = tuple  # (kind, start, end), apps.py:52


@dataclass(frozen=True)
class AnnealSchedule:
    """Scheduled parameter value (smoothing.py:112-160): constant, linear or a
    sigmoid rescaled to hit `start` and `end` exactly (midpoint slope 12)."""

    kind: str
    start: float
    end: float
    total: int = 1

    def __post_init__(self):
        if self.kind not in ("constant", "linear", "sigmoid"):
            raise ValueError(f"unknown schedule kind {self.kind!r}")
        if self.total < 1:
            raise ValueError("total steps must be >= 1")
        if not (self.start > 0 and self.end > 0):
            raise ValueError("schedule values must stay positive")

    def value(self, step: int) -> float:
        if self.kind == "constant":
            return self.start
        if not 0 <= step <= self.total:
            raise ValueError(f"step {step} outside [0, {self.total}]")
        p = step / self.total
        if self.kind == "linear":
            return self.start + (self.end - self.start) * p
        lo, hi = _sigmoid(-6.0), _sigmoid(6.0)
        frac = (_sigmoid(12.0 * (p - 0.5)) - lo) / (hi - lo)
        return self.start + (self.end - self.start) * frac


@dataclass(frozen=True)
class MiningConfig:
    """Descent settings (apps.py:234-249)."""

    gamma: float = 0.15
    lr: float = 1e-2
    steps: int = 5000
    init_interval: tuple = (0.1, 0.9)
    eps: float = 0.0
    temp_anneal: Schedule = ("sigmoid", 1.0, 30.0)
    sharp_anneal: Schedule = ("sigmoid", 2.0, 50.0)

    def __post_init__(self):
        if self.gamma < 0:
            raise ValueError("gamma must be nonnegative")
        if self.steps < 1:
            raise ValueError("steps must be >= 1")


def synth_step_dataset(seed: int, n: int = 64, length: int = 20,
                       truth: tuple = (0.23, 0.59), value_noise: float = 0.05) -> np.ndarray:
    """Noisy step signals, 1 inside the truth window and 0 outside, each window edge
    jittered by one sample (apps.py:252-269; same generator calls, so the same data for a
    seed).  The mining dataset and the C4 benchmark input (seed 3,
    n=4096, length=2000)."""
    rng = np.random.default_rng(seed)
    lo = int(math.ceil(truth[0] * length))
    hi = int(math.floor(truth[1] * length))
    data = np.zeros((n, length))
    for row in range(n):
        jlo = lo + int(rng.integers(-1, 2))
        jhi = hi + int(rng.integers(-1, 2))
        data[row, max(jlo, 0):min(jhi, length - 1) + 1] = 1.0
    data += rng.normal(0.0, value_noise, (n, length))
    return data


def _sigmoid(z: float) -> float:
    if z >= 0:
        return 1.0 / (1.0 + math.exp(-z))
    e = math.exp(z)
    return e / (1.0 + e)


def _schedule(spec, total):
    kind, start, end = spec
    if kind == "constant":
        return AnnealSchedule("constant", start, start, 1)
    return AnnealSchedule(kind, float(start), float(end), max(int(total), 1))


def _logit(p: float) -> float:
    if not 0.0 < p < 1.0:
        raise ValueError(f"initial bound must lie strictly inside (0, 1), got {p}")
    return math.log(p / (1.0 - p))


def _mode_code(cfg: SemanticsConfig):
    m = cfg.mode
    if isinstance(m, Hard):
        return 0, 1.0
    if isinstance(m, SoftMax):
        return 1, float(m.temp)
    if isinstance(m, LogSumExp):
        return 2, float(m.temp)
    raise TypeError(f"unsupported mode: {m!r}")


def _device_dataset(dataset):
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2501_04194_b200 requires a CUDA device; there is no CPU path")
    if isinstance(dataset, torch.Tensor):
        x = dataset.detach().to(device="cuda", dtype=torch.float32)
    else:
        x = torch.tensor(np.asarray(dataset, dtype=np.float64), dtype=torch.float32, device="cuda")
    if x.dim() != 2 or x.numel() == 0:
        raise ValueError("dataset must be a non-empty (n, length) array")
    return x.contiguous()


def _grid(x, a, b, sharp, eps, gamma, cfg, with_grad=False):
    """loss [P] (and d loss / d(a, b) [P, 2]) for device fp64 pair arrays a, b."""
    import torch
    lib = _lib.load()
    mode, temp = _mode_code(cfg)
    loss = torch.empty(a.numel(), dtype=torch.float64, device=x.device)
    dl = torch.empty(2 * a.numel(), dtype=torch.float64, device=x.device) if with_grad else None
    with torch.cuda.device(x.device):
        stream = ctypes.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
        _lib.check(lib.stlg_mining_grid(x.data_ptr(), x.shape[0], x.shape[1], x.stride(0), a.data_ptr(),
                                        b.data_ptr(), a.numel(), float(sharp), float(eps), mode, temp,
                                        float(gamma), loss.data_ptr(),
                                        dl.data_ptr() if dl is not None else None, stream))
    return loss, (dl.view(-1, 2) if dl is not None else None)


def mining_objective(a: float, b: float, dataset, gamma: float, sharp: float,
                     cfg: SemanticsConfig, eps: float = 0.0) -> float:
    """Mean hinge violation of staying positive over the smooth window [a, b]
    (apps.py:283-295), evaluated on the device."""
    import torch
    x = _device_dataset(dataset)
    av = torch.tensor([float(a)], dtype=torch.float64, device=x.device)
    bv = torch.tensor([float(b)], dtype=torch.float64, device=x.device)
    loss, _ = _grid(x, av, bv, sharp, eps, gamma, cfg)
    v = float(loss.item())
    if math.isnan(v):
        raise EmptyWindowError("smooth interval produced an all-zero weight vector")
    return v


def grid_eval_mining(a_grid, b_grid, dataset, gamma: float, sharp: float, cfg: SemanticsConfig,
                     eps: float = 0.0) -> np.ndarray:
    """`grid_eval(a_grid, b_grid, lambda a, b: mining_objective(a, b, ...))`
    (apps.py:326-335) in one launch: an [len(a), len(b)] matrix, NaN where a >= b."""
    import torch
    x = _device_dataset(dataset)
    ag = np.asarray(a_grid, dtype=np.float64).reshape(-1)
    bg = np.asarray(b_grid, dtype=np.float64).reshape(-1)
    out = np.full((ag.size, bg.size), np.nan)
    ii, jj = np.nonzero(ag[:, None] < bg[None, :])
    if ii.size == 0:
        return out
    av = torch.tensor(ag[ii], dtype=torch.float64, device=x.device)
    bv = torch.tensor(bg[jj], dtype=torch.float64, device=x.device)
    loss, _ = _grid(x, av, bv, sharp, eps, gamma, cfg)
    vals = loss.cpu().numpy()
    if np.isnan(vals).any():
        raise EmptyWindowError("smooth interval produced an all-zero weight vector")
    out[ii, jj] = vals
    return out


def mine_interval(dataset, cfg: MiningConfig = MiningConfig()) -> dict:
    """Gradient descent on sigmoid-reparameterised window bounds (apps.py:298-323):
    each step's loss and d loss / d(a, b) come from one device launch."""
    import torch
    x = _device_dataset(dataset)
    alpha = _logit(cfg.init_interval[0])
    beta = _logit(cfg.init_interval[1])
    temp_sched = _schedule(cfg.temp_anneal, cfg.steps)
    sharp_sched = _schedule(cfg.sharp_anneal, cfg.steps)
    ab = torch.empty(2, dtype=torch.float64, device=x.device)
    history = []
    for step in range(cfg.steps):
        sem = SemanticsConfig(mode=LogSumExp(temp_sched.value(step)))
        sa, sb = _sigmoid(alpha), _sigmoid(beta)
        # _ordered_bounds (apps.py:69-74): first-argmax ties route both bounds to alpha
        hi_is_a = sa >= sb
        lo_is_a = sa <= sb
        a, b = (sa if lo_is_a else sb), (sa if hi_is_a else sb)
        ab[0], ab[1] = a, b
        loss, dl = _grid(x, ab[0:1], ab[1:2], sharp_sched.value(step), cfg.eps, cfg.gamma, sem,
                         with_grad=True)
        lv, g = loss.item(), dl[0].tolist()
        if not math.isfinite(lv):
            raise DivergedError(f"mining loss became {lv} at step {step}")
        assert 0.0 <= a < b <= 1.0, "interval reparameterization escaped 0 <= a < b <= 1"
        history.append(lv)
        dsa = (g[0] if lo_is_a else 0.0) + (g[1] if hi_is_a else 0.0)
        dsb = (g[0] if not lo_is_a else 0.0) + (g[1] if not hi_is_a else 0.0)
        alpha -= cfg.lr * dsa * sa * (1.0 - sa)
        beta -= cfg.lr * dsb * sb * (1.0 - sb)
    a = _sigmoid(alpha)
    b = _sigmoid(beta)
    a, b = min(a, b), max(a, b)
    return {"interval": (a, b), "loss_history": history}
