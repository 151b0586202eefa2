"""B200-native masked STL robustness evaluation and backpropagation.

Drop-in for the hot path of the reference ``stlmask`` package
(``/root/reference/pkg/src/stlmask``): the formula AST, the semantics
configuration and ``robustness`` / ``robustness_trace`` / ``value_and_grad``
keep their names and behaviour; evaluation and gradients run in
hand-written sm_100a CUDA kernels (``csrc/``) behind the C ABI in
``include/stlg.h``.  ``trace`` is the batched, autograd-aware entry point
for ``[B, T]`` CUDA tensors.
"""

from .core import (DivergedError, EmptySignalError, EmptyWindowError, Hard, InvalidIntervalError,
                   LogSumExp, Mode, NamedSignals, NonFiniteSampleError, PaddingPolicy,
                   SemanticsConfig, ShapeError, Signal, SmoothInterval, SoftMax, StepInterval,
                   StlError, ValidationError, make_signal, window_size)
from .formula import (TRUE, Always, And, Eventually, Formula, Negation, NormPred, Not, Or, Pred,
                      Predicate, TrueFormula, Until, from_json, smooth_intervals, to_json,
                      validate_against, variables)
from .engine import (Compiled, Gradients, always_trace, compile_formula, eventually_trace,
                     robustness, robustness_trace, trace, until_trace, value_and_grad)

__version__ = "0.1.0"

from .mining import (AnnealSchedule, MiningConfig, grid_eval_mining, mine_interval, mining_objective,
                     synth_step_dataset)
from .planning import (PlannerConfig, box_formula, plan_trajectory, planning_formula, planning_objective,
                       rollout_single_integrator)

__all__ = [
    "DivergedError", "EmptySignalError", "EmptyWindowError", "Hard", "InvalidIntervalError",
    "LogSumExp", "Mode", "NamedSignals", "NonFiniteSampleError", "PaddingPolicy",
    "SemanticsConfig", "ShapeError", "Signal", "SmoothInterval", "SoftMax", "StepInterval",
    "StlError", "ValidationError", "make_signal", "window_size",
    "TRUE", "Always", "And", "Eventually", "Formula", "Negation", "NormPred", "Not", "Or", "Pred",
    "Predicate", "TrueFormula", "Until", "from_json", "smooth_intervals", "to_json",
    "validate_against", "variables",
    "Compiled", "Gradients", "always_trace", "compile_formula", "eventually_trace", "robustness",
    "robustness_trace", "trace", "until_trace", "value_and_grad",
    "AnnealSchedule", "MiningConfig", "grid_eval_mining", "mine_interval", "mining_objective",
    "synth_step_dataset",
    "PlannerConfig", "box_formula", "plan_trajectory", "planning_formula", "planning_objective",
    "rollout_single_integrator",
]
