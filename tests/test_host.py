"""Host-side logic that needs no GPU: types, validation, lowering, the C ABI surface."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2501_04194_b200 as P
from paper_2501_04194_b200 import _lib
from paper_2501_04194_b200.lower import lower, smooth_weights_np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


# --- core types mirror the reference's validation (core.py:157-279) -----------

def test_interval_validation():
    with pytest.raises(P.InvalidIntervalError):
        P.StepInterval(3, 2)
    with pytest.raises(P.InvalidIntervalError):
        P.StepInterval(-1, 2)
    with pytest.raises(P.InvalidIntervalError):
        P.StepInterval(0.5, 2)
    with pytest.raises(P.InvalidIntervalError):
        P.SmoothInterval(0.6, 0.5)
    with pytest.raises(P.InvalidIntervalError):
        P.SmoothInterval(0.1, 0.5, c=0.0)
    with pytest.raises(P.InvalidIntervalError):
        P.SmoothInterval(0.1, 0.5, eps=0.5)
    assert P.window_size(P.StepInterval(10, 100)) == 91


def test_config_validation():
    with pytest.raises(ValueError):
        P.LogSumExp(0.0)
    with pytest.raises(ValueError):
        P.SoftMax(-1.0)
    with pytest.raises(ValueError):
        P.SemanticsConfig(top_value=0.0)
    with pytest.raises(ValueError):
        P.PaddingPolicy("mirror")
    with pytest.raises(P.NonFiniteSampleError):
        P.PaddingPolicy.constant(float("inf"))
    with pytest.raises(TypeError):
        P.SemanticsConfig(mode="hard")


def test_signals_validation():
    with pytest.raises(P.EmptySignalError):
        P.make_signal([])
    with pytest.raises(P.NonFiniteSampleError):
        P.make_signal([1.0, float("nan")])
    with pytest.raises(P.ShapeError):
        P.NamedSignals.from_arrays({"x": [1.0, 2.0], "y": [1.0]})
    s = P.NamedSignals.from_arrays({"x": np.arange(4.0)})
    assert s.length == 4 and "x" in s and s.names() == ["x"]


def test_formula_nodes_and_aliases():
    f = P.Predicate("x", ">", 0.5) & ~P.Pred("y", "<=", 1.0)
    assert isinstance(f, P.And) and isinstance(f.right, P.Negation)
    assert P.variables(f) == {"x", "y"}
    with pytest.raises(ValueError):
        P.Pred("1x", ">", 0.0)
    with pytest.raises(ValueError):
        P.Pred("x", "==", 0.0)
    s = P.NamedSignals.from_arrays({"x": [1.0]})
    assert P.validate_against(f, s) == ["y"]
    assert P.from_json(P.to_json(f)) == f
    g = P.Until(P.TRUE, P.Eventually(P.NormPred(("a", "b"), "<", 0.5), P.SmoothInterval(0.1, 0.6, 4.0)),
                P.StepInterval(1, 4))
    assert P.from_json(P.to_json(g)) == g


def test_lowering_merges_shared_subformulas():
    leaf = P.Pred("x", ">", 0.0)
    f = P.And(P.Eventually(leaf, P.StepInterval(0, 3)), P.Eventually(leaf, P.StepInterval(0, 3)))
    low = lower(f, ["x"])
    # pred, F, And: the two identical F nodes are one node
    assert [n["op"] for n in low.nodes] == [_lib.OP_PRED, _lib.OP_EV, _lib.OP_AND]
    assert low.nodes[2]["left"] == low.nodes[2]["right"] == 1


def test_lowering_rejects_smooth_until():
    with pytest.raises(TypeError):
        lower(P.Until(P.Pred("x", ">", 0.0), P.Pred("x", ">", 0.0), P.SmoothInterval(0.1, 0.5)), ["x"])


def test_lowering_accepts_reference_like_objects():
    # duck typing by class name + fields: a look-alike class from "elsewhere"
    from dataclasses import dataclass

    @dataclass(frozen=True)
    class Pred:
        var: str
        cmp: str
        threshold: float

    @dataclass(frozen=True)
    class Eventually:
        arg: object
        interval: object = None

    low = lower(Eventually(Pred("x", "<", 1.0), P.StepInterval(2, 5)), ["x"])
    assert low.nodes[-1]["op"] == _lib.OP_EV and low.nodes[-1]["a"] == 2
    assert low.nodes[0]["cmp"] == 1


def test_smooth_weights_match_reference_formula():
    w = smooth_weights_np(0.3, 0.65, 9.0, 0.0, 2000)
    i = np.arange(2000.0)
    sig = lambda z: 1.0 / (1.0 + np.exp(-z))
    with np.errstate(over="ignore"):
        ref = np.maximum(sig(9.0 * (i - 600.0)) - sig(9.0 * (i - 1300.0)), 0.0)
    np.testing.assert_allclose(w, ref, rtol=1e-12, atol=1e-300)
    # the kept set is contiguous and includes tiny positive tails (SURVEY hard parts)
    kept = np.flatnonzero(w > 0)
    assert np.all(np.diff(kept) == 1)
    assert kept[0] < 600 - 50


# --- the C ABI library ---------------------------------------------------------

def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "stlg.h")).read()
    return sorted(set(re.findall(r"STLG_API\s+[\w\s\*]+?\b(stlg_\w+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _declared_symbols()
    assert set(declared) == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.stlg_abi_version() == _lib.ABI_VERSION


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_lib.StlgNode) == 64
    assert ctypes.sizeof(_lib.StlgCfg) == 56
    assert ctypes.sizeof(_lib.StlgChannel) == 24
    assert ctypes.sizeof(_lib.StlgGrad) == 32
    assert ctypes.sizeof(_lib.StlgSmooth) == 32


def test_compile_and_plan_info_without_gpu():
    f = P.And(P.Always(P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(0, 200))),
              P.Until(P.Pred("y", "<", 1.0), P.Pred("z", ">", 0.0)))
    c = P.compile_formula(f, ["x", "y", "z"], P.SemanticsConfig())
    assert (c.n_temporal, c.n_slots, c.root_temporal) == (3, 3, 0)
    fb, bb = c.workspace_bytes(256, 4000)
    assert fb >= 3 * 256 * 4000 * 4 and bb >= 3 * 256 * 4000 * 4


def test_independent_operands_get_a_second_lane():
    """exec.cu assign_lanes: operands under the root that share no channel, slot or smooth
    binding run on two streams, each lane with its own scratch — visible through the C ABI
    as one more lane block in both workspaces.  A shared channel keeps one lane."""
    cfg = P.SemanticsConfig()
    left = P.Always(P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(0, 200)))
    two = P.compile_formula(P.And(left, P.Until(P.Pred("y", "<", 1.0), P.Pred("z", ">", 0.0))),
                            ["x", "y", "z"], cfg)
    one = P.compile_formula(P.And(left, P.Until(P.Pred("y", "<", 1.0), P.Pred("x", ">", 0.5))),
                            ["x", "y", "z"], cfg)
    B, T = 64, 5000
    (f2, b2), (f1, b1) = two.workspace_bytes(B, T), one.workspace_bytes(B, T)
    assert f2 > f1 and b2 - b1 >= 3 * B * T * 4


def test_compile_errors_map_to_reference_exceptions():
    lib = _lib.load()
    arr = (_lib.StlgNode * 1)()
    arr[0].op = 99
    cfg = _lib.StlgCfg()
    plan = ctypes.c_void_p()
    rc = lib.stlg_compile(arr, 1, 0, 0, ctypes.byref(cfg), ctypes.byref(plan))
    assert rc == _lib.E_INVALID
    with pytest.raises(ValueError):
        _lib.check(rc)
    ws_f, ws_b = ctypes.c_size_t(), ctypes.c_size_t()
    c = P.compile_formula(P.Pred("x", ">", 0.0), ["x"], P.SemanticsConfig())
    with pytest.raises(P.ShapeError):
        _lib.check(lib.stlg_workspace_bytes(c.plan, 0, 10, ctypes.byref(ws_f), ctypes.byref(ws_b)))


def test_large_elementwise_trees_are_split():
    # 20 predicates under one temporal node exceed one fused expression:
    # the compiler materialises sub-trees into pointwise slots
    leaves = [P.Pred("x", ">", float(i)) for i in range(20)]
    f = leaves[0]
    for l in leaves[1:]:
        f = P.And(f, l)
    c = P.compile_formula(P.Eventually(f, P.StepInterval(0, 4)), ["x"], P.SemanticsConfig())
    assert c.n_slots >= 1 and c.root_temporal == 1


def test_anneal_schedule_matches_reference_formula():
    """smoothing.py:146-160: endpoints hit exactly, sigmoid midpoint."""
    from paper_2501_04194_b200.mining import AnnealSchedule
    s = AnnealSchedule("sigmoid", 1.0, 30.0, 100)
    assert abs(s.value(0) - 1.0) < 1e-12 and abs(s.value(100) - 30.0) < 1e-12
    assert abs(s.value(50) - 15.5) < 1e-12
    lin = AnnealSchedule("linear", 2.0, 4.0, 10)
    assert abs(lin.value(5) - 3.0) < 1e-12
    assert AnnealSchedule("constant", 7.0, 7.0, 1).value(123) == 7.0
    with pytest.raises(ValueError):
        AnnealSchedule("cubic", 1.0, 2.0, 3)


# --- reference error paths of the public wrappers (raised before any device call) ----

def test_value_and_grad_binding_errors():
    """autodiff.py:77-83 (test_autodiff.py:149-158): si= without a smooth node, and
    distinct smooth intervals without si=, raise ValueError; missing channels raise
    ValidationError (masking.py:353-355)."""
    sig = P.NamedSignals.from_arrays({"s": [1.0, 2.0]})
    with pytest.raises(ValueError, match="no smooth-interval node"):
        P.value_and_grad(P.Eventually(P.Pred("s", ">", 0.0)), sig, si=P.SmoothInterval(0.2, 0.8, 4.0))
    f = P.And(P.Always(P.Pred("s", ">", 0.0), P.SmoothInterval(0.1, 0.5, 4.0)),
              P.Eventually(P.Pred("s", ">", 0.0), P.SmoothInterval(0.2, 0.9, 4.0)))
    with pytest.raises(ValueError, match="multiple distinct smooth intervals"):
        P.value_and_grad(f, P.NamedSignals.from_arrays({"s": np.ones(8)}),
                         P.SemanticsConfig(mode=P.LogSumExp(5.0)))
    with pytest.raises(P.ValidationError):
        P.value_and_grad(P.Eventually(P.Pred("q", ">", 0.0)), sig)
    with pytest.raises(P.ValidationError):
        P.robustness_trace(P.Eventually(P.Pred("q", ">", 0.0)), sig)


def test_trace_wrapper_shape_errors():
    """masking.py:370-374, 398-399 (test_masking.py:177-179): empty traces and length
    mismatches raise ShapeError; a smooth Until raises TypeError (masking.py:239-240)."""
    with pytest.raises(P.ShapeError):
        P.eventually_trace([], P.StepInterval(0, 1))
    with pytest.raises(P.ShapeError):
        P.always_trace(np.zeros(0), None)
    with pytest.raises(P.ShapeError):
        P.until_trace([1.0, 2.0], [1.0], None)
    with pytest.raises(P.ShapeError):
        P.until_trace([], [], None)
    with pytest.raises(TypeError):
        P.until_trace([1.0, 2.0], [1.0, 0.0], P.SmoothInterval(0.1, 0.5))


def test_engine_hook_registers_b200_choice(tmp_path):
    """the reference CLI gains --engine b200 (cli.py:190-191) and its other
    engines keep working unchanged."""
    from conftest import import_reference
    import_reference()
    import json
    import stlmask.cli as cli
    from paper_2501_04194_b200 import stlmask_engine
    stlmask_engine.install(cli)
    stlmask_engine.install(cli)  # idempotent
    p = cli.build_parser()
    args = p.parse_args(["trace", "F[0,2] (x > 0)", "s.csv", "--engine", "b200"])
    assert args.engine == "b200"
    csv = tmp_path / "s.csv"
    csv.write_text("x\n1\n3\n2\n0\n")
    out = tmp_path / "o.json"
    assert cli.main(["trace", "F[0,2] (x > 0)", str(csv), "--engine", "masking", "--out", str(out)]) == 0
    assert json.loads(out.read_text()) == [3.0, 3.0, 0.0, 0.0]  # overrun -> last (masking.py:180-192)


def test_synth_step_dataset_matches_reference():
    """apps.py:252-269: the C4 / mining input generator reproduces the reference's data."""
    from conftest import import_reference
    import_reference()
    from stlmask.apps import synth_step_dataset as ref
    for seed, n, L in ((3, 8, 2000), (0, 64, 20)):
        assert np.array_equal(P.synth_step_dataset(seed, n, L), ref(seed, n=n, length=L))


def test_plan_cache_is_bounded_lru(monkeypatch):
    """compile_formula keeps at most PLAN_CACHE_SIZE plans (annealing loops in
    mining / planning compile a new temperature every step)."""
    from paper_2501_04194_b200 import engine
    monkeypatch.setattr(engine, "PLAN_CACHE_SIZE", 4)
    engine._PLANS.clear()
    f = P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(0, 3))
    plans = [engine.compile_formula(f, ["x"], P.SemanticsConfig(mode=P.LogSumExp(1.0 + k))) for k in range(6)]
    assert len(engine._PLANS) == 4
    assert engine.compile_formula(f, ["x"], P.SemanticsConfig(mode=P.LogSumExp(6.0))) is plans[-1]
    assert engine.compile_formula(f, ["x"], P.SemanticsConfig(mode=P.LogSumExp(1.0))) is not plans[0]
