"""The reference-facing wrappers on the device against the reference's own outputs.

``eventually_trace`` / ``always_trace`` / ``until_trace`` (masking.py:377-401) and
``value_and_grad`` (autodiff.py:64-107, including ``si=`` rebinding) are called exactly
as a ``stlmask`` user calls them, with host arrays / ``NamedSignals``; the expected
values are the reference's (tests/golden/api.npz, make_api_golden.py).

Tolerances (north star): hard mode bit-exact against float32(reference) for values and
exact for gradients; smooth modes |gpu - ref| / max(1, |ref|) <= 1e-5.
"""

import json

import numpy as np
import pytest

import golden_io
from devhelp import rel_err

import paper_2501_04194_b200 as P

pytestmark = pytest.mark.gpu

TOL = 1e-5
API = golden_io.load_api()
WRAP = [c for c in API if "op" in c.meta]
VAG = [c for c in API if "op" not in c.meta]


def _hard(case):
    return json.loads(case.meta["cfg"])["mode"] == "Hard"


@pytest.mark.parametrize("case", WRAP, ids=[f"{c.meta['op']}-{c.meta['src']}-{i}" for i, c in enumerate(WRAP)])
def test_wrappers_match_reference(cuda, case):
    m = case.meta
    iv = case.interval("iv")
    if m["op"] == "U":
        got = P.until_trace(case.arrays["l"], case.arrays["r"], iv, case.cfg)
    else:
        fn = P.eventually_trace if m["op"] == "F" else P.always_trace
        got = fn(case.arrays["x"], iv, case.cfg)
    ref = case.arrays["out"]
    assert isinstance(got, np.ndarray) and got.dtype == np.float64 and got.shape == ref.shape
    if _hard(case):
        assert np.array_equal(got.astype(np.float32).view(np.uint32), ref.astype(np.float32).view(np.uint32))
    else:
        assert rel_err(got, ref) <= TOL


@pytest.mark.parametrize("case", VAG, ids=[f"{c.meta['src']}-{i}" for i, c in enumerate(VAG)])
def test_value_and_grad_matches_reference(cuda, case):
    m = case.meta
    f = P.from_json(m["formula"])
    sig = P.NamedSignals.from_arrays({k: case.arrays["x_" + k] for k in m["channels"]})
    got = P.value_and_grad(f, sig, case.cfg, si=case.interval("si"))
    assert isinstance(got, P.Gradients)
    assert set(got.d_signal) == set(m["channels"])
    ref_v = case.arrays["value"][0]
    if _hard(case):
        assert np.float32(got.value) == np.float32(ref_v)
        for k in m["channels"]:
            np.testing.assert_array_equal(got.d_signal[k], case.arrays["g_" + k])
    else:
        assert rel_err([got.value], [ref_v]) <= TOL
        for k in m["channels"]:
            assert rel_err(got.d_signal[k], case.arrays["g_" + k]) <= TOL, k
    if "dabc" in case.arrays:
        assert rel_err([got.d_a, got.d_b, got.d_c], case.arrays["dabc"]) <= TOL
    else:
        assert got.d_a is None and got.d_b is None and got.d_c is None


def test_robustness_is_trace_entry_zero(cuda):
    rng = np.random.default_rng(3)
    sig = P.NamedSignals.from_arrays({"x": rng.normal(0, 1, 300).astype(np.float32),
                                      "y": rng.normal(0, 1, 300).astype(np.float32)})
    f = P.Until(P.Pred("x", "<", 1.0), P.Eventually(P.Pred("y", ">", 0.5), P.StepInterval(2, 9)))
    for cfg in (P.SemanticsConfig(), P.SemanticsConfig(mode=P.LogSumExp(4.0))):
        tr = P.robustness_trace(f, sig, cfg)
        assert tr.shape == (300,) and tr.dtype == np.float64
        assert P.robustness(f, sig, cfg) == tr[0]


# --- the reference's DSL / CSV / CLI with --engine b200 -----------------

DSL = ["G[0,50] (x > 0.5)", "F[10,100] (x < 0.5)", "(x > 0) U (y < 1)", "(x >= -0.5) U[2,9] (y <= 0.25)",
       "G (F[0,20] (x > 0)) & ((y < 1) U (x > 0))", "~(x > 0) | F (y > 1.5)"]


@pytest.mark.parametrize("mode", ["hard", "lse"])
@pytest.mark.parametrize("text", DSL)
def test_reference_cli_engine_b200(cuda, tmp_path, text, mode):
    """stlmask.formula.parse output and stlmask CSV signals go through the reference CLI
    unchanged; --engine b200 must reproduce --engine masking."""
    from conftest import import_reference
    import_reference()
    import stlmask.cli as cli
    from paper_2501_04194_b200 import stlmask_engine
    stlmask_engine.install(cli)
    rng = np.random.default_rng(len(text))
    L = 400
    x = np.asarray(rng.normal(0, 1, L), dtype=np.float32)
    y = np.asarray(rng.normal(0, 1, L), dtype=np.float32)
    csv = tmp_path / "sig.csv"
    csv.write_text("t,x,y\n" + "".join(f"{i},{repr(float(a))},{repr(float(b))}\n" for i, (a, b) in enumerate(zip(x, y))))
    outs = {}
    for eng in ("masking", "b200"):
        o = tmp_path / f"{eng}.json"
        argv = ["trace", text, str(csv), "--engine", eng, "--out", str(o), "--mode", mode]
        if mode == "lse":
            argv += ["--temp", "5"]
        assert cli.main(argv) == 0
        outs[eng] = np.array(json.loads(o.read_text()))
    if mode == "hard":
        assert np.array_equal(outs["b200"].astype(np.float32), outs["masking"].astype(np.float32))
    else:
        assert rel_err(outs["b200"], outs["masking"]) <= TOL


def test_reference_ast_objects_on_device(cuda):
    """A real stlmask AST, NamedSignals and SemanticsConfig fed to the device API."""
    from conftest import import_reference
    stlmask = import_reference()
    from stlmask import masking
    from stlmask.core import LogSumExp, NamedSignals, SemanticsConfig, SmoothInterval
    from stlmask.formula import Always, Pred, parse
    rng = np.random.default_rng(9)
    sig = NamedSignals.from_arrays({"x": np.asarray(rng.normal(0, 1, 120), dtype=np.float32).astype(np.float64),
                                    "y": np.asarray(rng.normal(0, 1, 120), dtype=np.float32).astype(np.float64)})
    cfg = SemanticsConfig(mode=LogSumExp(5.0))
    for f in (parse("G[0,5] (x > 0) & F (y < 0.5)"), Always(Pred("x", ">", 0.0), SmoothInterval(0.3, 0.65, 9.0))):
        assert rel_err(P.robustness_trace(f, sig, cfg), masking.robustness_trace(f, sig, cfg)) <= TOL
    from stlmask.autodiff import value_and_grad as ref_vag
    f = Always(Pred("x", ">", 0.0), SmoothInterval(0.3, 0.65, 9.0))
    got, ref = P.value_and_grad(f, sig, cfg), ref_vag(f, sig, cfg)
    assert rel_err([got.value, got.d_a, got.d_b, got.d_c], [ref.value, ref.d_a, ref.d_b, ref.d_c]) <= TOL
    with pytest.raises(stlmask.core.ValidationError):
        from paper_2501_04194_b200.stlmask_engine import b200_trace
        b200_trace(parse("F (q > 0)"), sig, cfg)
