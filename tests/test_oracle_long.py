"""Pins the O(L)-memory oracle restatements (oracle/stl_oracle.py: until_untimed_hard,
suffix_hard) to the tape oracle, which is itself pinned to the reference
(tests/test_oracle_golden.py).  The long-signal GPU tests (tests/test_gpu_long.py)
use these restatements where the tape oracle's O(L^2) memory does not fit.
Hard mode: values compared bitwise (signed zeros included), gradients exactly."""

import numpy as np
import pytest

import stl_oracle

import paper_2501_04194_b200 as P


def _ties(rng, shape):
    v = rng.integers(-2, 3, shape).astype(np.float64)
    v[rng.random(shape) < 0.1] = -0.0
    return v


@pytest.mark.parametrize("seed", range(6))
def test_until_untimed_hard_matches_tape_oracle(seed):
    rng = np.random.default_rng(seed)
    L = int(rng.integers(1, 70))
    x, y = _ties(rng, (3, L)), _ties(rng, (3, L))
    cot = np.ones((3, L)) if seed % 2 == 0 else rng.normal(0, 1, (3, L))
    f = P.Until(P.Pred("x", ">", 0.0), P.Pred("y", "<", 0.0))
    ref, g, _ = stl_oracle.trace_and_grad(f, {"x": x, "y": y}, P.SemanticsConfig(), cot)
    # the predicates' traces: x - 0 and -y + 0 (masking.py:316-322)
    out, dl, dr = stl_oracle.until_untimed_hard(x - 0.0, -y + 0.0, cot)
    assert np.array_equal(out.view(np.uint64), ref.view(np.uint64))
    np.testing.assert_allclose(dl, g["x"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(-dr, g["y"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("kind", ["max", "min"])
@pytest.mark.parametrize("seed", range(4))
def test_suffix_hard_matches_tape_oracle(kind, seed):
    rng = np.random.default_rng(10 + seed)
    L = int(rng.integers(1, 200))
    x = _ties(rng, (2, L))
    cot = rng.normal(0, 1, (2, L))
    node = P.Eventually if kind == "max" else P.Always
    ref, g, _ = stl_oracle.trace_and_grad(node(P.Pred("x", ">", 0.0)), {"x": x}, P.SemanticsConfig(), cot)
    out, gx = stl_oracle.suffix_hard(x - 0.0, cot, kind)
    assert np.array_equal(out.view(np.uint64), ref.view(np.uint64))
    np.testing.assert_allclose(gx, g["x"], rtol=0, atol=1e-12)
