"""Smooth-interval LSE branches (csrc/smooth.cu) against the oracle:

* cotangent scales 1e-9 and 1e7 (the factorised d/dw pass scales |g| by a power of two);
* kept-offset counts K around the 1024-offset staging chunk (S_CH) and K mod 4 != 0
  (the register-blocked 4-offset groups), plus K = 3000 (three chunks);
* tiles whose child span lands just below / above the factorised paths' range limits
  (96 / tau2 forward, 100 / tau2 d/dw), so both the fast and the exact branch run.

Tolerance: |gpu - ref| / max(1, |ref|) <= 1e-5 on the trace, d x and d(a, b, c), with
gradients divided by the cotangent scale first (masking.py:207-215, smoothing.py:85-109).
"""

import numpy as np
import pytest

import stl_oracle
from devhelp import rel_err, run_device

import paper_2501_04194_b200 as P
from paper_2501_04194_b200.lower import smooth_weights_np

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _kept(a, b, c, L):
    return int(np.count_nonzero(smooth_weights_np(a, b, c, 0.0, L) > 0))


def _interval_with_k(K, L, a=0.1, c=9.0):
    """SmoothInterval(a, b, c) whose kept-offset count over length L is exactly K."""
    lo, hi = a + 1e-6, 1.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if _kept(a, mid, c, L) < K:
            lo = mid
        else:
            hi = mid
    b = float(np.float32(hi))
    for cand in (b, float(np.nextafter(np.float32(b), np.float32(2))), float(np.nextafter(np.float32(b), np.float32(0)))):
        if _kept(a, cand, c, L) == K:
            return P.SmoothInterval(a, cand, c)
    pytest.skip(f"no fp32 b gives K={K} at L={L}")


def _check(f, x, cfg, si, cot):
    binding = (si.a, si.b, si.c)
    ref_tr, ref_g, ref_abc = stl_oracle.trace_and_grad(f, {"x": x}, cfg, cotangent=cot, smooth_binding=binding)
    tr, g, dabc = run_device(f, {"x": x}, cfg, cot, binding)
    scale = float(np.max(np.abs(cot)))
    assert rel_err(tr, ref_tr) <= TOL
    assert rel_err(g["x"] / scale, ref_g["x"] / scale) <= TOL
    assert rel_err(dabc / scale, np.array(ref_abc) / scale) <= TOL


@pytest.mark.parametrize("scale", [1e-9, 1.0, 1e7])
def test_smooth_lse_cotangent_scales(cuda, scale):
    rng = np.random.default_rng(17)
    B, L = 3, 700
    x = np.cumsum(np.asarray(rng.normal(0, 0.2, (B, L)), dtype=np.float32), axis=1).astype(np.float64)
    si = P.SmoothInterval(0.3, 0.65, 9.0)
    cot = np.asarray(rng.uniform(0.25, 1.75, (B, L)) * scale, dtype=np.float32).astype(np.float64)
    _check(P.Always(P.Pred("x", ">", 0.0), si), x, P.SemanticsConfig(mode=P.LogSumExp(5.0)), si, cot)


@pytest.mark.parametrize("K", [1021, 1022, 1023, 1024, 1025, 3000])
def test_smooth_lse_kept_counts(cuda, K):
    L = int(K / 0.55) + 40
    si = _interval_with_k(K, L)
    rng = np.random.default_rng(K)
    x = np.asarray(rng.normal(0, 1, (1, L)), dtype=np.float32).astype(np.float64)
    cot = np.asarray(rng.uniform(0.5, 1.5, (1, L)), dtype=np.float32).astype(np.float64)
    _check(P.Eventually(P.Pred("x", ">", 0.25), si), x, P.SemanticsConfig(mode=P.LogSumExp(3.0)), si, cot)


@pytest.mark.parametrize("span", [90.0, 95.5, 96.5, 99.5, 100.5, 104.0])
def test_smooth_lse_span_thresholds(cuda, span):
    """Two levels per tile, tau2 * (level gap) = span log2 units."""
    tau = 5.0
    tau2 = tau / np.log(2.0)
    L = 900
    rng = np.random.default_rng(int(span * 10))
    lev = (rng.random((2, L)) < 0.5) * (span / tau2)
    x = np.asarray(lev + rng.normal(0, 1e-3, (2, L)), dtype=np.float32).astype(np.float64)
    si = P.SmoothInterval(0.2, 0.7, 9.0)
    cot = np.asarray(rng.uniform(0.5, 1.5, (2, L)), dtype=np.float32).astype(np.float64)
    _check(P.Always(P.Pred("x", ">", 0.0), si), x, P.SemanticsConfig(mode=P.LogSumExp(tau)), si, cot)
