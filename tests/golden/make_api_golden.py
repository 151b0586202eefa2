"""Golden vectors for the reference-facing API wrappers (dev container only).

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests python tests/golden/make_api_golden.py

Imports the REFERENCE (``stlmask``) and records, into ``tests/golden/api.npz``:

* ``eventually_trace`` / ``always_trace`` / ``until_trace`` (masking.py:377-401) on the
  reference's own KATs (tests/test_masking.py:100-175) and on the random cases of
  ``test_matches_materialized_mask_reduction`` / ``test_matches_materialized_3d_reduction``
  (test_masking.py:130-155, 181-221; same generators, inputs rounded to float32), plus
  smooth-interval windows;
* ``value_and_grad`` (autodiff.py:64-107) on the reference's KATs (test_autodiff.py:38-67),
  random LSE formulas from its corpus generator (tests/helpers.py:16-51) with an unused
  channel, the interval-gradient setup (test_autodiff.py:101-119) with ``si=`` rebinding
  (including a non-zero eps), and the "binding overrides all nodes" case
  (test_autodiff.py:160-165).

Nothing at test time reads /root/reference; the fixture travels, the reference does not.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from stlmask import masking  # noqa: E402  (reference)
from stlmask.autodiff import value_and_grad as ref_vag  # noqa: E402
from stlmask.core import (Hard, LogSumExp, NamedSignals, PaddingPolicy,  # noqa: E402
                          SemanticsConfig, SmoothInterval, SoftMax, StepInterval)
from stlmask.formula import Always, And, Eventually, Not, Pred, parse  # noqa: E402

from paper_2501_04194_b200.formula import to_json  # noqa: E402

import helpers  # noqa: E402  (reference tests/helpers.py)
from make_golden import cfg_json, f32, f32_formula  # noqa: E402


def iv_json(iv):
    if iv is None:
        return None
    if type(iv).__name__ == "StepInterval":
        return {"step": [iv.a, iv.b]}
    return {"smooth": [iv.a, iv.b, iv.c, iv.eps]}


class Sink:
    def __init__(self):
        self.meta = []
        self.blob = {}

    def add(self, meta, **arrays):
        i = len(self.meta)
        meta = dict(meta, arrays=sorted(arrays))
        self.meta.append(meta)
        for k, v in arrays.items():
            self.blob[f"c{i}_{k}"] = np.asarray(v, dtype=np.float64)

    def save(self, path):
        np.savez_compressed(path, meta=np.array(json.dumps(self.meta)), **self.blob)


LAST = SemanticsConfig()
CONST_NEG = SemanticsConfig(padding=PaddingPolicy.constant(-1e5))


def wrappers(s):
    # KATs (test_masking.py:100-175)
    kats = [("F", np.arange(8.0), StepInterval(1, 3), LAST),
            ("F", np.arange(8.0), StepInterval(1, 3), CONST_NEG),
            ("F", [2.0, 9.0, 4.0], None, LAST),
            ("G", np.arange(8.0), StepInterval(1, 3), LAST),
            ("G", [2.0, 9.0, 4.0], None, LAST),
            ("G", [5.0], None, LAST),
            ("F", [1.0, 2.0], StepInterval(5, 6), SemanticsConfig(padding=PaddingPolicy.constant(-3.0)))]
    for kind, vals, iv, cfg in kats:
        x = f32(vals)
        fn = masking.eventually_trace if kind == "F" else masking.always_trace
        s.add({"op": kind, "iv": iv_json(iv), "cfg": cfg_json(cfg), "src": "kat"}, x=x, out=fn(x, iv, cfg))
    # random windows (test_masking.py:130-155 generator)
    rng = np.random.default_rng(31)
    for i in range(40):
        length = int(rng.integers(1, 15))
        inner = f32(rng.normal(0, 2, length))
        a = int(rng.integers(0, 5))
        iv = StepInterval(a, a + int(rng.integers(0, 5)))
        mode = [Hard(), LogSumExp(3.0), SoftMax(2.0)][int(rng.integers(0, 3))]
        pad = PaddingPolicy.constant(float(np.float32(rng.normal()))) if rng.random() < 0.5 \
            else PaddingPolicy.last_value()
        cfg = SemanticsConfig(mode=mode, padding=pad)
        kind = "F" if i % 2 == 0 else "G"
        fn = masking.eventually_trace if kind == "F" else masking.always_trace
        s.add({"op": kind, "iv": iv_json(iv), "cfg": cfg_json(cfg), "src": "rand31"},
              x=inner, out=fn(inner, iv, cfg))
    # smooth-interval and untimed windows through the wrappers
    rng = np.random.default_rng(35)
    for i in range(12):
        length = int(rng.integers(2, 40))
        inner = f32(rng.normal(0, 1, length))
        if i % 3 == 2:
            iv = None
        else:
            a = float(np.float32(rng.uniform(0.05, 0.5)))
            iv = SmoothInterval(a, float(np.float32(rng.uniform(a + 0.1, 1.0))),
                                float(np.float32(rng.uniform(2.0, 30.0))))
        mode = [Hard(), LogSumExp(5.0), SoftMax(2.0)][i % 3] if iv is not None else \
            [Hard(), LogSumExp(5.0)][i % 2]
        cfg = SemanticsConfig(mode=mode)
        kind = "F" if i % 2 == 0 else "G"
        fn = masking.eventually_trace if kind == "F" else masking.always_trace
        s.add({"op": kind, "iv": iv_json(iv), "cfg": cfg_json(cfg), "src": "smooth35"},
              x=inner, out=fn(inner, iv, cfg))
    # Until KATs (test_masking.py:159-175)
    rng = np.random.default_rng(32)
    right = f32(rng.normal(0, 2, 12))
    top = np.full(12, 1e5)
    cfg_top = SemanticsConfig(padding=PaddingPolicy.constant(1e5))
    left9 = f32(np.random.default_rng(33).normal(0, 1, 9))
    for l_, r_, iv, cfg in [(f32([1, 1, -1]), f32([-1, 1, 1]), None, LAST),
                            (top, right, None, cfg_top),
                            (left9, left9, StepInterval(0, 0), LAST)]:
        s.add({"op": "U", "iv": iv_json(iv), "cfg": cfg_json(cfg), "src": "kat"},
              l=l_, r=r_, out=masking.until_trace(l_, r_, iv, cfg))
    # random Until (test_masking.py:181-200 generator)
    rng = np.random.default_rng(34)
    for _ in range(30):
        length = int(rng.integers(1, 12))
        left = f32(rng.normal(0, 2, length))
        right = f32(rng.normal(0, 2, length))
        use_iv = rng.random() < 0.7
        a = int(rng.integers(0, 4))
        iv = StepInterval(a, a + int(rng.integers(0, 4))) if use_iv else None
        mode = [Hard(), LogSumExp(2.0), SoftMax(1.5)][int(rng.integers(0, 3))]
        pad = PaddingPolicy.constant(float(np.float32(rng.normal()))) if rng.random() < 0.5 \
            else PaddingPolicy.last_value()
        cfg = SemanticsConfig(mode=mode, padding=pad)
        s.add({"op": "U", "iv": iv_json(iv), "cfg": cfg_json(cfg), "src": "rand34"},
              l=left, r=right, out=masking.until_trace(left, right, iv, cfg))


def _vag(s, f, arrays, cfg, si=None, src=""):
    sig = NamedSignals.from_arrays(arrays)
    res = ref_vag(f, sig, cfg, si=si)
    out = {"x_" + k: v for k, v in arrays.items()}
    out.update({"g_" + k: res.d_signal[k] for k in arrays})
    out["value"] = [res.value]
    if res.d_a is not None:
        out["dabc"] = [res.d_a, res.d_b, res.d_c]
    s.add({"formula": to_json(f), "cfg": cfg_json(cfg), "si": iv_json(si), "channels": list(arrays),
           "src": src}, **out)


def vag(s):
    LSE5 = SemanticsConfig(mode=LogSumExp(5.0))
    # KATs (test_autodiff.py:38-67)
    _vag(s, parse("F (s > 0)"), {"s": f32([1.0, 3.0, 2.0])}, LAST, src="kat_onehot")
    _vag(s, parse("F (s > 0)"), {"s": f32([1.0, 3.0, 3.0])}, LAST, src="kat_tie")
    rng = np.random.default_rng(50)
    for _ in range(4):
        _vag(s, parse("G (s > 0)"), {"s": f32(rng.normal(0, 1, 9))}, LAST, src="kat_min")
    _vag(s, parse("G (s > 0)"), {"s": f32([0.5, -0.2, 0.9, 0.1])}, LSE5, src="kat_softmin")
    _vag(s, parse("F (s > 0)"), {"s": f32([1.0, 2.0]), "unused": f32([5.0, 5.0])}, LAST,
         src="kat_unused")
    # random LSE formulas (test_autodiff.py:81-99 generator), one unused channel
    rng = np.random.default_rng(52)
    for case in range(24):
        length = int(rng.integers(3, 15))
        arrays = {"x": f32(rng.normal(0, 1.5, length)), "y": f32(rng.normal(0, 1.5, length)),
                  "z": f32(rng.normal(0, 1.5, length))}
        f = f32_formula(rng, helpers.random_formula(rng, 2))
        tau = float(rng.choice([1.0, 5.0, 20.0]))
        mode = LogSumExp(tau) if case % 4 else Hard()
        cfg = SemanticsConfig(mode=mode, padding=PaddingPolicy.last_value(), top_value=100.0)
        _vag(s, f, arrays, cfg, src="rand52")
    # interval gradients + si= rebinding (test_autodiff.py:101-119)
    rng = np.random.default_rng(53)
    si = SmoothInterval(0.3, 0.65, 9.0)
    for i in range(6):
        arrays = {"x": f32(rng.normal(0, 1, 14)), "y": f32(rng.normal(0, 1, 14))}
        f = And(Always(Pred("x", ">", 0.0), si), Eventually(Pred("y", ">", -0.5)))
        _vag(s, f, arrays, LSE5, src="itv")
        rb = [SmoothInterval(0.25, 0.6, 9.0), SmoothInterval(0.3, 0.7, 12.0),
              SmoothInterval(0.2, 0.8, 4.0, 0.05)][i % 3]
        _vag(s, f, arrays, LSE5, si=rb, src="itv_rebind")
        _vag(s, Not(f), arrays, SemanticsConfig(mode=SoftMax(2.0)), si=rb, src="itv_rebind_soft")
    # binding overrides all nodes (test_autodiff.py:160-165), on a non-constant signal
    f2 = And(Always(Pred("s", ">", 0.0), SmoothInterval(0.1, 0.5, 4.0)),
             Eventually(Pred("s", ">", 0.0), SmoothInterval(0.2, 0.9, 4.0)))
    _vag(s, f2, {"s": f32(np.random.default_rng(54).normal(0, 1, 8))}, LSE5,
         si=SmoothInterval(0.3, 0.7, 6.0), src="override")
    # sharp mask (test_autodiff.py:121-131)
    vals = np.ones(20)
    vals[8] = 0.1
    _vag(s, Always(Pred("s", ">", 0.0), SmoothInterval(0.2, 0.7, 1e3)), {"s": f32(vals)},
         SemanticsConfig(mode=LogSumExp(20.0)), src="sharp")


def main():
    s = Sink()
    wrappers(s)
    vag(s)
    s.save(os.path.join(HERE, "api.npz"))
    print(len(s.meta), "cases")


if __name__ == "__main__":
    main()
