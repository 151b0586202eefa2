"""Generate golden vectors from the REFERENCE implementation (dev container only).

Run from the repo root in a container that mounts the reference:

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests python tests/golden/make_golden.py

It imports ``stlmask`` (the reference, /root/reference/pkg/src) and writes
``tests/golden/*.npz``.  Every case stores: the formula (JSON, see
``paper_2501_04194_b200.formula.to_json``), the config, the float32-
representable inputs (as float64), the reference's full robustness trace
(``masking.trace_var``, masking.py:308) and the reference's reverse-mode
gradients (``tape.backward``, tape.py:114) for a given cotangent, plus
d_a/d_b/d_c for smooth-interval bindings (``autodiff.value_and_grad``,
autodiff.py:64).  Nothing at test time reads /root/reference: the fixtures
travel, the reference does not.

Corpus sources:
  * KATs lifted from the reference tests (test_masking.py:100-175, 322-328,
    test_autodiff.py:38-67, test_acceptance.py:42-53);
  * random formulas from the reference's own generator
    (tests/helpers.py:16-71), with fp32-representable thresholds/signals;
  * smooth-interval cases (test_autodiff.py:101-119 setup);
  * NormPred cases built on the reference tape as sqrt(dx^2 + dy^2).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import stlmask  # noqa: E402  (reference)
from stlmask import masking, tape  # noqa: E402
from stlmask.autodiff import value_and_grad as ref_vag  # noqa: E402
from stlmask.core import (Hard, LogSumExp, NamedSignals, PaddingPolicy,  # noqa: E402
                          SemanticsConfig, SmoothInterval, SoftMax, StepInterval)
from stlmask.formula import (TRUE, Always, And, Eventually, Not, Or, Pred,  # noqa: E402
                             Until)

from paper_2501_04194_b200.formula import to_json  # noqa: E402

import helpers  # noqa: E402  (reference tests/helpers.py)


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def cfg_json(cfg):
    m = type(cfg.mode).__name__
    return json.dumps({"mode": m, "temp": getattr(cfg.mode, "temp", None),
                       "pad": cfg.padding.kind, "pad_value": cfg.padding.value,
                       "sentinel": cfg.sentinel, "top_value": cfg.top_value,
                       "masked_fill": cfg.masked_fill})


def f32_formula(rng, f):
    """Round thresholds to float32 so device and oracle see the same constants."""
    k = type(f).__name__
    if k == "Pred":
        return Pred(f.var, f.cmp, float(np.float32(f.threshold)))
    if k == "Not":
        return Not(f32_formula(rng, f.arg))
    if k in ("And", "Or"):
        return type(f)(f32_formula(rng, f.left), f32_formula(rng, f.right))
    if k in ("Eventually", "Always"):
        return type(f)(f32_formula(rng, f.arg), f.interval)
    if k == "Until":
        return Until(f32_formula(rng, f.left), f32_formula(rng, f.right), f.interval)
    return f


def run_ref(f, arrays, cfg, cot, norm=None):
    """Reference trace + VJP for batched arrays (B, L).  norm=(x, y, cx, cy, dname)."""
    chans = {k: tape.Var(v) for k, v in arrays.items()}
    feed = dict(chans)
    if norm is not None:
        xn, yn, cx, cy, dname = norm
        dx = chans[xn] - cx
        dy = chans[yn] - cy
        feed[dname] = tape.sqrt(tape.square(dx) + tape.square(dy))
    L = next(iter(arrays.values())).shape[-1]
    out = masking.trace_var(f, feed, L, cfg)
    tape.backward(out, cot)
    grads = {k: (v.grad if v.grad is not None else np.zeros_like(v.data)) for k, v in chans.items()}
    return out.data.copy(), grads


class Sink:
    def __init__(self):
        self.cases = []

    def add(self, name, f, arrays, cfg, cot, trace, grads, dabc=None, si=None, norm=None,
            formula_json=None):
        self.cases.append(dict(
            name=name, formula=formula_json or to_json(f), cfg=cfg_json(cfg),
            arrays={k: np.asarray(v, dtype=np.float64) for k, v in arrays.items()},
            cot=np.asarray(cot, dtype=np.float64), trace=np.asarray(trace, dtype=np.float64),
            grads={k: np.asarray(v, dtype=np.float64) for k, v in grads.items()},
            dabc=None if dabc is None else np.asarray(dabc, dtype=np.float64),
            si=None if si is None else np.asarray([si.a, si.b, si.c, si.eps])))

    def save(self, path):
        blob = {}
        meta = []
        for i, c in enumerate(self.cases):
            p = f"c{i}_"
            m = {"name": c["name"], "formula": c["formula"], "cfg": c["cfg"],
                 "channels": list(c["arrays"]), "has_dabc": c["dabc"] is not None,
                 "has_si": c["si"] is not None}
            meta.append(m)
            for k, v in c["arrays"].items():
                blob[p + "x_" + k] = v
            for k, v in c["grads"].items():
                blob[p + "g_" + k] = v
            blob[p + "cot"] = c["cot"]
            blob[p + "trace"] = c["trace"]
            if c["dabc"] is not None:
                blob[p + "dabc"] = c["dabc"]
            if c["si"] is not None:
                blob[p + "si"] = c["si"]
        blob["meta"] = np.array(json.dumps(meta))
        np.savez_compressed(path, **blob)
        print(f"wrote {path}: {len(self.cases)} cases")


def kats(sink):
    s8 = {"s": np.arange(8.0)[None, :]}
    last = SemanticsConfig()
    const_neg = SemanticsConfig(padding=PaddingPolicy.constant(-1e5))
    fill = SemanticsConfig(padding=PaddingPolicy.constant(-1e5), masked_fill=True)
    F13 = Eventually(Pred("s", ">", 0.0), StepInterval(1, 3))
    G13 = Always(Pred("s", ">", 0.0), StepInterval(1, 3))
    for nm, f, cfg in [("ex1_last", F13, last), ("ex1_const", F13, const_neg),
                       ("G13_last", G13, last), ("ex1_fill", F13, fill),
                       ("ex1_lse", F13, SemanticsConfig(mode=LogSumExp(5.0))),
                       ("ex1_soft", F13, SemanticsConfig(mode=SoftMax(2.0)))]:
        cot = np.ones((1, 8))
        tr, g = run_ref(f, s8, cfg, cot)
        sink.add(nm, f, s8, cfg, cot, tr, g)
    for nm, vals, f in [("untimed_F", [2.0, 9.0, 4.0], Eventually(Pred("s", ">", 0.0))),
                        ("untimed_G", [2.0, 9.0, 4.0], Always(Pred("s", ">", 0.0))),
                        ("tie_F", [1.0, 3.0, 3.0], Eventually(Pred("s", ">", 0.0))),
                        ("argmax_F", [1.0, 3.0, 2.0], Eventually(Pred("s", ">", 0.0))),
                        ("single", [5.0], Always(Pred("s", ">", 0.0))),
                        ("neg_pred", [0.0, 2.0], Not(Pred("s", ">", 1.0))),
                        ("true", [0.0, 1.0, 2.0], TRUE),
                        ("zeros_F", [0.0, -0.0, 0.0, -0.0, 1.0, -0.0, 0.0],
                         Eventually(Pred("s", ">", 0.0), StepInterval(0, 2))),
                        ("zeros_Funt", [0.0, -0.0, 0.0, -0.0, -1.0, -0.0, 0.0],
                         Eventually(Pred("s", ">", 0.0))),
                        ("zeros_and", [0.0, -0.0, 0.0, -0.0], And(Pred("s", ">", 0.0),
                                                                  Not(Pred("s", "<", 0.0)))),
                        ("past_end", [1.0, 2.0], Eventually(Pred("s", ">", 0.0), StepInterval(5, 6)))]:
        arrs = {"s": np.asarray(vals, dtype=np.float64)[None, :]}
        for cfg in (last, SemanticsConfig(padding=PaddingPolicy.constant(-3.0)),
                    SemanticsConfig(mode=LogSumExp(5.0))):
            cot = np.ones_like(arrs["s"])
            tr, g = run_ref(f, arrs, cfg, cot)
            sink.add(nm, f, arrs, cfg, cot, tr, g)
    # until KATs (test_masking.py:159-175) and tie routing
    for nm, l, r, iv in [("until_kat", [1, 1, -1], [-1, 1, 1], None),
                         ("until_tie", [3, 1, 2, 5], [0, 4, 1, 2], StepInterval(1, 2)),
                         ("until_tie_unt", [3, 1, 2, 5, 1, 1], [0, 4, 1, 2, 1, 0], None),
                         ("until_00", [0.5, -1.0, 2.0, 0.25], [1.0, 0.0, -2.0, 3.0], StepInterval(0, 0))]:
        arrs = {"l": np.asarray(l, float)[None, :], "r": np.asarray(r, float)[None, :]}
        f = Until(Pred("l", ">", 0.0), Pred("r", ">", 0.0), iv)
        for cfg in (last, SemanticsConfig(mode=LogSumExp(2.0)), SemanticsConfig(mode=SoftMax(1.5))):
            cot = np.ones_like(arrs["l"])
            tr, g = run_ref(f, arrs, cfg, cot)
            sink.add(nm, f, arrs, cfg, cot, tr, g)


def random_corpus(sink, seed, n, modes, max_len=40, batch=2, fill_frac=0.0):
    rng = np.random.default_rng(seed)
    made = 0
    while made < n:
        f, _sig = helpers.equivalence_case(rng, depth=3, max_len=max_len)
        f = f32_formula(rng, f)
        L = int(rng.integers(1, max_len + 1))
        arrays = {c: f32(rng.normal(0, 2, (batch, L))) for c in helpers.CHANNELS}
        mode = modes[made % len(modes)]
        pad = helpers.random_padding(rng)
        if pad.kind == "const":
            pad = PaddingPolicy.constant(float(np.float32(pad.value)))
        cfg = SemanticsConfig(mode=mode, padding=pad, top_value=100.0,
                              masked_fill=bool(rng.random() < fill_frac))
        cot = f32(rng.normal(0, 1, (batch, L))) if made % 3 == 2 else np.ones((batch, L))
        try:
            tr, g = run_ref(f, arrays, cfg, cot)
        except stlmask.EmptyWindowError:
            continue
        sink.add(f"rand{seed}_{made}", f, arrays, cfg, cot, tr, g)
        made += 1


def smooth_cases(sink):
    rng = np.random.default_rng(53)
    for i in range(24):
        L = int(rng.integers(2, 40))
        arrays = {"x": f32(rng.normal(0, 1, (1, L))), "y": f32(rng.normal(0, 1, (1, L)))}
        a = float(np.float32(rng.uniform(0.05, 0.5)))
        si = SmoothInterval(a, float(np.float32(rng.uniform(a + 0.1, 1.0))),
                            float(np.float32(rng.uniform(2.0, 30.0))))
        node = Always if i % 2 == 0 else Eventually
        inner = [Pred("x", ">", 0.0), And(Pred("x", ">", -0.25), Pred("y", "<", 0.5)),
                 Eventually(Pred("y", ">", 0.0), StepInterval(0, 2))][i % 3]
        f = node(inner, si)
        mode = [Hard(), LogSumExp(5.0), SoftMax(2.0)][i % 3]
        pad = PaddingPolicy.last_value() if i % 4 < 2 else PaddingPolicy.constant(-0.5)
        cfg = SemanticsConfig(mode=mode, padding=pad, top_value=100.0)
        # full-trace VJP, interval fixed (no binding)
        cot = np.ones((1, L))
        tr, g = run_ref(f, arrays, cfg, cot)
        sink.add(f"smooth_trace_{i}", f, arrays, cfg, cot, tr, g)
        # value_and_grad with binding: entry-0 cotangent + d_a, d_b, d_c
        sig = NamedSignals.from_arrays({k: v[0] for k, v in arrays.items()})
        res = ref_vag(f, sig, cfg)
        cot0 = np.zeros((1, L))
        cot0[0, 0] = 1.0
        trv = masking.robustness_trace(f, sig, cfg)[None, :]
        grads = {k: res.d_signal[k][None, :] for k in arrays}
        dabc = [res.d_a, res.d_b, res.d_c] if res.d_a is not None else None
        sink.add(f"smooth_vag_{i}", f, arrays, cfg, cot0, trv, grads, dabc=dabc, si=si)


def c4_like(sink):
    """The C4 operator at small size (test_autodiff.py:15,103 parameters)."""
    from stlmask.apps import synth_step_dataset
    data = f32(synth_step_dataset(3, n=4, length=60))
    si = SmoothInterval(0.3, 0.65, 9.0)
    f = Always(Pred("x", ">", 0.0), si)
    cfg = SemanticsConfig(mode=LogSumExp(5.0))
    arrays = {"x": data}
    # full trace + ones cotangent, with the (a, b, c) binding so d_abc is recorded
    chans = {"x": tape.Var(data)}
    params = (tape.Var(si.a), tape.Var(si.b), tape.Var(si.c))
    out = masking.trace_var(f, chans, data.shape[-1], cfg, smooth_binding=params)
    cot = np.ones_like(data)
    tape.backward(out, cot)
    sink.add("c4_small", f, arrays, cfg, cot, out.data.copy(), {"x": chans["x"].grad},
             dabc=[float(p.grad) for p in params], si=si)


def norm_cases(sink):
    rng = np.random.default_rng(11)
    from paper_2501_04194_b200.formula import NormPred, Eventually as BEv
    from paper_2501_04194_b200.core import StepInterval as BSI
    for i in range(6):
        L = int(rng.integers(20, 80))
        p0 = rng.uniform(-1, 1, (2, 2))
        steps = 0.05 * rng.normal(0, 1, (2, L, 2))
        p = f32(p0[:, None, :] + np.cumsum(steps, axis=1))
        arrays = {"px": p[..., 0], "py": p[..., 1]}
        a, b = [(10, 30), (0, 5), (3, 3)][i % 3]
        mode = [LogSumExp(10.0), Hard(), SoftMax(3.0)][i % 3]
        cfg = SemanticsConfig(mode=mode)
        f_ref = Eventually(Pred("d", "<", 0.5), StepInterval(a, b))
        cot = np.ones((2, L))
        tr, g = run_ref(f_ref, arrays, cfg, cot, norm=("px", "py", 0.0, 0.0, "d"))
        f_b200 = BEv(NormPred(("px", "py"), "<", 0.5, (0.0, 0.0)), BSI(a, b))
        sink.add(f"norm_{i}", f_b200, arrays, cfg, cot, tr, g, formula_json=to_json(f_b200))


def main():
    out = HERE
    s = Sink()
    kats(s)
    s.save(os.path.join(out, "kats.npz"))
    s = Sink()
    random_corpus(s, 2024, 160, [Hard(), LogSumExp(1.0), LogSumExp(5.0), LogSumExp(20.0)])
    random_corpus(s, 2025, 60, [SoftMax(2.0), Hard()], max_len=20)
    random_corpus(s, 2026, 40, [Hard(), LogSumExp(5.0)], max_len=16, fill_frac=1.0)
    s.save(os.path.join(out, "random.npz"))
    s = Sink()
    smooth_cases(s)
    c4_like(s)
    norm_cases(s)
    s.save(os.path.join(out, "smooth_norm.npz"))


if __name__ == "__main__":
    main()
