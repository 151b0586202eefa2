"""The reference's phi1..phi6 benchmark at GPU scale (reference
bench.py:32-154, PAPER Table III).

Formulas (restated from the reference's `bench_formulas`): box leaves
`lo < c < lo + 1` with lo = -0.5 - 0.1 level over channels x, y ~ N(0, 1); windows
[0, 5]:
  phi1 Always(pair0)                 phi2 Eventually(Always(pair0))
  phi3 Until(leaf0(x), leaf0(y))     phi4 four nested sequenced visits (depth 3)
  phi5 visit then stabilise (depth 2) phi6 ten regions in any order (depth 0)
Per (formula, T, B): the device forward in Hard mode and forward + robustness-mode
gradient (d rho[:, 0] / d signals) in LogSumExp(10) — the reference's `run_bench`
measurements (bench.py:87-100) — as medians of CUDA-event timings, plus the oracle port
(numpy f64, the reference algorithm) on the host at the reference's own sizes.

    python scripts/phi_bench.py [--quick]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np
import torch

import paper_2501_04194_b200 as P

W = P.StepInterval(0, 5)


def leaf(level, ch):
    lo = -0.5 - 0.1 * level
    return P.And(P.Pred(ch, ">", lo), P.Pred(ch, "<", lo + 1.0))


def pair(level):
    return P.And(leaf(level, "x"), leaf(level, "y"))


def formulas():
    phi4 = P.Eventually(pair(0), W)
    for lvl in (1, 2, 3):
        phi4 = P.Eventually(P.And(pair(lvl), phi4), W)
    phi5 = P.Eventually(P.And(pair(2), P.Eventually(P.Always(pair(0), W), W)), W)
    phi6 = P.Eventually(pair(0), W)
    for lvl in range(1, 10):
        phi6 = P.And(P.Eventually(pair(lvl), W), phi6)
    return {"phi1": P.Always(pair(0)), "phi2": P.Eventually(P.Always(pair(0))),
            "phi3": P.Until(leaf(0, "x"), leaf(0, "y")), "phi4": phi4, "phi5": phi5, "phi6": phi6}


def device_ms(f, B, T, mode, grad, reps):
    g = torch.Generator(device="cuda").manual_seed(B * 7 + T)
    x = torch.randn(B, T, device="cuda", generator=g)
    y = torch.randn(B, T, device="cuda", generator=g)
    cfg = P.SemanticsConfig(mode=mode)

    def step():
        xs = x.requires_grad_(grad)
        ys = y.requires_grad_(grad)
        out = P.trace(f, {"x": xs, "y": ys}, cfg)
        if grad:
            torch.autograd.grad(out[:, 0].sum(), [xs, ys], allow_unused=True)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def oracle_ms(f, B, T, mode, grad, reps=3):
    import stl_oracle
    rng = np.random.default_rng(0)
    data = {"x": rng.normal(0, 1, (B, T)), "y": rng.normal(0, 1, (B, T))}
    cfg = P.SemanticsConfig(mode=mode)
    cot = np.zeros((B, T))
    cot[:, 0] = 1.0
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        if grad:
            stl_oracle.trace_and_grad(f, data, cfg, cot)
        else:
            stl_oracle.trace(f, data, cfg)
        ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    fs = formulas()
    shapes = [(8, 512, True), (1024, 10_000, False)] if not a.quick else [(8, 512, True)]
    for name, f in fs.items():
        for B, T, with_oracle in shapes:
            if name == "phi3" and T > 4000 and not a.quick:
                T = 4000  # untimed LSE Until is O(T^2) per signal
            for mname, mode, grad in (("hard_fwd", P.Hard(), False), ("lse10_fwd_grad", P.LogSumExp(10.0), True)):
                line = {"formula": name, "B": B, "T": T, "measure": mname,
                        "device_ms": round(device_ms(f, B, T, mode, grad, 7), 4)}
                if with_oracle:
                    line["oracle_cpu_ms"] = round(oracle_ms(f, B, T, mode, grad), 2)
                    line["speedup"] = round(line["oracle_cpu_ms"] / line["device_ms"], 1)
                print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
