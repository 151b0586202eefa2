"""Table III of the paper on this box: the reference's phi1..phi6 benchmark
(reference bench.py:32-154, recurrent.py:159-198).

For each formula and signal length of the reference's own benchmark (batch 8,
L in {32, ..., 512}), three engines run the same measurement as the reference's
`run_bench` (bench.py:87-154): the robustness trace in Hard mode ("value") and the
entry-0 gradient in LogSumExp(10) ("grad"):
  * masking   — the reference's masking engine (stlmask from baseline/_ref, numpy, CPU);
  * recurrent — the reference's recurrent engine (same package, CPU);
  * b200      — this package's device engine (libstlg.so on cuda:0, CUDA-event timed,
                inputs resident, one trace call + autograd per repetition).
`relative` = masking / recurrent - 1 as in the paper's table (negative: masking faster),
plus b200 / recurrent - 1.  At GPU scale (B=1024, T=10k; phi3 at T=4k since untimed LSE
Until is O(T^2) per signal) only the device engine runs — the reference engines would take
hours; their per-sample cost at L=512 is reported for scale.

    python scripts/phi_bench.py [--quick] [--out profiles/r2_phi_bench.jsonl]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_2501_04194_b200 as P
from paper_2501_04194_b200.formula import from_json, to_json


def reference():
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "stlmask")):
        path = "/root/reference/pkg/src"
    sys.path.append(path)
    import stlmask.bench as rb
    return rb


def device_ms(f, B, T, mode, grad, reps, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed + B * 7 + T)
    x = torch.randn(B, T, device="cuda", generator=g)
    y = torch.randn(B, T, device="cuda", generator=g)
    cfg = P.SemanticsConfig(mode=mode)

    def step():
        xs = x.detach().requires_grad_(grad)
        ys = y.detach().requires_grad_(grad)
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rb = reference()
    sizes = (32, 128, 512) if a.quick else (32, 64, 128, 256, 512)
    reps = 5 if a.quick else 11
    # the reference's own measurement (CPU, both engines)
    ref = rb.run_bench(sizes=sizes, reps=reps, batch=8, include_grad=True, seed=0)
    lines = []
    by = {(r["formula"], r["engine"], r["length"]): r for r in ref["results"]}
    for name, rf in rb.BENCH_FORMULAS.items():
        f = from_json(to_json(rf))  # the same AST in this package's classes
        for L in sizes:
            mask, rec = by[(name, "masking", L)], by[(name, "recurrent", L)]
            dv = device_ms(f, 8, L, P.Hard(), False, reps) / 1e3
            dg = device_ms(f, 8, L, P.LogSumExp(10.0), True, reps) / 1e3
            line = {"formula": name, "batch": 8, "length": L,
                    "masking_value_s": mask["value_median_s"], "recurrent_value_s": rec["value_median_s"],
                    "b200_value_s": dv,
                    "masking_grad_s": mask["grad_median_s"], "recurrent_grad_s": rec["grad_median_s"],
                    "b200_grad_s": dg,
                    "value_relative_masking_vs_recurrent": mask["value_median_s"] / rec["value_median_s"] - 1,
                    "grad_relative_masking_vs_recurrent": mask["grad_median_s"] / rec["grad_median_s"] - 1,
                    "value_relative_b200_vs_recurrent": dv / rec["value_median_s"] - 1,
                    "grad_relative_b200_vs_recurrent": dg / rec["grad_median_s"] - 1}
            lines.append(line)
            print(json.dumps(line), flush=True)
    # GPU scale: device engine only
    for name, rf in rb.BENCH_FORMULAS.items():
        f = from_json(to_json(rf))
        B, T = 1024, (4000 if name == "phi3" else 10_000)
        dv = device_ms(f, B, T, P.Hard(), False, 7)
        dg = device_ms(f, B, T, P.LogSumExp(10.0), True, 5)
        ref512 = by[(name, "masking", sizes[-1])]
        line = {"formula": name, "batch": B, "length": T, "b200_value_ms": dv, "b200_grad_ms": dg,
                "b200_value_timesteps_per_s": B * T / (dv / 1e3),
                "reference_masking_grad_s_per_timestep_at_L%d" % sizes[-1]: ref512["grad_median_s"] / (8 * sizes[-1])}
        lines.append(line)
        print(json.dumps(line), flush=True)
    if a.out:
        with open(a.out, "w") as fh:
            for ln in lines:
                fh.write(json.dumps(ln) + "\n")


if __name__ == "__main__":
    main()
