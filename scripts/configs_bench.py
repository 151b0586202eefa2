"""Forward + backward timings of every BASELINE.json config on one GPU.

One JSON line per (config, mode): trace-mode step = full trace forward + ones-cotangent
VJP into every signal channel (and d(a, b, c) for C4), CUDA events around eager calls
through the engine API (plan cached, workspace preallocated), median of `reps` after
warm-up.  Inputs per SURVEY §8(d): C1 x ~ N(0,1); C2 2-D random walks; C3 x, y, z ~
N(0,1); C4 smooth-interval bounds (0.3, 0.65, 9.0) over synth_step_dataset(seed=3)
(apps.py:252-269); C5 x, y ~ N(0,1).

    python scripts/configs_bench.py [--quick]
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
from paper_2501_04194_b200.engine import compile_formula

dev = torch.device("cuda", 0)


def timed(comp, chans, B, T, smooth=None, reps=5, warm=2):
    names = list(chans)
    xs = [chans[k] for k in names]
    fb, bb = comp.workspace_bytes(B, T)
    fws = torch.empty(max(fb, 1), dtype=torch.uint8, device=dev)
    bws = torch.empty(max(bb, 1), dtype=torch.uint8, device=dev)
    out = torch.empty(B, T, device=dev)
    ones = torch.ones(B, T, device=dev)
    grads = [torch.empty(B, T, device=dev) for _ in xs]
    params = comp.smooth_params(smooth) if smooth is not None else comp.smooth_params()
    dsm = torch.zeros(3 * max(1, len(params)), dtype=torch.float64, device=dev) if smooth is not None else None
    import ctypes

    def cur():
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def step():
        comp.forward(xs, params, out, fws, cur())
        comp.backward(xs, params, out, ones, grads, dsm, fws, bws, cur())

    for _ in range(warm):
        step()
    torch.cuda.synchronize()
    fw, bw = [], []
    for _ in range(reps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        comp.forward(xs, params, out, fws, cur())
        e[1].record()
        comp.backward(xs, params, out, ones, grads, dsm, fws, bws, cur())
        e[2].record()
        torch.cuda.synchronize()
        fw.append(e[0].elapsed_time(e[1]))
        bw.append(e[1].elapsed_time(e[2]))
    return statistics.median(fw), statistics.median(bw)


def emit(name, mode, B, T, fms, bms, **kw):
    line = {"config": name, "mode": mode, "B": B, "T": T, "fwd_ms": round(fms, 4), "bwd_ms": round(bms, 4),
            "timesteps_per_s": B * T / ((fms + bms) / 1e3)}
    line.update(kw)
    print(json.dumps(line), flush=True)


def modes_of(names):
    table = {"hard": P.Hard(), "lse10": P.LogSumExp(10.0), "lse5": P.LogSumExp(5.0), "soft10": P.SoftMax(10.0)}
    return [(n, table[n]) for n in names]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default="", help="comma-separated configs, e.g. C2,C4")
    a = ap.parse_args()

    def want(c):
        return not a.only or c in a.only.split(",")
    g = torch.Generator(device=dev).manual_seed(0)

    def randn(B, T):
        return torch.randn(B, T, device=dev, generator=g)

    # C1: Always[0,50](x > 0.5), Hard (reference CPU case) and the same formula at B=1024, T=10k
    f1 = P.Always(P.Pred("x", ">", 0.5), P.StepInterval(0, 50))
    for B, T in ((1, 1000), (1024, 10_000)) if want("C1") else ():
        comp = compile_formula(f1, ["x"], P.SemanticsConfig(mode=P.Hard()))
        fm, bm = timed(comp, {"x": randn(B, T)}, B, T)
        emit("C1", "hard", B, T, fm, bm, alg_bytes_per_unit=16)

    # C2: Eventually[10,100](||p - g|| < 0.5), 2-D random walks, B=1024, T=10k
    B, T = 1024, 10_000
    rng = np.random.default_rng(1)
    p = torch.tensor(np.asarray(rng.uniform(-1, 1, (B, 1, 2)) + np.cumsum(0.05 * rng.normal(0, 1, (B, T, 2)), 1),
                                dtype=np.float32), device=dev)
    f2 = P.Eventually(P.NormPred(("px", "py"), "<", 0.5), P.StepInterval(10, 100))
    for mname, m in modes_of(["lse10", "hard", "soft10"] if want("C2") else []):
        comp = compile_formula(f2, ["px", "py"], P.SemanticsConfig(mode=m))
        fm, bm = timed(comp, {"px": p[..., 0], "py": p[..., 1]}, B, T)
        emit("C2", mname, B, T, fm, bm, alg_bytes_per_unit=24)

    # C3: And(Always(Eventually[0,200](x > 0)), Until(y < 1, z > 0)), untimed Always / Until
    B, T = 256, 4000
    f3 = P.And(P.Always(P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(0, 200))),
               P.Until(P.Pred("y", "<", 1.0), P.Pred("z", ">", 0.0)))
    c3 = {"x": randn(B, T), "y": randn(B, T), "z": randn(B, T)}
    for mname, m in modes_of(["hard", "lse10"] if want("C3") else []):
        comp = compile_formula(f3, ["x", "y", "z"], P.SemanticsConfig(mode=m))
        fm, bm = timed(comp, c3, B, T, reps=3 if mname != "hard" else 5)
        emit("C3", mname, B, T, fm, bm)

    # C4: Always(x > 0, SmoothInterval(0.3, 0.65, 9)), LSE(5), B=4096, T=2k, grads to x and (a, b, c)
    B, T = 4096, 2000
    si = P.SmoothInterval(0.3, 0.65, 9.0)
    f4 = P.Always(P.Pred("x", ">", 0.0), si)
    comp = compile_formula(f4, ["x"], P.SemanticsConfig(mode=P.LogSumExp(5.0)))
    x4 = torch.tensor(np.asarray(P.synth_step_dataset(3, B, T), dtype=np.float32), device=dev)
    if want("C4"):
        fm, bm = timed(comp, {"x": x4}, B, T, smooth=(si.a, si.b, si.c), reps=3)
        emit("C4", "lse5", B, T, fm, bm, grads="x and (a, b, c)")

    # C5: long-horizon sweep (subset): F[0,100], untimed F, U[0,100], untimed U; Hard / LSE(10)
    Ts = ((1_000, 10_000, 100_000) if not a.quick else (10_000,)) if want("C5") else ()
    for T in Ts:
        B = min(16384, int(1.6e9 // (2 * T)), 4096)
        xs = {"x": randn(B, T), "y": randn(B, T)}
        ops = [("F[0,100]", P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(0, 100)), ["x"]),
               ("F", P.Eventually(P.Pred("x", ">", 0.0)), ["x"]),
               ("U[0,100]", P.Until(P.Pred("x", ">", 0.0), P.Pred("y", ">", 0.0), P.StepInterval(0, 100)), ["x", "y"]),
               ("U", P.Until(P.Pred("x", ">", 0.0), P.Pred("y", ">", 0.0)), ["x", "y"])]
        for oname, f, names in ops:
            for mname, m in modes_of(["hard", "lse10"]):
                if oname == "U" and mname != "hard" and B * T * T > 1e12:
                    continue  # O(T^2) per signal (SURVEY §8(d) C5 skip rule)
                comp = compile_formula(f, names, P.SemanticsConfig(mode=m))
                fm, bm = timed(comp, {k: xs[k] for k in names}, B, T, reps=3)
                emit("C5", mname, B, T, fm, bm, op=oname)


if __name__ == "__main__":
    main()
