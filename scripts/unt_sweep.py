"""Untimed scans (F / G hard + LSE, hard Until) across batch sizes: the multi-CTA look-back
kernels (fg_unt.cu, until.cu) against small-batch long-horizon and large-batch shapes.

    python scripts/unt_sweep.py            # one JSON line per (op, mode, B, T)
"""
import json, os, statistics, sys
sys.path.insert(0, os.environ.get("STLG_ROOT", os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))))
import torch
import paper_2501_04194_b200 as P
from paper_2501_04194_b200.engine import compile_formula
import ctypes

dev = torch.device("cuda", 0)


def run(f, names, mode, B, T, reps=5):
    comp = compile_formula(f, names, P.SemanticsConfig(mode=mode))
    g = torch.Generator(device="cuda").manual_seed(B + T)
    xs = [torch.randn(B, T, device=dev, generator=g) for _ in names]
    fb, bb = comp.workspace_bytes(B, T)
    fws = torch.empty(max(fb, 1), dtype=torch.uint8, device=dev)
    bws = torch.empty(max(bb, 1), dtype=torch.uint8, device=dev)
    out = torch.empty(B, T, device=dev)
    ones = torch.ones(B, T, device=dev)
    grads = [torch.empty(B, T, device=dev) for _ in xs]
    params = comp.smooth_params()
    st = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(2):
        comp.forward(xs, params, out, fws, st())
        comp.backward(xs, params, out, ones, grads, None, fws, bws, st())
    torch.cuda.synchronize()
    fw, bw = [], []
    for _ in range(reps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        comp.forward(xs, params, out, fws, st())
        e[1].record()
        comp.backward(xs, params, out, ones, grads, None, fws, bws, st())
        e[2].record()
        torch.cuda.synchronize()
        fw.append(e[0].elapsed_time(e[1]))
        bw.append(e[1].elapsed_time(e[2]))
    return statistics.median(fw), statistics.median(bw)


ops = [("F", lambda: P.Eventually(P.Pred("x", ">", 0.0)), ["x"], ["hard", "lse10"]),
       ("U", lambda: P.Until(P.Pred("x", ">", 0.0), P.Pred("y", ">", 0.0)), ["x", "y"], ["hard"])]
modes = {"hard": P.Hard(), "lse10": P.LogSumExp(10.0)}
for B, T in ((64, 100_000), (16, 1_000_000), (256, 4_000), (4096, 10_000)):
    for oname, mk, names, ms in ops:
        for m in ms:
            fm, bm = run(mk(), names, modes[m], B, T)
            print(json.dumps({"op": oname, "mode": m, "B": B, "T": T, "fwd_ms": round(fm, 4), "bwd_ms": round(bm, 4)}), flush=True)
