"""Profile target: one of the paper's phi formulas (reference bench.py BENCH_FORMULAS) at
GPU scale, LSE(10) trace + gradient, a few eager steps.

    python scripts/prof_phi.py [phi6] [B] [T]
"""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
import paper_2501_04194_b200 as P
from paper_2501_04194_b200.formula import from_json, to_json

name = sys.argv[1] if len(sys.argv) > 1 else "phi6"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
T = int(sys.argv[3]) if len(sys.argv) > 3 else 10_000
sys.path.append(os.path.join(os.path.dirname(__file__), "..", "baseline", "_ref"))
import stlmask.bench as rb
f = from_json(to_json(rb.BENCH_FORMULAS[name]))
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(B, T, device="cuda", generator=g)
y = torch.randn(B, T, device="cuda", generator=g)
cfg = P.SemanticsConfig(mode=P.LogSumExp(10.0))
for _ in range(3):
    xs, ys = x.clone().requires_grad_(True), y.clone().requires_grad_(True)
    out = P.trace(f, {"x": xs, "y": ys}, cfg)
    torch.autograd.grad(out[:, 0].sum(), [xs, ys])
torch.cuda.synchronize()
print("ok")
