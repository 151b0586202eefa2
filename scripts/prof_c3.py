"""Profile target: C3 (BASELINE configs[2]) hard or LSE step, B=256, T=4000, a few eager steps.

    python scripts/prof_c3.py [hard|lse10]
"""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
import paper_2501_04194_b200 as P
mode = sys.argv[1] if len(sys.argv) > 1 else "hard"
B, T = 256, 4000
g = torch.Generator(device="cuda").manual_seed(0)
ch = {k: torch.randn(B, T, device="cuda", generator=g).requires_grad_(True) for k in "xyz"}
f = P.And(P.Always(P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(0, 200))),
          P.Until(P.Pred("y", "<", 1.0), P.Pred("z", ">", 0.0)))
cfg = P.SemanticsConfig(mode=P.Hard() if mode == "hard" else P.LogSumExp(10.0))
for _ in range(4):
    out = P.trace(f, ch, cfg)
    out.backward(torch.ones_like(out))
torch.cuda.synchronize()
print("ok")
