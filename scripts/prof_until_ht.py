"""Profile target: C5 hard U[0,100] at B=4096, T=10k (csrc/until_ht.cu), a few eager steps."""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
import paper_2501_04194_b200 as P
B, T = 4096, 10_000
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(B, T, device="cuda", generator=g).requires_grad_(True)
y = torch.randn(B, T, device="cuda", generator=g).requires_grad_(True)
f = P.Until(P.Pred("x", ">", 0.0), P.Pred("y", ">", 0.0), P.StepInterval(0, 100))
for _ in range(3):
    out = P.trace(f, {"x": x, "y": y}, P.SemanticsConfig())
    out.backward(torch.ones_like(out))
torch.cuda.synchronize()
print("ok")
