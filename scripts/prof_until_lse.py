"""Profile target: C5-shape timed LSE Until U[0,100] (B=1024, T=10k), two eager steps."""
import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2501_04194_b200 as P
B, T = 1024, 10_000
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(B, T, device="cuda", generator=g).requires_grad_(True)
y = torch.randn(B, T, device="cuda", generator=g).requires_grad_(True)
f = P.Until(P.Pred("x", ">", 0.0), P.Pred("y", ">", 0.0), P.StepInterval(0, 100))
for _ in range(2):
    out = P.trace(f, {"x": x, "y": y}, P.SemanticsConfig(mode=P.LogSumExp(10.0)))
    out.backward(torch.ones_like(out))
torch.cuda.synchronize()
print("ok")
