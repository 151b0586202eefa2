"""Hard timed Until fwd+bwd step time vs window length K (B=1024, T=10k), eager."""
import sys, time
sys.path.insert(0, "/root/repo")
import torch, paper_2501_04194_b200 as P
B, T = 1024, 10000
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(B, T, device="cuda", generator=g); y = torch.randn(B, T, device="cuda", generator=g)
for K in (101, 300, 1000):
    f = P.Until(P.Pred("x", ">", 0.0), P.Pred("y", ">", 0.0), P.StepInterval(0, K - 1))
    def step():
        xs, ys = x.clone().requires_grad_(True), y.clone().requires_grad_(True)
        out = P.trace(f, {"x": xs, "y": ys}, P.SemanticsConfig())
        out.backward(torch.ones_like(out))
    for _ in range(3): step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): step()
    e1.record(); torch.cuda.synchronize()
    print("K", K, "ms/step", e0.elapsed_time(e1) / 10)
