"""Which C2 forward tiles does the fast LSE kernel hand to the exact kernel?"""
import ctypes, os, sys
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2501_04194_b200 as P
from paper_2501_04194_b200.engine import compile_formula
B, T = 1024, 10_000
rng = np.random.default_rng(1)
p = np.asarray(rng.uniform(-1, 1, (B, 1, 2)) + np.cumsum(0.05 * rng.normal(0, 1, (B, T, 2)), 1), dtype=np.float32)
dev = torch.device("cuda", 0)
cfg = P.SemanticsConfig(mode=P.LogSumExp(10.0))
f = P.Eventually(P.NormPred(("px", "py"), "<", 0.5), P.StepInterval(10, 100))
comp = compile_formula(f, ["px", "py"], cfg)
pt = torch.tensor(p, device=dev)
fb, bb = comp.workspace_bytes(B, T)
fws = torch.zeros(fb, dtype=torch.uint8, device=dev)
out = torch.empty(B, T, device=dev)
comp.forward([pt[..., 0], pt[..., 1]], [], out, fws, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
fl = fws[: 4 * (1 + B * 3)].view(torch.int32).cpu().numpy()
print("any slow", fl[0], "slow tiles", int((fl[1:] != 0).sum()), "of", B * 3, "first", np.flatnonzero(fl[1:])[:10])
u = 0.5 - np.sqrt(p[..., 0].astype(np.float64) ** 2 + p[..., 1].astype(np.float64) ** 2)
tau2 = 10 * 1.4426950408889634
K = 91
worst = 0
for r in range(4):
    for q in range(0, T - K, K):
        blk = u[r, 10 + q:10 + q + K]
        worst = max(worst, np.abs(tau2 * (blk - blk[0])).max())
print("max |tau2 (u - c_block)| in rows 0-3:", worst)
