"""Small driver for ncu: a few C2 fwd+bwd steps at full size (B=1024, T=10k)."""
import ctypes
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_2501_04194_b200 as P
from paper_2501_04194_b200.engine import compile_formula

mode = sys.argv[1] if len(sys.argv) > 1 else "lse"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
B, T = 1024, 10_000
rng = np.random.default_rng(1)
p = np.asarray(rng.uniform(-1, 1, (B, 1, 2)) + np.cumsum(0.05 * rng.normal(0, 1, (B, T, 2)), 1),
               dtype=np.float32)
dev = torch.device("cuda", 0)
pt = torch.tensor(p, device=dev)
cfg = P.SemanticsConfig(mode={"lse": P.LogSumExp(10.0), "hard": P.Hard(), "hard1d": P.Hard(),
                               "soft": P.SoftMax(10.0)}[mode])
if mode == "hard1d":  # C1's formula at full size, contiguous 1-D signal
    f = P.Always(P.Pred("x", ">", 0.5), P.StepInterval(0, 50))
    names = ["x"]
    chans = [pt[..., 0].contiguous()]
elif mode == "hard":
    f = P.Eventually(P.NormPred(("px", "py"), "<", 0.5), P.StepInterval(10, 100))
    names = ["px", "py"]
    chans = [pt[..., 0], pt[..., 1]]
else:
    f = P.Eventually(P.NormPred(("px", "py"), "<", 0.5), P.StepInterval(10, 100))
    names = ["px", "py"]
    chans = [pt[..., 0], pt[..., 1]]
comp = compile_formula(f, names, cfg)
fb, bb = comp.workspace_bytes(B, T)
fws = torch.empty(fb, dtype=torch.uint8, device=dev)
bws = torch.empty(bb, dtype=torch.uint8, device=dev)
out = torch.empty(B, T, device=dev)
ones = torch.ones(B, T, device=dev)
dp = torch.zeros(B, T, 2, device=dev)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(steps):
    comp.forward(chans, [], out, fws, s)
    grads = [dp[..., 0].contiguous()] if mode == "hard1d" else [dp[..., i] for i in range(len(chans))]
    comp.backward(chans, [], out, ones, grads, None, fws, bws, s)
torch.cuda.synchronize()
print("ok", float(out[0, 0]), float(dp.abs().sum()))
