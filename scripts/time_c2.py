"""Time the C2 forward / backward kernels with CUDA graphs (no host overhead in the window)."""
import ctypes, os, sys, json
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2501_04194_b200 as P
from paper_2501_04194_b200.engine import compile_formula
mode = sys.argv[1] if len(sys.argv) > 1 else "lse"
B, T = 1024, 10_000
rng = np.random.default_rng(1)
p = np.asarray(rng.uniform(-1, 1, (B, 1, 2)) + np.cumsum(0.05 * rng.normal(0, 1, (B, T, 2)), 1), dtype=np.float32)
dev = torch.device("cuda", 0)
cfg = P.SemanticsConfig(mode={"lse": P.LogSumExp(10.0), "hard": P.Hard(), "hard1d": P.Hard(),
                               "soft": P.SoftMax(10.0)}[mode])
if mode == "hard1d":  # C1's formula at full size: Always[0,50](x > 0.5), contiguous 1-D signal
    f = P.Always(P.Pred("x", ">", 0.5), P.StepInterval(0, 50))
    comp = compile_formula(f, ["x"], cfg)
else:
    f = P.Eventually(P.NormPred(("px", "py"), "<", 0.5), P.StepInterval(10, 100))
    comp = compile_formula(f, ["px", "py"], cfg)
sets = [torch.tensor(np.roll(p, 17 * i, 1), device=dev) for i in range(3)]
if mode == "hard1d":
    sets = [s_[..., 0].contiguous() for s_ in sets]
fb, bb = comp.workspace_bytes(B, T)
fws = torch.empty(fb, dtype=torch.uint8, device=dev); bws = torch.empty(bb, dtype=torch.uint8, device=dev)
outs = [torch.empty(B, T, device=dev) for _ in range(3)]
dps = [torch.empty(B, T, 2, device=dev) for _ in range(3)]
ones = torch.ones(B, T, device=dev)
def cur(): return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
if mode == "hard1d":
    dps = [torch.empty(B, T, device=dev) for _ in range(3)]
    def fwd(i): comp.forward([sets[i]], [], outs[i], fws, cur())
    def bwd(i): comp.backward([sets[i]], [], outs[i], ones, [dps[i]], None, fws, bws, cur())
else:
    def fwd(i): comp.forward([sets[i][..., 0], sets[i][..., 1]], [], outs[i], fws, cur())
    def bwd(i): comp.backward([sets[i][..., 0], sets[i][..., 1]], [], outs[i], ones, [dps[i][..., 0], dps[i][..., 1]], None, fws, bws, cur())
for i in range(6): fwd(i % 3); bwd(i % 3)
torch.cuda.synchronize()
gf, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
with torch.cuda.graph(gf):
    for i in range(3): fwd(i)
with torch.cuda.graph(gb):
    for i in range(3): bwd(i)
for _ in range(3): gf.replay(); gb.replay()
torch.cuda.synchronize()
N = 10
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
e[0].record()
for _ in range(N): gf.replay()
e[1].record()
for _ in range(N): gb.replay()
e[2].record()
torch.cuda.synchronize()
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("STLG_"))
print(json.dumps({"cfg": tag or "default", "mode": mode, "fwd_us": 1e3 * e[0].elapsed_time(e[1]) / (3 * N),
                  "bwd_us": 1e3 * e[1].elapsed_time(e[2]) / (3 * N)}))
