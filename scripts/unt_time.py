import os, sys, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "scripts"))
import torch, paper_2501_04194_b200 as P
from configs_bench import timed
from paper_2501_04194_b200.engine import compile_formula
g = torch.Generator(device="cuda").manual_seed(0)
for T in (10_000, 100_000):
    B = 4096 if T == 10_000 else 1024
    x = torch.randn(B, T, device="cuda", generator=g)
    for mname, m in (("hard", P.Hard()), ("lse10", P.LogSumExp(10.0))):
        comp = compile_formula(P.Eventually(P.Pred("x", ">", 0.0)), ["x"], P.SemanticsConfig(mode=m))
        fm, bm = timed(comp, {"x": x}, B, T, reps=5)
        print(json.dumps({"reg": os.environ.get("STLG_REG", "1"), "T": T, "B": B, "mode": mname, "fwd_ms": fm, "bwd_ms": bm}))
