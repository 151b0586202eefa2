"""Error report for the smooth-interval density test inputs (tests/test_gpu_parity.py), per component."""
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import paper_2501_04194_b200 as P
from oracle import stl_oracle
from devhelp import run_device, rel_err
for mode in (P.LogSumExp(5.0), P.SoftMax(2.0)):
    for zf in (0.0, 0.5, 0.995):
        rng = np.random.default_rng(1234)
        B, L = 4, 1500
        if type(mode).__name__ == "LogSumExp":
            x = np.cumsum(np.asarray(rng.normal(0, 0.3, (B, L)), dtype=np.float32), axis=1).astype(np.float64)
        else:
            x = np.asarray(rng.normal(0, 1, (B, L)), dtype=np.float32).astype(np.float64)
        si = P.SmoothInterval(0.2, 0.6, 9.0)
        f = P.Always(P.Pred("x", ">", 0.0), si)
        cfg = P.SemanticsConfig(mode=mode)
        cot = rng.uniform(0.25, 1.75, (B, L)); cot[rng.random((B, L)) < zf] = 0.0
        cot = np.asarray(cot, dtype=np.float32).astype(np.float64)
        b = (si.a, si.b, si.c)
        rt, rg, ra = stl_oracle.trace_and_grad(f, {"x": x}, cfg, cotangent=cot, smooth_binding=b)
        tr, g, da = run_device(f, {"x": x}, cfg, cot, b)
        print(type(mode).__name__, zf, "tr", rel_err(tr, rt), "gx", rel_err(g["x"], rg["x"]),
              "abc", rel_err(da, np.array(ra)), np.asarray(da), np.asarray(ra), flush=True)
