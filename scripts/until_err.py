"""Error anatomy of long untimed LSE Until on the device vs the oracle (precision A/B)."""
import os, sys
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests")); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import paper_2501_04194_b200 as P
import stl_oracle
from devhelp import rel_err, run_device
for T in (1000, 3000, 6000):
    rng = np.random.default_rng(6000)
    x = np.asarray(rng.normal(0, 1, (1, T)), dtype=np.float32).astype(np.float64)
    y = np.asarray(rng.normal(0, 1, (1, T)), dtype=np.float32).astype(np.float64)
    f = P.Until(P.Pred("x", ">", 0.0), P.Pred("y", ">", 0.0))
    cfg = P.SemanticsConfig(mode=P.LogSumExp(10.0))
    for cname, cot in (("ones", np.ones((1, T))), ("randn", rng.normal(0, 1, (1, T)))):
        tr, g, _ = run_device(f, {"x": x, "y": y}, cfg, cot=cot)
        ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, {"x": x, "y": y}, cfg, cot)
        ex = np.abs(g["x"] - ref_g["x"]) / np.maximum(1, np.abs(ref_g["x"]))
        ey = np.abs(g["y"] - ref_g["y"]) / np.maximum(1, np.abs(ref_g["y"]))
        i = int(np.argmax(ex))
        print(T, cname, "tr %.2e gx %.2e gy %.2e" % (rel_err(tr, ref_tr), ex.max(), ey.max()),
              "worst x at", i, "ref", ref_g["x"][0, i], "got", g["x"][0, i], "|ref| max", np.abs(ref_g["x"]).max())
