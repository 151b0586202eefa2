"""Softmax window trace / gradient errors vs the oracle (precision A/B across kernel families)."""
import os, sys
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests")); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import paper_2501_04194_b200 as P
import stl_oracle
from devhelp import rel_err, run_device
from test_gpu_windows import _data
for (a, b) in [(0, 15), (5, 36), (10, 100), (7, 1030)]:
    for L in (1000, 9001):
        rng = np.random.default_rng(17 + 1000 * a + b + L)
        x = _data(rng, 3, L, False)
        iv = P.StepInterval(a, b)
        f = P.Eventually(P.Pred("x", ">", 0.1), iv) if (a + L) % 2 else P.Always(P.Pred("x", "<", 0.3), iv)
        cfg = P.SemanticsConfig(mode=P.SoftMax(10.0))
        cot = rng.normal(0, 1, (3, L))
        tr, g, _ = run_device(f, {"x": x}, cfg, cot=cot)
        ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, {"x": x}, cfg, cot)
        print(os.environ.get("STLG_REG", "1"), a, b, L, "tr %.2e g %.2e" % (rel_err(tr, ref_tr), rel_err(g["x"], ref_g["x"])),
              "max|x| %.1f" % np.abs(x).max(), flush=True)
