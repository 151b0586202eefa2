"""Reproduce tests/test_gpu_parity.py::test_random_formulas_vs_oracle[seed] and locate mismatches."""
import os, sys
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)
import numpy as np
import stl_oracle
from devhelp import run_device, rel_err
import test_gpu_parity as T
import paper_2501_04194_b200 as P
seed = int(sys.argv[1])
rng = np.random.default_rng(1000 + seed)
mode = T.MODES[seed % len(T.MODES)]
pad = P.PaddingPolicy.last_value() if seed % 3 else P.PaddingPolicy.constant(-0.75)
cfg = P.SemanticsConfig(mode=mode, padding=pad, top_value=100.0)
f = T._rand_formula(rng, int(rng.integers(1, 4)))
B, L = 3, int(rng.integers(20, 400))
arrays = {c: np.asarray(rng.normal(0, 1.5, (B, L)), dtype=np.float32).astype(np.float64) for c in ("x", "y")}
cot = np.ones((B, L)) if seed % 2 == 0 else np.asarray(rng.normal(0, 1, (B, L)), dtype=np.float32).astype(np.float64)
print("formula", P.to_json(f), "mode", mode, "pad", pad, "L", L)
ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, arrays, cfg, cot)
tr, g, _ = run_device(f, arrays, cfg, cot)
print("trace err", rel_err(tr, ref_tr))
for k in ref_g:
    e = np.abs(g[k] - ref_g[k]) / np.maximum(1, np.abs(ref_g[k]))
    idx = np.argwhere(e > 1e-5)
    print(k, "max err", e.max(), "n bad", len(idx), idx[:10].tolist())
    for b_, j in idx[:5]:
        print("   ", b_, j, "got", g[k][b_, j], "ref", ref_g[k][b_, j])
