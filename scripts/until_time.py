"""Forward / backward timings of untimed Until (LSE and Hard) at the C3 / C5 shapes.

    STLG_UL=0|1 python scripts/until_time.py
STLG_UL=0 routes untimed LSE Until through the per-pair kernels (the reciprocal-form
kernels are the default).
"""
import json
import os
import statistics
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

import torch

import paper_2501_04194_b200 as P
from paper_2501_04194_b200.engine import compile_formula

sys.path.insert(0, os.path.join(ROOT, "scripts"))
from configs_bench import timed  # noqa: E402

dev = torch.device("cuda", 0)


def main():
    g = torch.Generator(device=dev).manual_seed(0)
    cases = [("C3-until", 256, 4000), ("C5-U", 4096, 1000), ("C5-U", 1024, 10000)]
    for name, B, T in cases:
        xs = {"y": torch.randn(B, T, device=dev, generator=g), "z": torch.randn(B, T, device=dev, generator=g)}
        f = P.Until(P.Pred("y", "<", 1.0), P.Pred("z", ">", 0.0))
        for mname, m in (("lse10", P.LogSumExp(10.0)), ("lse1", P.LogSumExp(1.0))):
            comp = compile_formula(f, ["y", "z"], P.SemanticsConfig(mode=m))
            fm, bm = timed(comp, xs, B, T, reps=3)
            pairs = B * T * (T + 1) / 2
            print(json.dumps({"case": name, "mode": mname, "B": B, "T": T, "UL": os.environ.get("STLG_UL", "1"),
                              "fwd_ms": round(fm, 4), "bwd_ms": round(bm, 4),
                              "fwd_pairs_per_s": pairs / (fm * 1e-3)}), flush=True)


if __name__ == "__main__":
    main()
