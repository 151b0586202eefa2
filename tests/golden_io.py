"""Load the reference-generated golden vectors (tests/golden/*.npz)."""

from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

from paper_2501_04194_b200.core import (Hard, LogSumExp, PaddingPolicy, SemanticsConfig, StepInterval,
                                        SmoothInterval, SoftMax)
from paper_2501_04194_b200.formula import from_json

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@dataclass
class Case:
    name: str
    formula: object
    cfg: SemanticsConfig
    arrays: dict
    cot: np.ndarray
    trace: np.ndarray
    grads: dict
    dabc: object
    si: object

    @property
    def mode(self):
        return type(self.cfg.mode).__name__


def cfg_from_json(s: str) -> SemanticsConfig:
    d = json.loads(s)
    mode = {"Hard": lambda t: Hard(), "LogSumExp": LogSumExp, "SoftMax": SoftMax}[d["mode"]](d["temp"])
    pad = PaddingPolicy("last") if d["pad"] == "last" else PaddingPolicy("const", d["pad_value"])
    return SemanticsConfig(mode=mode, padding=pad, sentinel=d["sentinel"],
                           top_value=d["top_value"], masked_fill=d["masked_fill"])


def load(name: str) -> list[Case]:
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    meta = json.loads(str(z["meta"]))
    cases = []
    for i, m in enumerate(meta):
        p = f"c{i}_"
        arrays = {k: z[p + "x_" + k] for k in m["channels"]}
        grads = {k: z[p + "g_" + k] for k in m["channels"]}
        si = None
        if m["has_si"]:
            a, b, c, eps = z[p + "si"]
            si = SmoothInterval(float(a), float(b), float(c), float(eps))
        cases.append(Case(m["name"], from_json(m["formula"]), cfg_from_json(m["cfg"]), arrays,
                          z[p + "cot"], z[p + "trace"], grads,
                          z[p + "dabc"] if m["has_dabc"] else None, si))
    return cases


def load_all() -> list[Case]:
    return load("kats") + load("random") + load("smooth_norm")


@dataclass
class ApiCase:
    """One reference call of the public wrappers (tests/golden/make_api_golden.py)."""
    meta: dict
    arrays: dict

    @property
    def cfg(self):
        return cfg_from_json(self.meta["cfg"])

    def interval(self, key):
        d = self.meta.get(key)
        if d is None:
            return None
        if "step" in d:
            return StepInterval(*[int(v) for v in d["step"]])
        return SmoothInterval(*d["smooth"])


def load_api() -> list[ApiCase]:
    z = np.load(os.path.join(GOLDEN, "api.npz"))
    meta = json.loads(str(z["meta"]))
    return [ApiCase(m, {k: z[f"c{i}_{k}"] for k in m["arrays"]}) for i, m in enumerate(meta)]
