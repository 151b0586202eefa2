"""Formula AST (host side).

Node classes carry the reference's names and fields
(``/root/reference/pkg/src/stlmask/formula.py:65-135``) so that ASTs built
for ``stlmask`` — including ones produced by its DSL ``parse`` — can be
handed to this package unchanged; the compiler (``compile.py``) dispatches
on class *name* and fields, so reference objects are accepted duck-typed.

STLCG++ spellings are provided as aliases: ``Predicate`` = ``Pred``,
``Negation`` = ``Not``.

``NormPred`` is a build-side extension: the signed margin
of a Euclidean distance ``||(x, y) - center||`` against a radius.  The
reference has no such node; its equivalent is a ``Pred`` on a channel that
holds the distance, built on the tape with ``sqrt``/``square``
(``apps.py:150-151``).
"""

from __future__ import annotations

import json
import re
from dataclasses import dataclass
from typing import Optional, Union

from .core import SmoothInterval, StepInterval

__all__ = [
    "Formula", "TrueFormula", "TRUE", "Pred", "Predicate", "Not", "Negation", "And", "Or",
    "Eventually", "Always", "Until", "NormPred", "variables", "validate_against",
    "to_json", "from_json", "smooth_intervals",
]

_CMPS = (">", "<", ">=", "<=")
_IDENT = re.compile(r"[A-Za-z_]\w*")


@dataclass(frozen=True)
class Formula:
    """Base node; ``&``, ``|`` and ``~`` build And / Or / Not."""

    def __and__(self, other):
        return And(self, other)

    def __or__(self, other):
        return Or(self, other)

    def __invert__(self):
        return Not(self)


@dataclass(frozen=True)
class TrueFormula(Formula):
    pass


TRUE = TrueFormula()


def _check_var(name):
    if not name or not _IDENT.fullmatch(name):
        raise ValueError(f"predicate variable must be an identifier, got {name!r}")


def _check_cmp(cmp):
    if cmp not in _CMPS:
        raise ValueError(f"comparator must be one of {_CMPS}, got {cmp!r}")


@dataclass(frozen=True)
class Pred(Formula):
    """``var cmp threshold``; ``>=``/``<=`` behave as ``>``/``<`` (formula.py:16-18)."""

    var: str
    cmp: str
    threshold: float

    def __post_init__(self):
        _check_var(self.var)
        _check_cmp(self.cmp)


Predicate = Pred


@dataclass(frozen=True)
class NormPred(Formula):
    """``||(vars[0], vars[1]) - center|| cmp threshold`` (extension, see module doc)."""

    vars: tuple
    cmp: str
    threshold: float
    center: tuple = (0.0, 0.0)

    def __post_init__(self):
        if len(self.vars) != 2 or len(self.center) != 2:
            raise ValueError("NormPred takes exactly two channels and a 2-D center")
        for v in self.vars:
            _check_var(v)
        _check_cmp(self.cmp)
        object.__setattr__(self, "vars", tuple(self.vars))
        object.__setattr__(self, "center", tuple(float(c) for c in self.center))


@dataclass(frozen=True)
class Not(Formula):
    arg: Formula


Negation = Not


@dataclass(frozen=True)
class And(Formula):
    left: Formula
    right: Formula


@dataclass(frozen=True)
class Or(Formula):
    left: Formula
    right: Formula


@dataclass(frozen=True)
class Eventually(Formula):
    arg: Formula
    interval: Union[StepInterval, SmoothInterval, None] = None


@dataclass(frozen=True)
class Always(Formula):
    arg: Formula
    interval: Union[StepInterval, SmoothInterval, None] = None


@dataclass(frozen=True)
class Until(Formula):
    left: Formula
    right: Formula
    interval: Optional[StepInterval] = None


# --------------------------------------------------------------------------
# structural queries (formula.py:403-420)
# --------------------------------------------------------------------------

def _kind(f) -> str:
    return type(f).__name__


def variables(f) -> set:
    k = _kind(f)
    if k == "Pred":
        return {f.var}
    if k == "NormPred":
        return set(f.vars)
    if k == "TrueFormula":
        return set()
    if k == "Not":
        return variables(f.arg)
    if k in ("And", "Or", "Until"):
        return variables(f.left) | variables(f.right)
    if k in ("Eventually", "Always"):
        return variables(f.arg)
    raise TypeError(f"not a Formula node: {f!r}")


def validate_against(f, signals) -> list:
    names = set(signals.names()) if hasattr(signals, "names") else set(signals)
    return sorted(variables(f) - names)


def smooth_intervals(f) -> list:
    """Smooth-interval objects in pre-order (autodiff.py:41-49)."""
    k = _kind(f)
    if k in ("Eventually", "Always"):
        here = [f.interval] if _kind(f.interval) == "SmoothInterval" else []
        return here + smooth_intervals(f.arg)
    if k == "Not":
        return smooth_intervals(f.arg)
    if k in ("And", "Or", "Until"):
        return smooth_intervals(f.left) + smooth_intervals(f.right)
    return []


# --------------------------------------------------------------------------
# JSON encoding (used by the golden fixtures and the bench config)
# --------------------------------------------------------------------------

def _iv_json(iv):
    if iv is None:
        return None
    if _kind(iv) == "StepInterval":
        return {"step": [int(iv.a), int(iv.b)]}
    return {"smooth": [float(iv.a), float(iv.b), float(iv.c), float(iv.eps)]}


def to_json(f) -> str:
    def enc(g):
        k = _kind(g)
        if k == "TrueFormula":
            return ["T"]
        if k == "Pred":
            return ["P", g.var, g.cmp, float(g.threshold)]
        if k == "NormPred":
            return ["N", list(g.vars), g.cmp, float(g.threshold), list(g.center)]
        if k == "Not":
            return ["~", enc(g.arg)]
        if k in ("And", "Or"):
            return ["&" if k == "And" else "|", enc(g.left), enc(g.right)]
        if k in ("Eventually", "Always"):
            return ["F" if k == "Eventually" else "G", enc(g.arg), _iv_json(g.interval)]
        if k == "Until":
            return ["U", enc(g.left), enc(g.right), _iv_json(g.interval)]
        raise TypeError(f"not a Formula node: {g!r}")
    return json.dumps(enc(f))


def _iv_from(d):
    if d is None:
        return None
    if "step" in d:
        return StepInterval(*[int(v) for v in d["step"]])
    return SmoothInterval(*d["smooth"])


def from_json(s: str, ns=None):
    """Decode; ``ns`` may supply alternative node classes (e.g. the reference's)."""
    ns = ns or globals()

    def dec(e):
        tag = e[0]
        if tag == "T":
            return ns["TRUE"]
        if tag == "P":
            return ns["Pred"](e[1], e[2], e[3])
        if tag == "N":
            return NormPred(tuple(e[1]), e[2], e[3], tuple(e[4]))
        if tag == "~":
            return ns["Not"](dec(e[1]))
        if tag in ("&", "|"):
            return ns["And" if tag == "&" else "Or"](dec(e[1]), dec(e[2]))
        if tag in ("F", "G"):
            return ns["Eventually" if tag == "F" else "Always"](dec(e[1]), _iv_from_ns(e[2], ns))
        if tag == "U":
            return ns["Until"](dec(e[1]), dec(e[2]), _iv_from_ns(e[3], ns))
        raise ValueError(f"bad formula tag {tag!r}")
    return dec(json.loads(s))


def _iv_from_ns(d, ns):
    if d is None:
        return None
    if "step" in d:
        return ns["StepInterval"](*[int(v) for v in d["step"]])
    return ns["SmoothInterval"](*d["smooth"])
