"""``--engine b200`` for the reference's own host plumbing.

The reference CLI (``stlmask/cli.py``) parses formulas with its DSL
(``formula.parse``, formula.py:310-321), reads CSV signals (``fileio``) and routes
``eval`` / ``trace`` through ``_trace_for(engine, f, signals, cfg)`` (cli.py:56-61)
with the engine choices declared in ``_add_semantics_flags`` (cli.py:190-191).  Those
pieces are reused unchanged; ``install()`` adds one engine name, ``"b200"``, whose
trace is ``paper_2501_04194_b200.robustness_trace`` — the reference's AST, signals and
``SemanticsConfig`` objects are accepted as they are (duck-typed by class name).

    python -m paper_2501_04194_b200.stlmask_engine trace "F[0,3] (x > 0)" data.csv --engine b200

Errors raised by the device path are re-raised as the reference's exception class of
the same name, so the CLI's own handlers (cli.py:247-254) map them to its exit codes.
"""

from __future__ import annotations

import sys

import numpy as np

ENGINE = "b200"

__all__ = ["ENGINE", "b200_trace", "install", "main"]


def _as_reference_error(exc, core):
    cls = getattr(core, type(exc).__name__, None)
    if cls is None or not isinstance(cls, type) or not issubclass(cls, Exception):
        return exc
    if type(exc).__name__ == "ValidationError":
        return cls(getattr(exc, "missing", []))
    return cls(str(exc))


def b200_trace(f, signals, cfg) -> np.ndarray:
    """``masking.robustness_trace`` (masking.py:350-357) on the device."""
    from . import engine
    from . import core as our_core
    try:
        return engine.robustness_trace(f, signals, cfg)
    except our_core.StlError as exc:
        import stlmask.core as ref_core
        raise _as_reference_error(exc, ref_core) from exc


def install(cli=None):
    """Register ``--engine b200`` in the reference CLI module (idempotent)."""
    if cli is None:
        import stlmask.cli as cli
    if getattr(cli, "_b200_installed", False):
        return cli
    orig_trace_for = cli._trace_for
    orig_flags = cli._add_semantics_flags

    def _trace_for(engine, f, signals, cfg):
        if engine == ENGINE:
            return b200_trace(f, signals, cfg)
        return orig_trace_for(engine, f, signals, cfg)

    def _add_semantics_flags(p):
        orig_flags(p)
        for action in p._actions:
            if action.dest == "engine" and action.choices is not None and ENGINE not in action.choices:
                action.choices = tuple(action.choices) + (ENGINE,)

    cli._trace_for = _trace_for
    cli._add_semantics_flags = _add_semantics_flags
    cli._b200_installed = True
    return cli


def main(argv=None) -> int:
    cli = install()
    return cli.main(argv)


if __name__ == "__main__":
    sys.exit(main())
