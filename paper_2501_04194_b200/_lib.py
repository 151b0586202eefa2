"""ctypes binding of libstlg.so (include/stlg.h).

The library is built in-tree by ``build_lib.py`` (``__graft_entry__.build()``).
There is no fallback: if the shared object is missing or from another ABI
version, every compute call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_size_t, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libstlg.so")
ABI_VERSION = 1

# opcodes / codes (stlg.h)
OP_TRUE, OP_PRED, OP_NOT, OP_AND, OP_OR, OP_EV, OP_AL, OP_UNTIL, OP_NORM = range(9)
ITV_NONE, ITV_STEP, ITV_SMOOTH = 0, 1, 2
MODE_HARD, MODE_SOFTMAX, MODE_LSE = 0, 1, 2
OK, E_SHAPE, E_EMPTY_WINDOW, E_UNSUPPORTED, E_CUDA, E_INVALID = range(6)

EXPORTS = ("stlg_abi_version", "stlg_last_error", "stlg_compile", "stlg_free", "stlg_plan_info",
           "stlg_workspace_bytes", "stlg_forward", "stlg_backward", "stlg_launch_count",
           "stlg_mining_grid")


class StlgNode(ctypes.Structure):
    _fields_ = [("op", c_int32), ("left", c_int32), ("right", c_int32), ("chan", c_int32),
                ("chan2", c_int32), ("cmp", c_int32), ("threshold", c_double),
                ("center0", c_double), ("center1", c_double), ("itv_kind", c_int32),
                ("a", c_int32), ("b", c_int32), ("smooth_slot", c_int32)]


class StlgCfg(ctypes.Structure):
    _fields_ = [("mode", c_int32), ("temp", c_double), ("pad_last", c_int32),
                ("pad_value", c_double), ("top_value", c_double), ("sentinel", c_double),
                ("masked_fill", c_int32)]


class StlgChannel(ctypes.Structure):
    _fields_ = [("ptr", c_void_p), ("row_stride", c_int64), ("elem_stride", c_int64)]


class StlgGrad(ctypes.Structure):
    _fields_ = [("ptr", c_void_p), ("row_stride", c_int64), ("elem_stride", c_int64),
                ("accumulate", c_int32)]


class StlgSmooth(ctypes.Structure):
    _fields_ = [("a", c_double), ("b", c_double), ("c", c_double), ("eps", c_double)]


_lib = None
_lock = threading.Lock()


def load():
    """Load (once) and return the library handle; raises if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = LIB_PATH
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} is missing: build it with `python -m paper_2501_04194_b200.build_lib` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        lib.stlg_abi_version.restype = c_int
        lib.stlg_last_error.restype = ctypes.c_char_p
        lib.stlg_compile.argtypes = [POINTER(StlgNode), c_int32, c_int32, c_int32, POINTER(StlgCfg),
                                     POINTER(c_void_p)]
        lib.stlg_compile.restype = c_int
        lib.stlg_free.argtypes = [c_void_p]
        lib.stlg_free.restype = None
        lib.stlg_plan_info.argtypes = [c_void_p, POINTER(c_int32), POINTER(c_int32), POINTER(c_int32)]
        lib.stlg_plan_info.restype = c_int
        lib.stlg_workspace_bytes.argtypes = [c_void_p, c_int64, c_int64, POINTER(c_size_t),
                                             POINTER(c_size_t)]
        lib.stlg_workspace_bytes.restype = c_int
        lib.stlg_forward.argtypes = [c_void_p, POINTER(StlgChannel), c_int64, c_int64,
                                     POINTER(StlgSmooth), c_void_p, c_void_p, c_size_t, c_void_p]
        lib.stlg_forward.restype = c_int
        lib.stlg_backward.argtypes = [c_void_p, POINTER(StlgChannel), c_int64, c_int64,
                                      POINTER(StlgSmooth), c_void_p, c_void_p, POINTER(StlgGrad),
                                      c_void_p, c_void_p, c_size_t, c_void_p, c_size_t, c_void_p]
        lib.stlg_backward.restype = c_int
        lib.stlg_launch_count.argtypes = [c_int]
        lib.stlg_launch_count.restype = c_int64
        lib.stlg_mining_grid.argtypes = [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_int64,
                                         c_double, c_double, c_int32, c_double, c_double, c_void_p,
                                         c_void_p, c_void_p]
        lib.stlg_mining_grid.restype = c_int
        got = lib.stlg_abi_version()
        if got != ABI_VERSION:
            raise RuntimeError(f"libstlg ABI {got} != expected {ABI_VERSION}; rebuild the library")
        _lib = lib
        return lib


def check(rc: int):
    """Map a status code to the reference's exception classes (stlg.h)."""
    if rc == OK:
        return
    from .core import EmptyWindowError, ShapeError
    msg = load().stlg_last_error().decode(errors="replace")
    if rc == E_SHAPE:
        raise ShapeError(msg)
    if rc == E_EMPTY_WINDOW:
        raise EmptyWindowError(msg)
    if rc == E_UNSUPPORTED:
        raise TypeError(msg)
    if rc == E_CUDA:
        raise RuntimeError(msg)
    raise ValueError(msg)
