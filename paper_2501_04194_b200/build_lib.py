"""Build libstlg.so in-tree with nvcc for sm_100a (no torch involvement).

    python -m paper_2501_04194_b200.build_lib [--force]
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.abspath(os.path.join(HERE, "..", "include"))
LIB = os.path.join(HERE, "libstlg.so")
SOURCES = ["exec.cu", "fg.cu", "fg_reg_fwd.cu", "fg_unt.cu", "fg_soft64.cu", "until.cu", "until_ht.cu", "smooth.cu", "mining.cu"]
# (object name, source, defines): fg_reg_inst.cu once per tile width and direction
VARIANTS = [(f"fg_reg_{'b' if bwd else 'f'}{nw}", "fg_reg_inst.cu", [f"-DREG_NW={nw}", f"-DREG_BWD={bwd}"])
            for bwd in (1, 0) for nw in (3, 4, 5, 6, 7, 8)]
HEADERS = ["common.cuh", "kernels.cuh", "fg_reg.cuh", "fg_cav.cuh", "detacc.cuh", "lookback.cuh"]
UNITS = [(os.path.splitext(s)[0], s, []) for s in SOURCES] + VARIANTS

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "--extended-lambda",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-cudart", "static", "-shared",
]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS + ["fg_reg_inst.cu"]] + [os.path.join(INCLUDE, "stlg.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = True) -> str:
    """Compile each translation unit in parallel (objects newer than their sources and
    headers are kept unless force=True), then link libstlg.so."""
    lib_out = LIB
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f not in ("-shared",)]

    hdr_t = max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS)
    hdr_t = max(hdr_t, os.path.getmtime(os.path.join(INCLUDE, "stlg.h")), os.path.getmtime(__file__))
    import time

    def compile_one(unit):
        name, src, defs = unit
        obj = os.path.join(objdir, name + ".o")
        srcp = os.path.join(CSRC, src)
        # incremental: an object newer than its source, every header and this file is kept
        # (force=True rebuilds everything)
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) > max(os.path.getmtime(srcp), hdr_t)):
            return obj
        cmd = [_nvcc(), *compile_flags, *defs, "-I", INCLUDE, "-c", "-o", obj, srcp]
        if verbose:
            print(" ".join(cmd), flush=True)
        t0 = time.time()
        subprocess.run(cmd, check=True)
        if verbose:
            print(f"  {name}: {time.time() - t0:.0f} s", flush=True)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(UNITS), os.cpu_count() or 8)) as ex:
        objs = list(ex.map(compile_one, sorted(UNITS, key=lambda u: u[1] != "fg_reg_inst.cu")))
    tmp = lib_out + ".tmp"
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
           "-Xcompiler", "-fPIC", "-o", tmp, *objs]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib_out)
    return lib_out


if __name__ == "__main__":
    build(force="--force" in sys.argv)
