"""In-tree build of libcrn.so (sm_100a) with plain nvcc.

``python -m paper_1905_01141_b200.build`` or ``build()`` from Python.  The .so
lands next to this file so it travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libcrn.so")
SOURCES = ["crn_host.cpp", "crn_runtime.cpp", "crn_decode.cu", "crn_encode.cu", "crn_tb.cu", "crn_ratematch.cu", "crn_tbseg.cu", "crn_tasks.cu", "crn_ubench.cu"]
HEADERS = ["crn_internal.h", "crn_plan.h", "qpp_table.h", os.path.join("..", "..", "include", "crn.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, so: str | None = None, defines=(), replace=None) -> str:
    """Compile libcrn.so (or, for profiling / A-B experiments, ``so`` with extra
    ``-D`` defines, e.g. CRN_PHASE_PROF, and ``replace`` = {source: alternative
    file} for A/B variants; never the product library)."""
    if so is None and not force and not _stale():
        return SO
    from concurrent.futures import ThreadPoolExecutor
    target = SO if so is None else so
    bdir = os.path.join(HERE, "build" if so is None else "build_" + os.path.basename(so).replace(".so", ""))
    os.makedirs(bdir, exist_ok=True)
    cmds, objs = [], []
    for s in SOURCES:
        o = os.path.join(bdir, s + ".o")
        src = (replace or {}).get(s, os.path.join(CSRC, s))
        cmd = [NVCC, *ARCH, *FLAGS, *(f"-D{d}" for d in defines), "-I", CSRC, "-c", src, "-o", o]
        if verbose and s.endswith(".cu"):
            cmd.insert(1, "-Xptxas=-v")
        cmds.append(cmd)
        objs.append(o)
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:   # independent units
        list(ex.map(subprocess.check_call, cmds))
    tmp = target + ".tmp"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs])
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    if "--prof" in sys.argv:            # phase-profiler build (tools/phase_prof.py): libcrn_prof.so
        print(build(so=os.path.join(HERE, "libcrn_prof.so"), defines=("CRN_PHASE_PROF",)))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
