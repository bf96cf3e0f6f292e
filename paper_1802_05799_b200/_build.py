"""Build the C-ABI shared library ``libhvd_b200.so`` in-tree with nvcc (sm_100a).

The library is the product: every step of the hot path runs in its kernels.
It is built in the package directory so that it travels with the repo
snapshot to the GPU box (gpurun) and is what the tests and bench load.
"""
from __future__ import annotations

import hashlib
import os
import pathlib
import shutil
import subprocess

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libhvd_b200.so"
SOURCES = ["hvd_kernels.cu", "hvd_runtime.cpp", "hvd_plan.cpp", "hvd_negotiate.cpp", "hvd_jobtrace.cpp"]
HEADERS = ["hvd_internal.h", "hvd_plan.h", "hvd_negotiate.h", "hvd_jobtrace.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: no FMA contraction anywhere (bit parity with the oracle, SURVEY §7 hard part 5)
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC,-O2",
              "-Xptxas", "-warn-spills"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def source_hash() -> str:
    """sha256 over every source, header, this file and the extra flags: the build id the
    library embeds (``hvd_build_id()``), so a stale or foreign .so is never reused."""
    h = hashlib.sha256()
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "hvd.h", pathlib.Path(__file__)]
    for d in deps:
        h.update(d.name.encode())
        h.update(d.read_bytes())
    h.update(os.environ.get("HVD_NVCC_EXTRA", "").encode())
    return h.hexdigest()[:32]


def _stale() -> bool:
    if not LIB.exists():
        return True
    # the id string is a literal in the library's .rodata: no need to load it
    return ("hvd-src-" + source_hash()).encode() not in LIB.read_bytes()


def build(force: bool = False, verbose: bool = False) -> pathlib.Path:
    if not force and not _stale():
        return LIB
    nvcc = _nvcc()
    bid = ["-DHVD_BUILD_ID=\"hvd-src-%s\"" % source_hash()]
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = objdir / (src + ".o")
        # HVD_NVCC_EXTRA: tuning experiments only (e.g. -DHVD_SOLO_U=8); the product build sets none
        extra = os.environ.get("HVD_NVCC_EXTRA", "").split()
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *extra, *bid, "-I", str(ROOT / "include"), "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *objs, "-cudart", "static", "-ldl"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
