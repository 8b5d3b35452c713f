"""Build libmdrq_b200.so (sm_100a) in-tree with nvcc.

The shared library is the product's only compute path; it is built here
(cross-compiled, no GPU needed) and shipped to the GPU box with the repo.
``python -m paper_1801_03644_b200.build`` rebuilds it when a source changed.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libmdrq_b200.so")

SOURCES = ["store.cu", "scan_columnar.cu", "scan_rowwise.cu", "vafile.cu", "masks.cu", "expand.cu", "vabatch.cu", "pack.cu"]
# plain host C++ (g++): the multi-threaded id unpacker
HOST_SOURCES = ["unpack_host.cpp"]
HEADERS = ["common.cuh", "launch.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# Exact IEEE semantics: the kernels only compare, but never let a fast-math
# flag flush subnormals or contract anything (SURVEY.md 7 "Bit-exactness").
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true", "-fmad=false",
    "-Xptxas", "-v", "-I", CSRC, "-I", INCLUDE,
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


LIB_CHECKED = os.path.join(PKG, "libmdrq_b200_checked.so")


def build(force: bool = False, verbose: bool = False, checked: bool = False,
          variant: str = "", defines=()) -> str:
    """Build libmdrq_b200.so; ``checked`` builds libmdrq_b200_checked.so with
    the device-side bounds checks (MDRQ_CHECKS, common.cuh) into its own
    object directory.  The product loads the release library; the checked one
    is for tests (MDRQ_LIB=checked)."""
    build_dir = BUILD + ("_checked" if checked else "")
    lib_path = LIB_CHECKED if checked else LIB
    extra = ["-DMDRQ_CHECKS"] if checked else []
    if variant:
        # experiment builds (tools/): libmdrq_b200_<variant>.so with extra
        # defines, loaded with MDRQ_LIB=<variant>; never the product library
        build_dir = BUILD + "_" + variant
        lib_path = os.path.join(PKG, f"libmdrq_b200_{variant}.so")
        extra = [f"-D{d}" for d in defines]
    os.makedirs(build_dir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "mdrq_b200.h")]
    objs = []
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([nvcc(), *NVCC_FLAGS, *extra, "-c", s, "-o", o])

    for src in HOST_SOURCES:
        sp = os.path.join(CSRC, src)
        o = os.path.join(build_dir, src.replace(".cpp", ".o"))
        objs.append(o)
        if force or _stale(o, [sp] + hdrs):
            jobs.append([shutil.which("g++") or "g++", "-O3", "-std=c++17", "-fPIC", "-pthread", "-I", INCLUDE,
                         "-c", sp, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        with open(cmd[-1] + ".ptxas.txt", "w") as fh:
            fh.write(r.stderr)

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(lib_path, objs):
        tmp = lib_path + ".tmp"
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
               "-Xcompiler", "-fPIC", "-Xlinker", "--no-undefined"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__" and "--variant" in sys.argv:
    i = sys.argv.index("--variant")
    print(build(variant=sys.argv[i + 1], defines=sys.argv[i + 2:]))
elif __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
