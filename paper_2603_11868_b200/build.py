"""Build libsphb200.so (sm_100a) in-tree with nvcc.

``python -m paper_2603_11868_b200.build`` or ``build_library()``.  Each .cu
compiles in parallel to an object, then links into
``paper_2603_11868_b200/_lib/libsphb200.so``.  Flags: ``--fmad=false`` (no
FMA contraction; the kernels also use explicit round-to-nearest intrinsics),
IEEE division / square root (nvcc defaults, stated explicitly), -lineinfo for
ncu source mapping.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libsphb200.so")
# the same sources with periodic boxes compiled in (common.cuh SPH_PERIODIC)
LIB_PERIODIC = os.path.join(OUT_DIR, "libsphb200_periodic.so")
PERIODIC_FLAGS = ("-DSPH_PERIODIC=1",)
OBJ_DIR = os.path.join(ROOT, "build", "obj")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "--fmad=false", "-prec-div=true", "-prec-sqrt=true",
    "-ftz=false", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas",
    "-warn-spills", "--expt-relaxed-constexpr",
    "-I" + os.path.join(ROOT, "include"),
]


def nvcc():
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found; cannot build libsphb200.so")
    return path


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith(".cu"))


def _deps():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(ROOT, "include", "sph_b200.h"))
    files.append(os.path.abspath(__file__))
    return files


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_library(force=False, verbose=False, extra_flags=(), out=None):
    """Build the library (to `out`, default the in-tree path; the default
    build also produces the periodic-box variant)."""
    if out is None and not extra_flags:
        # both libraries at once: their engine.cu compiles are the long poles
        with cf.ThreadPoolExecutor(max_workers=2) as ex:
            per = ex.submit(_build_one, force, verbose, PERIODIC_FLAGS, LIB_PERIODIC)
            lib = ex.submit(_build_one, force, verbose, extra_flags, out)
            per.result()
            return lib.result()
    return _build_one(force, verbose, extra_flags, out)


def _build_one(force, verbose, extra_flags, out):
    deps = _deps()
    target = out or LIB
    if not force and not _stale(target, deps):
        return target
    os.makedirs(os.path.dirname(target), exist_ok=True)
    obj_dir = OBJ_DIR if out is None else os.path.join(
        OBJ_DIR, os.path.basename(os.path.dirname(target)))
    os.makedirs(obj_dir, exist_ok=True)
    exe = nvcc()
    flags = NVCC_FLAGS + list(extra_flags)

    def compile_one(src):
        obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
        cmd = [exe] + flags + ["-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr.strip():
            print(r.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = target + ".tmp"
    cmd = [exe] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose=True))
