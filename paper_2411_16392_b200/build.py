"""Build libqgs_b200.so in-tree (paper_2411_16392_b200/lib/) with nvcc for sm_100a.

    python -m paper_2411_16392_b200.build [--force]

The fp64 translation units (preprocess.cu, binning.cu) are compiled with
-fmad=false so that screen boxes and tile sort keys round exactly like the
reference; the raster translation unit keeps FMA contraction on.
"""

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "lib", "obj")
LIB = os.path.join(HERE, "lib", "libqgs_b200.so")
# the same sources with device bounds checks (QGS_DEBUG_CHECKS: a failed check
# traps), loaded instead of LIB when QGS_LIB_VARIANT=debug (tests only)
LIB_DEBUG = os.path.join(HERE, "lib", "libqgs_b200_debug.so")
PEAKS_LIB = os.path.join(HERE, "lib", "libqgs_peaks.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-I", INCLUDE, "-Xptxas", "-warn-spills"]
UNITS = {
    "preprocess.cu": ["-fmad=false"],
    "binning.cu": ["-fmad=false"],
    # approximate reciprocal / sqrt in the fp32 shading (every decision that
    # must match the reference is confirmed in fp64 first, see shade.cuh)
    "raster_warp.cu": ["-fmad=true", "-prec-div=false", "-prec-sqrt=false", "-ftz=true"],
    "losses.cu": ["-fmad=false"],
    "optim.cu": ["-fmad=false"],
    "multiview.cu": ["-fmad=false"],
    "det_reduce.cu": [],
    "abi.cu": [],
}


def nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, debug=None):
    """the product library, and (debug, default unless QGS_BUILD_DEBUG=0) its
    bounds-checking twin"""
    if debug is None:
        debug = os.environ.get("QGS_BUILD_DEBUG", "1") != "0"
    _build(OBJ, LIB, [], force, verbose)
    if debug:
        _build(OBJ + "_debug", LIB_DEBUG, ["-DQGS_DEBUG_CHECKS=1"], force, verbose)
    _build_peaks(force, verbose)
    return LIB


def _build(obj_dir, lib, defines, force, verbose):
    os.makedirs(obj_dir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in sorted(os.listdir(CSRC)) if h.endswith(".cuh")]
    hdrs.append(os.path.join(INCLUDE, "qgs_b200.h"))
    objs = []
    relinked = False
    extra = os.environ.get("QGS_NVCC_EXTRA", "").split()   # experiments only
    for unit, flags in UNITS.items():
        src = os.path.join(CSRC, unit)
        obj = os.path.join(obj_dir, unit.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [nvcc(), *ARCH, *COMMON, *flags, *defines, *extra, "-c", src, "-o", obj]
        # the command line is part of the object's identity: an experiment
        # build (QGS_NVCC_EXTRA) is never mistaken for the product
        stamp = obj + ".cmd"
        same_cmd = os.path.exists(stamp) and open(stamp).read() == " ".join(cmd)
        if force or not same_cmd or _stale(obj, [src] + hdrs):
            if verbose:
                print(" ".join(cmd))
            if os.path.exists(stamp):
                os.remove(stamp)
            subprocess.check_call(cmd)
            with open(stamp, "w") as f:
                f.write(" ".join(cmd))
            relinked = True
    if force or relinked or _stale(lib, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", lib, *objs]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)


def _build_peaks(force, verbose):
    # measurement helper (not part of the product ABI): FP32 / MUFU peaks
    src = os.path.join(os.path.dirname(HERE), "tools", "peaks.cu")
    if os.path.exists(src) and (force or _stale(PEAKS_LIB, [src])):
        cmd = [nvcc(), *ARCH, "-O3", "-Xcompiler", "-fPIC", "-shared", src, "-o", PEAKS_LIB]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
