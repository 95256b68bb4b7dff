"""Build the sm_100a shared library libsemd_b200.so in-tree (nvcc, no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.dirname(HERE)
LIB = os.path.join(PKG, "libsemd_b200.so")
SRCS = ["semd_eval.cu", "semd_sift.cu", "semd_aux.cu", "semd_resident.cu", "semd_capi.cu"]
HDRS = ["semd_types.cuh", "semd_device.cuh", "semd_launch.h", "semd_libm.cuh", "semd_libm_tables.h", "semd_libm.cuh", "semd_libm_tables.h", os.path.join("..", "..", "include", "semd_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# -fmad=false: the sift arithmetic must round exactly like the reference's
# -ffp-contract=off build (bit-exact parity); FMA is used only where written.
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "--expt-relaxed-constexpr"]


def needs_build() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(os.path.join(PKG, "semd-cli")):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(os.path.join(HERE, f)) > t for f in SRCS + HDRS + ["semd_cli.cpp"])


CHECKED = os.path.join(PKG, "libsemd_b200_checked.so")


def build_checked(verbose: bool = False) -> str:
    """The bounds-checked variant (-DSEMD_CHECK: SEMD_ASSERT traps; tests/test_gpu_checked.py)."""
    if os.path.exists(CHECKED) and os.path.getmtime(CHECKED) >= max(
            os.path.getmtime(os.path.join(HERE, f)) for f in SRCS + HDRS):
        return CHECKED
    return build(force=True, verbose=verbose, checked=True)


TOL = os.path.join(PKG, "libsemd_b200_tol.so")


def build_tol(verbose: bool = False) -> str:
    """EXPERIMENT ONLY (tests/probes/tol_experiment.py): the engine with a
    tolerance-mode spline (-DSEMD_TOL_SPLINE: reciprocal multiplications and FMAs instead of the
    correctly rounded divisions). Not loaded by the package; select it with SEMD_LIB."""
    return build(force=True, verbose=verbose, variant="tol")


def build(force: bool = False, verbose: bool = False, checked: bool = False, variant: str = "") -> str:
    if not force and not needs_build():
        return LIB
    objs = []
    tol = variant == "tol"
    for src in SRCS:
        obj = os.path.join(HERE, src.replace(".cu", "_chk.o" if checked else ("_tol.o" if tol else ".o")))
        cmd = [NVCC, *FLAGS, *(["-DSEMD_CHECK"] if checked else []), *(["-DSEMD_TOL_SPLINE"] if tol else []), "-c",
               os.path.join(HERE, src), "-o", obj]
        if verbose:
            print(" ".join(cmd))
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        objs.append(obj)
    out = CHECKED if checked else (TOL if tol else LIB)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out + ".tmp", *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(out + ".tmp", out)
    if not checked and not tol:
        build_cli(verbose)
    return out


CLI = os.path.join(PKG, "semd-cli")
INC = os.path.join(PKG, "..", "include")


def build_cli(verbose: bool = False) -> str:
    """The reference's `decompose` front-end (semd_cli.cpp) linked against libsemd_b200.so."""
    cmd = ["g++", "-std=c++20", "-O2", "-I" + INC, os.path.join(HERE, "semd_cli.cpp"), "-o", CLI + ".tmp",
           "-L" + PKG, "-lsemd_b200", "-Wl,-rpath,$ORIGIN"]
    if verbose:
        print(" ".join(cmd))
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"semd-cli build failed:\n{r.stdout}\n{r.stderr}")
    os.replace(CLI + ".tmp", CLI)
    return CLI


if __name__ == "__main__":
    if "--checked" in sys.argv:
        print(build_checked(verbose=True))
    elif "--tol" in sys.argv:
        print(build_tol(verbose=True))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
