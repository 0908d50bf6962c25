"""Build libipm.so in-tree with nvcc for sm_100a (no JIT, no CPU fallback)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libipm.so")
SOURCES = ["ipm_kernels.cu", "ipm_api.cu", "ipm_mesh.cpp"]
DEPS = SOURCES + ["ipm_device.cuh", "ipm_internal.h", "ipm_dual_group.cuh", "ipm_dual_mma.cuh", "ipm_dual_big.cuh", "ipm_dual_lbfgs.cuh", "ipm_flux_strip.cuh", "ipm_host.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-shared",
         "-I", os.path.join(ROOT, "include")]


STAMP = LIB + ".cmd"  # the exact nvcc command the product library was built with


def product_cmd(out: str) -> list:
    return [NVCC, *FLAGS, *[os.path.join(CSRC, s) for s in SOURCES], "-o", out]


def stale() -> bool:
    """rebuild when a source is newer than the library OR the library was built with other flags
    (e.g. an instrumented experiment written over it): the stamp must hold the product command"""
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return True
    if open(STAMP).read() != " ".join(product_cmd("libipm.so")):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, d) for d in DEPS] + [os.path.join(ROOT, "include", "ipm.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, timers: bool = False, variant: str = "",
          defines=()) -> str:
    """variant/defines: experimental builds (libipm_<variant>.so), never the product default."""
    if defines and not (variant or timers):
        raise ValueError("experimental -D defines build libipm_<variant>.so (--variant=...), never the product")
    name = "libipm_timers.so" if timers else (f"libipm_{variant}.so" if variant else "libipm.so")
    lib = os.path.join(HERE, name)
    if not force and not timers and not variant and not stale():
        return LIB
    tmp = lib + f".tmp{os.getpid()}"
    extra = (["-DIPM_PHASE_TIMERS"] if timers else []) + [f"-D{d}" for d in defines]
    cmd = [NVCC, *FLAGS, *extra, *[os.path.join(CSRC, s) for s in SOURCES], "-o", tmp]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    if lib == LIB:
        with open(STAMP, "w") as f:
            f.write(" ".join(product_cmd("libipm.so")))
    elif os.path.exists(STAMP) and os.path.abspath(lib) == os.path.abspath(LIB):
        os.remove(STAMP)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    var = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--variant=")), "")
    print(build(force="--force" in sys.argv, verbose=True, timers="--timers" in sys.argv, variant=var, defines=defs))
