"""Build libplenoct.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache)."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libplenoct.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-shared", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")) + glob.glob(os.path.join(PKG, "csrc", "*.cuh"))
                  + glob.glob(os.path.join(PKG, "csrc", "*.h")) + [os.path.join(ROOT, "include", "plenoct.h")])


STAMP = LIB + ".flags"   # the extra nvcc flags the library was built with (e.g. -DPO_DIAG)
PTXAS_INFO = os.path.join(ROOT, "build", "ptxas_info.txt")   # untracked (build/ is git-ignored)


def _extra():
    return os.environ.get("PO_NVCC_EXTRA", "").split()   # -DPO_DIAG: diagnostics build


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    try:
        with open(STAMP) as f:
            if f.read().split() != _extra():
                return True
    except OSError:
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    cu = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))
    tmp = LIB + f".tmp{os.getpid()}"
    extra = _extra()
    cmd = [NVCC, *FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-I", os.path.join(PKG, "csrc"), *cu, "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    if verbose:
        print(res.stderr)
    os.makedirs(os.path.dirname(PTXAS_INFO), exist_ok=True)
    with open(PTXAS_INFO, "w") as f:
        f.write(res.stderr)
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write(" ".join(extra))
    return LIB


EXAMPLE_SRC = os.path.join(ROOT, "examples", "render_uniform.c")
EXAMPLE_BIN = os.path.join(ROOT, "examples", "render_uniform")


def build_example() -> str:
    """The plain-C example against include/plenoct.h + libplenoct.so (no CUDA headers)."""
    lib = build()
    if os.path.exists(EXAMPLE_BIN) and os.path.getmtime(EXAMPLE_BIN) >= max(os.path.getmtime(EXAMPLE_SRC),
                                                                         os.path.getmtime(lib)):
        return EXAMPLE_BIN
    cmd = ["gcc", "-O2", "-Wall", "-Wextra", "-Werror", EXAMPLE_SRC, "-I", os.path.join(ROOT, "include"), "-L", PKG,
           "-lplenoct", "-Wl,-rpath,$ORIGIN/../paper_2103_14024_b200", "-lm", "-o", EXAMPLE_BIN]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("gcc failed on the C example:\n" + res.stdout + res.stderr)
    return EXAMPLE_BIN


if __name__ == "__main__":
    print(build(force=True, verbose=True))
