"""Builds the sm_100a shared library libp2s.so in-tree (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libp2s.so")
LIB_PROF = os.path.join(PKG, "libp2s_prof.so")  # -DP2S_PROFILE variant (tools only)
SOURCES = [os.path.join(CSRC, "p2s_host.cu"), os.path.join(CSRC, "p2s_sampler.cu"), os.path.join(CSRC, "p2s_anchor.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("p2s_kernels.cuh", "sm100.cuh", "p2s_adjoint.cuh", "p2s_mlp_backward.cuh")] + \
    [os.path.join(ROOT, "include", "p2s.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-Xptxas", "-v", "-maxrregcount=144", f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]


def build(force: bool = False, verbose: bool = False, profile: bool = False) -> str:
    lib = LIB_PROF if profile else LIB
    stale = force or not os.path.exists(lib) or \
        any(os.path.getmtime(d) > os.path.getmtime(lib) for d in DEPS)
    if not stale:
        return lib
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, *(["-DP2S_PROFILE"] if profile else []), *SOURCES, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libp2s.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, lib)
    return lib


EXAMPLE_SRC = os.path.join(ROOT, "examples", "render_c_abi.c")
EXAMPLE_BIN = os.path.join(ROOT, "examples", "render_c_abi")


def build_example() -> str:
    """Compiles examples/render_c_abi.c, a plain-C client of the C ABI (gcc, no C++/PyTorch)."""
    cuda = os.path.dirname(os.path.dirname(NVCC))
    cmd = ["gcc", "-O2", "-std=c99", "-Wall", f"-I{os.path.join(ROOT, 'include')}", f"-I{cuda}/include",
           EXAMPLE_SRC, f"-L{PKG}", "-lp2s", f"-L{cuda}/lib64", "-lcudart", "-lm",
           "-Wl,-rpath,$ORIGIN/../paper_2107_11627_b200", f"-Wl,-rpath,{cuda}/lib64", "-o", EXAMPLE_BIN]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("gcc failed building examples/render_c_abi")
    return EXAMPLE_BIN


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, profile="--profile" in sys.argv))
