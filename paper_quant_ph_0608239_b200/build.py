"""Build libqsim_b200.so in-tree: nvcc for sm_100a (+ g++ for the host C++).

    python -m paper_quant_ph_0608239_b200.build [--force]
"""
from __future__ import annotations

import importlib.util
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
# QSB_BUILD_TAG=<t>: an experiment build (e.g. QSB_TILE_BITS=13) into
# _build_<t>/ and libqsim_b200_<t>.so, loaded with QSIM_LIB=<that path>
_TAG = os.environ.get("QSB_BUILD_TAG", "")
BUILD = os.path.join(HERE, "_build" + ("_" + _TAG if _TAG else ""))
LIB = os.path.join(HERE, "libqsim_b200" + ("_" + _TAG if _TAG else "") + ".so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    spec = importlib.util.find_spec("nvidia")
    for loc in (spec.submodule_search_locations or []) if spec else []:
        d = os.path.join(loc, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("NCCL headers not found (expected the torch-bundled nvidia/nccl)")


def _sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
            if f.endswith((".cu", ".cpp", ".h"))] + [os.path.join(INCLUDE, "qsim.h")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in _sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    nccl = nccl_dir()
    tile = os.environ.get("QSB_TILE_BITS")
    regs = os.environ.get("QSB_REG_BITS")
    defs = (["-DQSB_TILE_BITS=" + tile] if tile else []) + (["-DQSB_REG_BITS=" + regs] if regs else [])
    inc = [*defs, "-I", CSRC, "-I", INCLUDE, "-I", os.path.join(nccl, "include"), "-I", os.path.join(CUDA, "include")]
    objs = []
    cmds = []
    for f in sorted(os.listdir(CSRC)):
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, f + ".o")
        if f.endswith(".cu"):
            cmds.append([os.path.join(CUDA, "bin", "nvcc"), *ARCH, "-lineinfo", "-O3", "-std=c++17",
                         "-Xcompiler", "-fPIC", "-Xptxas", "-v", *inc, "-c", src, "-o", obj])
        elif f.endswith(".cpp"):
            cmds.append(["g++", "-O2", "-std=c++17", "-fPIC", "-Wall", "-Werror=return-type", "-Wno-unused-function", *inc,
                         "-c", src, "-o", obj])
        else:
            continue
        objs.append(obj)
    for c in cmds:
        r = subprocess.run(c, capture_output=True, text=True)
        if verbose or r.returncode != 0:
            sys.stderr.write(" ".join(c) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {c[-3]}")
        if "-Xptxas" in c:
            with open(os.path.join(BUILD, "ptxas.log"), "w") as fh:
                fh.write(r.stderr)
    link = ["g++", "-shared", "-o", LIB + ".tmp", *objs,
            "-L", os.path.join(CUDA, "lib64"), "-lcudart_static", "-lrt", "-ldl", "-lpthread",
            "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2", "-Wl,-rpath," + os.path.join(nccl, "lib"),
            "-ldl"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(link) + "\n" + r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
