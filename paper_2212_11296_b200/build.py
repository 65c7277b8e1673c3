"""In-tree build of the native library (sm_100a only).

``python -m paper_2212_11296_b200.build`` compiles csrc/ into
``paper_2212_11296_b200/_lib/libvqnqs_b200.so`` with nvcc. The .so is
git-ignored but travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libvqnqs_b200.so")
SOURCES = ["engine.cu", "grad.cu", "capi.cpp", "host_model.cpp", "comm.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "vqnqs_b200.h"))
    if not force and _newer(LIB, deps):
        return LIB
    cmds, objs = [], []
    for src in SOURCES:
        obj = os.path.join(LIBDIR, src + ".o")
        cmd = [nvcc(), *ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
               "-Xcompiler", "-O3", "-I", os.path.join(ROOT, "include"), "-c",
               os.path.join(CSRC, src), "-o", obj]
        # developer instrumentation switches (e.g. -DVQNQS_ATTN_TRACE)
        cmd[1:1] = os.environ.get("VQNQS_EXTRA_NVCC", "").split()
        if src.endswith(".cu"):
            cmd[1:1] = ["--expt-relaxed-constexpr", "-Xptxas", "-v"] if verbose else \
                ["--expt-relaxed-constexpr"]
        else:
            cmd[1:1] = ["-x", "cu"] if False else []
        if verbose:
            print(" ".join(cmd), flush=True)
        cmds.append(cmd)
        objs.append(obj)
    # the translation units compile in parallel (engine.cu dominates)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(len(cmds)) as ex:
        for r in ex.map(lambda c: subprocess.run(c, check=True), cmds):
            pass
    tmp = LIB + ".tmp"
    subprocess.run([nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-ldl"],
                   check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
