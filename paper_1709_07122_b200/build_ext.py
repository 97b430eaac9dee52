"""Compile the CUDA sources under csrc/ into the in-tree libpcpm.so (sm_100a).

    python -m paper_1709_07122_b200.build_ext        # or __graft_entry__.build()
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libpcpm.so")
# A/B variants: PCPM_NVCC_DEFS="-DX=1" builds with extra defines into PCPM_LIB (default LIB)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in sources() + headers() + [__file__])


def build(force: bool = False, verbose: bool = False, lib: str = "", defs=()) -> str:
    lib = lib or LIB
    if not defs and lib == LIB and not force and not needs_build():
        return LIB
    objdir = os.path.join(HERE, "build_obj" + ("_" + os.path.basename(lib).replace(".so", "") if defs else ""))
    os.makedirs(objdir, exist_ok=True)
    common = ARCH + list(defs) + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                     "-I", os.path.join(ROOT, "include"), "-Xptxas", "-v" if verbose else "-O3"]
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        objs.append(obj)
        procs.append((src, subprocess.Popen([NVCC, "-c", src, "-o", obj] + common,
                                            stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = False
    for src, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            failed = True
            sys.stderr.write(f"nvcc failed for {src}:\n{out}\n")
        elif verbose and out:
            sys.stderr.write(out)
    if failed:
        raise RuntimeError("CUDA build failed")
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, "-shared", "-o", tmp] + objs + ARCH + ["-Xcompiler", "-fPIC"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python -m paper_1709_07122_b200.build_ext [--force] [-v] [--lib out.so -DNAME=V ...]
    lib = sys.argv[sys.argv.index("--lib") + 1] if "--lib" in sys.argv else ""
    defs = [a for a in sys.argv[1:] if a.startswith("-D")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, lib=lib, defs=defs))
