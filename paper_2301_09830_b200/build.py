"""Builds libocc.so (the C-ABI library of include/occ.h) in-tree for sm_100a.

    python -m paper_2301_09830_b200.build [--force] [--trace]

--trace also builds libocc_trace.so: the same library compiled with
-DOCC_TRACE (per-CTA phase stamps for tools/trace.py).  The product library
carries no instrumentation.

nvcc cross-compiles without a GPU.  The NCCL it links is the one bundled with
torch (nvidia/nccl), found through an rpath so that the process shares a
single libnccl.so.2 with torch.distributed.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libocc.so")
LIB_TRACE = os.path.join(HERE, "libocc_trace.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("occ_api.cu", "occ_step.cu", "occ_v2.cu", "occ_umma.cu")] + \
    [os.path.join(HERE, "csrc", f"occ_step_r{r}.cu") for r in (4, 8, 16, 32, 64)]
DEPS = SOURCES + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + \
    glob.glob(os.path.join(HERE, "csrc", "*.h")) + [os.path.join(ROOT, "include", "occ.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return c
    raise RuntimeError("torch-bundled NCCL (nvidia/nccl) not found")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(d) <= t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    """Compiles every source to an object in parallel (one nvcc per .cu), then
    links libocc.so; objects whose inputs did not change are reused."""
    from concurrent.futures import ThreadPoolExecutor
    lib = LIB_TRACE if trace else LIB
    if not force and up_to_date(lib):
        return lib
    nd = nccl_dir()
    objdir = os.path.join(HERE, "build", "trace" if trace else "prod")
    os.makedirs(objdir, exist_ok=True)
    common = [nvcc(), *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
              *(["-DOCC_TRACE"] if trace else []),
              "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(nd, "include")]
    if verbose:
        common.insert(1, "-Xptxas=-v")
    headers = [d for d in DEPS if not d.endswith(".cu")]
    newest_hdr = max((os.path.getmtime(h) for h in headers if os.path.exists(h)), default=0)

    def obj(src):
        o = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(src), newest_hdr):
            cmd = common + ["-c", src, "-o", o + ".tmp"]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
            os.replace(o + ".tmp", o)
        return o

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(obj, SOURCES))
    tmp = lib + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-L" + os.path.join(nd, "lib"), "-l:libnccl.so.2",
           "-Xlinker", "-rpath," + os.path.join(nd, "lib"), "-o", tmp]
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
    if "--trace" in sys.argv:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace=True))
