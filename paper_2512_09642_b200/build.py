"""Build libsscg.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2512_09642_b200.build [--force]

The library links cudart statically, and NCCL from the pip wheel torch also
loads (same soname, so one NCCL per process).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libsscg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        inc, lib = os.path.join(base, "nccl", "include"), os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "sscg.h"), __file__]


def build(force: bool = False, verbose: bool = False, defs=(), variant: str = "") -> str:
    """Compile libsscg.so; with `variant`, compile libsscg_<variant>.so with the
    extra -D flags `defs` (tuning experiments; load it with SSCG_LIB=<path>)."""
    lib = os.path.join(HERE, "libsscg_%s.so" % variant) if variant else LIB
    bdir = os.path.join(BUILD, variant) if variant else BUILD
    if not force and os.path.exists(lib):
        t = os.path.getmtime(lib)
        if all(os.path.getmtime(d) <= t for d in deps()):
            return lib
    os.makedirs(bdir, exist_ok=True)
    inc, libdir = nccl_dirs()
    common = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
                     "-I", inc, "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]
    if verbose:
        common += ["-Xptxas", "-v"]
    common += list(defs)
    objs = [os.path.join(bdir, os.path.basename(src) + ".o") for src in sources()]
    cmds = [[NVCC] + common + ["-c", src, "-o", obj] for src, obj in zip(sources(), objs)]
    # one nvcc per source, in parallel (each is single-threaded)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
        list(ex.map(subprocess.check_call, cmds))
    link = [NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-L", libdir, "-l:libnccl.so.2",
                                                           "-Xlinker", "-rpath=" + libdir, "-cudart", "static"]
    subprocess.check_call(link)
    return lib


if __name__ == "__main__":
    a = sys.argv[1:]
    var = a[a.index("--variant") + 1] if "--variant" in a else ""
    print(build(force="--force" in a or bool(var), verbose="-v" in a, defs=[x for x in a if x.startswith("-D")],
                variant=var))
