"""Build libwalklap.so in-tree with nvcc for sm_100a (no torch extension machinery: the
library is a plain C ABI; the Python binding uses ctypes)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIB_DIR, "libwalklap.so")


def nccl_paths():
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is not None and spec.submodule_search_locations:
        d = list(spec.submodule_search_locations)[0]
        inc, lib = os.path.join(d, "include"), os.path.join(d, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "walklap.h")]
    return any(os.path.getmtime(f) > t for f in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every csrc/*.cu to an object in parallel (nvcc -c, sm_100a), then link the shared library."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(LIB_DIR, exist_ok=True)
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    inc, libdir = nccl_paths()
    tag = f"tmp{os.getpid()}"
    flags = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
             "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
             "-I", os.path.join(ROOT, "include"), "-I", inc,
             *os.environ.get("WL_EXTRA_NVCC", "").split()]  # developer experiments (e.g. -DWL_SPMV_HINTS=1)
    objs = [os.path.join(LIB_DIR, os.path.basename(src)[:-3] + f".{tag}.o") for src in sources()]

    def compile_one(job):
        src, obj = job
        cmd = [nvcc, *flags, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0 or verbose:
            sys.stderr.write(r.stdout + r.stderr)
        return r.returncode

    try:
        with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
            rcs = list(ex.map(compile_one, zip(sources(), objs)))
        if any(rcs):
            raise subprocess.CalledProcessError(max(rcs), "nvcc -c")
        tmp = LIB + f".{tag}"
        cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", tmp,
               "-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath={libdir}"]
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
