"""Build libsom.so in-tree for sm_100a (nvcc; no JIT, no torch extension).

Each .cu is compiled to its own object in parallel (build/obj/), then linked
into libsom.so with nvcc -shared."""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsom.so")
OBJ = os.path.join(HERE, "build_obj")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
    "-Xptxas", "-v",
]
LINK_LIBS = ["-lnccl"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(ROOT, "include", "som.h")]


def deps():
    return sources() + headers()


def nccl_flags():
    """NCCL headers/library: the torch wheel's nvidia-nccl package (2.28) if
    present, else the system one."""
    inc, lib = [], []
    try:
        import nvidia.nccl as nn   # noqa: F401
        base = os.path.dirname(nn.__file__) if getattr(nn, "__file__", None) else list(nn.__path__)[0]
        if os.path.exists(os.path.join(base, "include", "nccl.h")):
            inc = ["-I", os.path.join(base, "include")]
            lib = ["-L", os.path.join(base, "lib"), "-Xlinker", "-rpath=" + os.path.join(base, "lib")]
            if not glob.glob(os.path.join(base, "lib", "libnccl.so")) and glob.glob(os.path.join(base, "lib", "libnccl.so.2")):
                lib = ["-Xlinker", os.path.join(base, "lib", "libnccl.so.2"), "-Xlinker",
                       "-rpath=" + os.path.join(base, "lib")]
                return inc, lib, True
    except Exception:
        pass
    return inc, lib, False


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(p) <= t for p in deps()):
            return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    os.makedirs(OBJ, exist_ok=True)
    inc, nlib, direct = nccl_flags()
    hdr_t = max(os.path.getmtime(p) for p in headers())

    def compile_one(src):
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        if (not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_t)):
            return src, 0, "", ""
        cmd = [nvcc, *NVCC_FLAGS, *inc, "-I", os.path.join(ROOT, "include"), "-c", "-o", obj + ".tmp", src]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode == 0:
            os.replace(obj + ".tmp", obj)
        return src, r.returncode, r.stdout, r.stderr

    with ThreadPoolExecutor(max_workers=max(1, min(16, os.cpu_count() or 4))) as ex:
        results = list(ex.map(compile_one, sources()))
    info = []
    failed = False
    for src, rc, out, err in results:
        if verbose or rc != 0:
            print(out[-20000:])
            print(err[-20000:])
        if rc != 0:
            failed = True
        info.append(f"==== {os.path.basename(src)}\n{err}")
    if failed:
        raise RuntimeError("nvcc failed building libsom.so")
    objs = [os.path.join(OBJ, os.path.basename(s)[:-3] + ".o") for s in sources()]
    libs = nlib if direct else nlib + LINK_LIBS
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB + ".tmp", *objs, *libs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        print(r.stdout[-20000:])
        print(r.stderr[-20000:])
    if r.returncode != 0:
        raise RuntimeError("nvcc failed linking libsom.so")
    os.replace(LIB + ".tmp", LIB)
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
        f.write("".join(i for i in info if "ptxas" in i or "Compiling" in i))
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
