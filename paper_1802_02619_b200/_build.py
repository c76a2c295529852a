"""In-tree build of liblco.so for sm_100a (nvcc; no JIT cache, the .so travels with the
repo snapshot to the GPU box).

Every source is compiled to its own object in parallel, then linked.  Freshness is a
content hash (sources, headers, flags) stored beside the library, never file times:
``up_to_date()`` is false as soon as any input differs from what the .so was built from,
and ``lco.lib()`` rebuilds a stale library before loading it."""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "liblco.so")
STAMP = LIB + ".sha256"
OBJ = os.path.join(ROOT, "build", "obj")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-fvisibility=hidden"]
LINK_FLAGS = [*ARCH, "-shared", "--cudart", "static"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _inputs():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.h")) +
                              glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(ROOT, "include", "lco.h")]


def digest() -> str:
    h = hashlib.sha256()
    h.update(" ".join(NVCC_FLAGS + LINK_FLAGS).encode())
    for p in _inputs():
        h.update(os.path.relpath(p, ROOT).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def up_to_date() -> bool:
    if not (os.path.exists(LIB) and os.path.exists(STAMP)):
        return False
    with open(STAMP) as f:
        return f.read().strip() == digest()


def _nvcc():
    nvcc = os.environ.get("NVCC", "nvcc")
    if os.path.sep not in nvcc and os.path.exists("/usr/local/cuda/bin/nvcc"):
        nvcc = "/usr/local/cuda/bin/nvcc"
    return nvcc


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    want = digest()
    nvcc = _nvcc()
    os.makedirs(OBJ, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include")]

    def compile_one(src):
        obj = os.path.join(OBJ, os.path.basename(src) + f".{os.getpid()}.o")
        cmd = [nvcc, *NVCC_FLAGS, *inc, "-c", "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        return obj

    srcs = sources()
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc, *LINK_FLAGS, "-o", tmp, *objs])
    for o in objs:
        os.remove(o)
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write(want + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
