"""Build libprism_b200.so in-tree with nvcc for sm_100a (the .so travels to the GPU box).

Every source is compiled to its own object in parallel (the cell kernel's variants live in separate
cells_k_*.cu units), then linked with nvcc -shared. Objects are cached under build/ and rebuilt
when their source, any header of csrc/ or include/prism.h, or the flags change.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(_HERE, "csrc")
OUT = os.path.join(_HERE, "libprism_b200.so")
OBJ = os.path.join(_HERE, "..", "build", "obj")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(_HERE, "..", "include", "prism.h")])


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(d) > t for d in sources() + _headers())


def _key(src: str, extra) -> str:
    h = hashlib.sha1()
    for p in [src] + _headers():
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(NVCC_FLAGS + list(extra)).encode())
    return h.hexdigest()[:16]


def build(force: bool = False, verbose: bool = False, extra=()) -> str:
    """extra: additional nvcc flags (e.g. -DPRISM_CELL_STATS for the tools/ probes)."""
    if not force and not _stale():
        return OUT
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    os.makedirs(OBJ, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(OBJ, f"{os.path.basename(src)}.{_key(src, extra)}.o")
        if os.path.exists(obj):
            return obj, ""
        tmp = obj + f".tmp{os.getpid()}"
        res = subprocess.run([nvcc, *NVCC_FLAGS, *extra, "-Xptxas", "-v", "-c", src, "-o", tmp],
                             capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n" + res.stdout + res.stderr)
        os.replace(tmp, obj)
        return obj, res.stderr

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(sources()), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, sources()))
    keep = {os.path.abspath(o) for o, _ in results}
    for old in glob.glob(os.path.join(OBJ, "*.o")):  # objects of earlier sources / flags
        if os.path.abspath(old) not in keep:
            try:
                os.remove(old)
            except OSError:
                pass
    tmp = OUT + f".tmp{os.getpid()}"
    res = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp,
                          *[o for o, _ in results]], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + res.stdout + res.stderr)
    if verbose:
        for _, log in results:
            if log:
                print(log)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
