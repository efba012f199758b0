"""Build libhm.so (the C-ABI of include/hm.h) in-tree with nvcc for sm_100a.

    python -m paper_1909_07909_b200.build [--force] [-DNAME=VALUE ...] [--out=PATH]

The library is plain CUDA C++ with an extern "C" surface; it links the CUDA
runtime statically and no torch library, so the ABI carries no torch type.
Every csrc/*.cu translation unit is compiled to an object in parallel, then
linked into one shared library.

Staleness: the SHA-256 of every source (csrc/*.cu, csrc/*.cuh, include/hm.h)
and of the compile flags is embedded in the library as the string
"HM_SRC_HASH=<hex>". build() rebuilds whenever the library on disk does not
carry the hash of the sources on disk, so a stale binary that travelled with a
snapshot is never the one loaded.
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhm.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]
LINK_LIBS = ["-ldl"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _inputs():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "hm.h")]


def source_hash(defines=()) -> str:
    h = hashlib.sha256()
    for f in _inputs():
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    h.update(" ".join(NVCC_FLAGS + LINK_LIBS + [f"-D{d}" for d in defines]).encode())
    return h.hexdigest()[:32]


def built_hash(path: str = LIB):
    """The HM_SRC_HASH string embedded in a built library (None if absent)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        return None
    i = data.find(b"HM_SRC_HASH=")
    if i < 0:
        return None
    return data[i + 12:i + 44].decode(errors="replace")


def needs_build(defines=()) -> bool:
    return built_hash(LIB) != source_hash(defines)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = LIB) -> str:
    """Compile every csrc/*.cu into `out` (default: the in-tree libhm.so). `defines`
    (e.g. ["HM_LEAF_PF=2"]) build development variants under another name."""
    if not force and out == LIB and not defines and not needs_build():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    digest = source_hash(defines)
    objdir = os.path.join(os.path.dirname(out), f".hm_obj_{os.getpid()}")
    os.makedirs(objdir, exist_ok=True)
    common = [*NVCC_FLAGS, *[f"-D{d}" for d in defines], f"-DHM_SRC_HASH_STR=\"HM_SRC_HASH={digest}\"",
              "-I", os.path.join(ROOT, "include")]
    log = os.path.join(PKG, "build.log")

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc, *common, "-c", "-o", obj, src]
        res = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, cmd, res

    jobs = max(1, min(len(sources()), os.cpu_count() or 1))
    with ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(compile_one, sources()))
    with open(log, "w") as f:
        for _, _, cmd, res in results:
            f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    bad = [r for r in results if r[3].returncode != 0]
    if bad:
        for _, _, _, res in bad:
            sys.stderr.write(res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    tmp = out + f".tmp{os.getpid()}"
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp,
           *[r[1] for r in results], *LINK_LIBS]
    res = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "a") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    for _, obj, _, _ in results:
        os.remove(obj)
    os.rmdir(objdir)
    if res.returncode != 0:
        sys.stderr.write(res.stderr)
        raise RuntimeError(f"nvcc link failed (see {log})")
    if verbose:
        for _, _, _, r in results:
            sys.stderr.write(r.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    defs = [a[2:] for a in args if a.startswith("-D")]
    out = next((a.split("=", 1)[1] for a in args if a.startswith("--out=")), LIB)
    print(build(force="--force" in args or out != LIB, verbose=True, defines=defs, out=out))
