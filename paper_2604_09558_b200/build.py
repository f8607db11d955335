"""Build the native library libvtc.so (C++ host + CUDA sm_100a kernels), in-tree.

Every translation unit under csrc/ is compiled by nvcc for
``-gencode arch=compute_100a,code=sm_100a`` with ``-lineinfo``; the result is
``paper_2604_09558_b200/libvtc.so`` (git-ignored, shipped to the GPU box by
gpurun).  No GPU is needed to build.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
OBJ = PKG / "build" / "obj"
LIB = PKG / "libvtc.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++20", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-Wall", f"-I{INCLUDE}", f"-I{CSRC}"]
CU_FLAGS = ["--expt-relaxed-constexpr", "-Xptxas", "-O3"]


def _sources():
    return sorted(list(CSRC.glob("*.cpp")) + list(CSRC.glob("*.cu")))


def _headers_digest() -> str:
    h = hashlib.sha256()
    for p in sorted(list(CSRC.glob("*.h*")) + list(CSRC.glob("*.cuh")) + list(INCLUDE.rglob("*.h*"))):
        h.update(p.read_bytes())
    return h.hexdigest()[:16]


def _compile(src: Path, hdr: str, verbose: bool) -> Path:
    obj = OBJ / (src.name + ".o")
    stamp = OBJ / (src.name + ".stamp")
    key = hashlib.sha256(src.read_bytes() + hdr.encode() + " ".join(ARCH + COMMON + CU_FLAGS).encode()).hexdigest()
    if obj.exists() and stamp.exists() and stamp.read_text() == key:
        return obj
    cmd = [NVCC, *ARCH, *COMMON]
    if src.suffix == ".cu":
        cmd += CU_FLAGS
    cmd += ["-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and verbose:
        print(r.stderr, file=sys.stderr)
    stamp.write_text(key)
    return obj


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    hdr = _headers_digest()
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, hdr, verbose), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if not LIB.exists() or LIB.stat().st_mtime < newest:
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
