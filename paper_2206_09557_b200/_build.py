"""Build liblutgemm.so in-tree with nvcc for sm_100a (no torch needed).

    python paper_2206_09557_b200/_build.py [--verbose] [--force]

Compiles every csrc/*.cu to an object in parallel, then links one shared
library against the CUDA runtime and the NCCL that PyTorch ships (pip
nvidia-nccl, 2.28.x) so a process never holds two libnccl.so.2.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "liblutgemm.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs() -> tuple[str, str]:
    cands = [os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl")]
    try:
        import nvidia  # type: ignore

        for p in getattr(nvidia, "__path__", []):
            cands.append(os.path.join(p, "nccl"))
    except Exception:
        pass
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")) and os.path.exists(os.path.join(c, "lib", "libnccl.so.2")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    raise RuntimeError("pip NCCL (nvidia/nccl) not found; cannot build the TP part of liblutgemm")


def nvcc() -> str:
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if p and os.path.exists(p):
            return p
    return "nvcc"


FLAGS = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr"]
HASH_MARK = b"LUTGEMM_SRC_HASH:"


def source_files() -> list[str]:
    srcs = glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(INCLUDE, "lutgemm.h")]
    return sorted(srcs)


def source_hash() -> str:
    """sha256 (first 24 hex digits) over every source file's name and bytes and the compile flags:
    embedded in the library (lutgemm_source_hash) so a loaded .so provably matches the tree."""
    h = hashlib.sha256()
    for p in source_files():
        h.update(os.path.basename(p).encode() + b"\0")
        with open(p, "rb") as f:
            h.update(f.read())
        h.update(b"\0")
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()[:24]


def library_hash(path: str = LIB) -> str | None:
    """The source hash embedded in a built library (None if absent or unmarked)."""
    if not os.path.exists(path):
        return None
    with open(path, "rb") as f:
        data = f.read()
    i = data.find(HASH_MARK)
    if i < 0:
        return None
    return data[i + len(HASH_MARK):i + len(HASH_MARK) + 24].decode(errors="replace")


def build(verbose: bool = False, force: bool = False) -> str:
    """Compile unless the library already embeds the hash of the current sources (force: always)."""
    os.makedirs(BUILD, exist_ok=True)
    inc, lib = nccl_dirs()
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    want = source_hash()
    if not force and library_hash() == want:
        return LIB
    flags = [*FLAGS, "-I", INCLUDE, "-I", CSRC, "-I", inc, f"-DLUTGEMM_SOURCE_HASH=\"{want}\""]

    def compile_one(src: str) -> tuple[str, str]:
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        cmd = [nvcc(), *flags, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        return obj, r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, srcs))
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    objs = [o for o, _ in results]
    tmp = LIB + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-L", lib, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath,{lib}", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force="--force" in sys.argv))
