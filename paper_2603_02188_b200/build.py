"""Build libmlra_b200.so in-tree with nvcc for sm_100a (no torch extension machinery).

``python -m paper_2603_02188_b200.build`` or ``__graft_entry__.build()``.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmlra_b200.so")
SOURCES = ["capi.cu", "decode_inst_a.cu", "decode_inst_b.cu", "decode_inst_c.cu", "decode_inst_d.cu", "proj.cu"]
HEADERS = ["ptx.cuh", "decode_kernel.cuh", "aux_kernels.cuh", "outproj_kernel.cuh", "allreduce_kernel.cuh",
           "fused_step.cuh", "host_common.cuh", "peer_common.cuh", "proj_kernel.cuh", "prefill_kernel.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]
# dev builds only (e.g. MLRA_NVCC_DEFS=MLRA_PF_WAIT_STATS for tools/prefill_waits.py); part of the
# source hash, so a dev library is never mistaken for the product one
FLAGS += [f"-D{d}" for d in os.environ.get("MLRA_NVCC_DEFS", "").split(",") if d]
STAMP = LIB + ".srchash"  # source hash of the shipped library (travels with it)


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def source_hash() -> str:
    """SHA-256 over the sources, headers and the compile command: the shipped .so is rebuilt
    whenever any of them differs from what it was built from (mtimes do not survive a copy)."""
    h = hashlib.sha256()
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "mlra_b200.h"))
    for d in deps:
        h.update(os.path.basename(d).encode())
        with open(d, "rb") as f:
            h.update(f.read())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()


def _stale() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return True
    with open(STAMP) as f:
        return f.read().strip() != source_hash()


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every translation unit (in parallel) and link libmlra_b200.so in-tree."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        cmd = [nvcc(), *ARCH, *FLAGS, "-Xptxas", "-v" if verbose else "-O3", "-c", "-o", obj, os.path.join(CSRC, src)]
        return obj, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    for obj, res in results:
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed compiling {os.path.basename(obj)}")
        if verbose:
            sys.stderr.write(res.stderr)
    cmd = [nvcc(), *ARCH, "--shared", "-o", LIB + ".tmp", *[o for o, _ in results], "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libmlra_b200.so")
    os.replace(LIB + ".tmp", LIB)
    with open(STAMP, "w") as f:
        f.write(source_hash() + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
