"""Build librsk.so in-tree with nvcc for sm_100a (explicit -gencode, -lineinfo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librsk.so")
SOURCES = ["apply.cu", "apply_strip.cu", "apply_rank2.cu", "cg_persist.cu", "cg_stream.cu", "cg_cluster.cu", "vec.cu", "cg_group.cu", "rsk.cu", "minres.cu", "ct.cu", "host_dense.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "rsk.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objs = []
    os.makedirs(os.path.join(HERE, "build"), exist_ok=True)
    cmds = []
    for src in SOURCES:
        obj = os.path.join(HERE, "build", src + ".o")
        extra = os.environ.get("RSK_NVCC_DEFS", "").split()   # e.g. -DRSK_STRIP_PROF (probes)
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", *extra, "-Xcompiler", "-fPIC,-O3",
               "-Xptxas", "-v" if verbose else "-O3", "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC, "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-x", "c++", "-c",
                   os.path.join(CSRC, src), "-o", obj]
        cmds.append((src, cmd))
        objs.append(obj)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(cmds)) as ex:
        results = list(ex.map(lambda sc: (sc[0], subprocess.run(sc[1], capture_output=True, text=True)), cmds))
    for src, r in results:
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
